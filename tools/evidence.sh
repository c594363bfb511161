#!/bin/bash
# Round evidence on one GPU (round 2): the GPU suite, bench lines for every config (CPU baselines
# included), reference arms, stage profiles, the ncu launch list of the default bench command and
# full ncu captures of the hot kernels.  Text/JSON only comes back (gpurun_out/ev/).
set -u
mkdir -p gpurun_out/ev
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/ev/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ev/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev/smoke.txt
for c in cfg4 cfg2 cfg1 cfg3 cfg5 f3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/ev/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/ev/bench_$c.log > gpurun_out/ev/bench_$c.json
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_reference_cfg4.log 2>&1; echo "ref cfg4 rc=$?"
tail -1 gpurun_out/ev/bench_reference_cfg4.log > gpurun_out/ev/bench_reference_cfg4.json
timeout 900 python bench.py --impl reference --config cfg2 --steps 3 --warmup 1 > gpurun_out/ev/bench_reference_cfg2.log 2>&1; echo "ref cfg2 rc=$?"
tail -1 gpurun_out/ev/bench_reference_cfg2.log > gpurun_out/ev/bench_reference_cfg2.json
timeout 900 python bench.py --impl reference --config f3 --steps 2 --warmup 1 > gpurun_out/ev/bench_reference_f3.log 2>&1; echo "ref f3 rc=$?"
tail -1 gpurun_out/ev/bench_reference_f3.log > gpurun_out/ev/bench_reference_f3.json
python tools/stage_profile.py cfg4 > gpurun_out/ev/stages_cfg4.txt 2>&1
python tools/stage_profile.py cfg2 > gpurun_out/ev/stages_cfg2.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
cap() {  # cap <config> <kernel-regex> <name>
  ncu --set full --import-source on --clock-control none -k regex:$2 -s 3 -c 1 -f -o /tmp/$3 \
    python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $3 rc=$?"
  python tools/ncu_summary.py /tmp/$3.ncu-rep > gpurun_out/ev/ncu_$3.txt 2>&1
  python tools/ncu_lines.py /tmp/$3.ncu-rep "$2" paper_2112_10239_b200/libtq_engine.so 30 >> gpurun_out/ev/ncu_$3.txt 2>&1
}
python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && {
  cap cfg4 rl_sweep rl_cfg4
  cap cfg4 lr_sweep lr_cfg4
  cap cfg4 adj_sweep adj_cfg4
}
python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && {
  cap cfg2 rl_sweep rl_cfg2
  cap cfg2 lr_sweep lr_cfg2
  cap cfg2 adj_sweep adj_cfg2
}
python bench.py --config f3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && cap f3 tt_kernel tt_f3
ls -la gpurun_out/ev
