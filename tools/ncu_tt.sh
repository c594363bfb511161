set -u
mkdir -p gpurun_out/ev
ncu --set full --import-source on --clock-control none -k regex:tt_kernel -s 3 -c 1 -f -o /tmp/tt_f3 \
    python bench.py --config f3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev/tt_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/tt_f3.ncu-rep > gpurun_out/ev/ncu_tt_f3.txt 2>&1
python tools/ncu_lines.py /tmp/tt_f3.ncu-rep "tt_kernel" paper_2112_10239_b200/libtq_engine.so 30 >> gpurun_out/ev/ncu_tt_f3.txt 2>&1
