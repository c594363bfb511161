set -x
python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg2.log 2>&1
python tools/stage_profile.py cfg2 > gpurun_out/stages_cfg2.txt 2>&1
for k in rl_sweep lr_sweep adj_sweep; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -f -o gpurun_out/$k.cfg2 \
    python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
tail -2 gpurun_out/b_cfg2.log
