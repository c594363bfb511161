#!/bin/bash
# ncu --set full captures of the three sweep kernels for one config (default cfg2).
C=${1:-cfg2}
for k in rl_sweep lr_sweep adj_sweep; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -f -o gpurun_out/$k.$C \
    python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.$C.log 2>&1
  echo "$k rc=$?"
done
