#!/bin/bash
# A/B of engine build variants on one box: bash tools/exp_variant.sh CONFIG "v0 v1 ..." [STAGECFG]
# (libtq_engine_<v>.so and libtq_engine_timing_<v>.so built beforehand with the variant's -D flags)
D=paper_2112_10239_b200
CFG=${1:-cfg2}
for v in ${2:-v0 v1}; do
  for rep in 1 2; do
    TQ_ENGINE_LIB=$D/libtq_engine_$v.so python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e_${CFG}_$v.log 2>&1
    python - gpurun_out/e_${CFG}_$v.log $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print(sys.argv[2], round(d["value"], 1), "rl/lr/adj ms", round(r.get("rl_ms", 0), 4), round(r.get("lr_ms", 0), 4), round(r.get("adj_ms", 0), 4), "frac", round(r["frac"], 3))
PY
  done
  TQ_TIMING_LIB=$D/libtq_engine_timing_$v.so python tools/stage_profile.py ${3:-$CFG} > gpurun_out/st_$v.txt 2>&1; grep "RL\|resolve\|N gemm\|P gemm" gpurun_out/st_$v.txt
done
