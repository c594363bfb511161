#!/bin/bash
# GPU parity suite + bench lines + stage profiles (one gpurun call).
# usage: bash tools/quick_check.sh "cfg2 cfg4" "cfg2 cfg4"
CONFIGS=${1:-cfg2 cfg4}
STAGES=${2:-cfg2}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in $CONFIGS; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.log 2>&1
  python - $c <<'PY'
import json, sys
l = open(f"gpurun_out/b_{sys.argv[1]}.log").read().strip().splitlines()[-1]
d = json.loads(l); r = d["roofline"]
print(sys.argv[1], round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "rl/lr/adj ms", round(r.get("rl_ms", 0), 4), round(r.get("lr_ms", 0), 4), round(r.get("adj_ms", 0), 4), "frac", round(r["frac"], 3))
PY
done
for c in $STAGES; do python tools/stage_profile.py $c > gpurun_out/stages_$c.txt 2>&1; grep -v " 0 cyc" gpurun_out/stages_$c.txt; done
