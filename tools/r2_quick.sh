#!/bin/bash
# Quick GPU iteration: parity on the benched plans + core goldens, cfg4/cfg2 bench lines, cfg4 stages.
set -u
mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py tests/test_gpu_edges.py -q --timeout 600 > gpurun_out/q/pytest.txt 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/q/pytest.txt | tail -8
for c in cfg4 cfg2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/q/bench_$c.log 2>&1; echo "bench $c rc=$?"
  python - "$c" <<'PY'
import json,sys
l=json.loads(open(f"gpurun_out/q/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
r=l["roofline"]; print(sys.argv[1], "value %.1f e2e %.1f ms %.4f rl %.4f lr %.4f adj %.4f frac %.3f step_frac %.3f clocks %s" % (l["value"], l["e2e"]["value"], l["ms_per_step"], r["rl_ms"], r["lr_ms"], r["adj_ms"], r["frac"], r["step"]["frac"], l["clocks"]))
PY
done
timeout 300 python tools/stage_profile.py cfg4 > gpurun_out/q/stages_cfg4.txt 2>&1; cat gpurun_out/q/stages_cfg4.txt | head -20
