D=paper_2112_10239_b200
for v in "" _gt2; do
  echo "== variant [$v]"
  TQ_ENGINE_LIB=$D/libtq_engine$v.so python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e_cfg4$v.log 2>&1
  python - gpurun_out/e_cfg4$v.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]
print(round(d["value"], 1), "rl/lr/adj ms", round(r["rl_ms"], 4), round(r["lr_ms"], 4), round(r["adj_ms"], 4), "frac", round(r["frac"], 3))
PY
  TQ_TIMING_LIB=$D/libtq_engine_timing$v.so python tools/stage_profile.py cfg4 > gpurun_out/st_cfg4$v.txt 2>&1; grep -v " 0 cyc" gpurun_out/st_cfg4$v.txt
done
TQ_ENGINE_LIB=$D/libtq_engine_gt2.so python -m pytest tests -m gpu -x -q 2>&1 | tail -2
