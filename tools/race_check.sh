#!/bin/bash
# Production library vs the race-stress build: every output bitwise identical and finite.
set -e
mkdir -p gpurun_out/race
python tools/race_stress.py gpurun_out/race/prod.npz 2
TQ_ENGINE_LIB=paper_2112_10239_b200/libtq_engine_debug.so python tools/race_stress.py gpurun_out/race/debug.npz 3
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/race/prod.npz"), np.load("gpurun_out/race/debug.npz")
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("outputs compared:", len(a.files), "differing:", bad if bad else "none")
raise SystemExit(1 if bad else 0)
PY
