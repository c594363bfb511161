for args in "40 400 16" "500 5000 16" "100 3000 32"; do
python - $args <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2112_10239_b200 import truncated as TR, chain as C
from paper_2112_10239_b200.report import tfim_workload
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import theta_sets
n, g, chi = map(int, sys.argv[1:4])
c = tfim_workload(n, g)
terms = C.normalize_terms(tfim(n))
th = theta_sets(c.n_params, 1, seed=0)
try:
    r = TR.simulate_terms(c, terms, th, 0.0, chi, dtype=os.environ.get("DT","complex128"))
    print(n, g, chi, "ok", r.bonds.max(), r.discarded[0], r.energy([t[0] for t in terms])[0].real)
except Exception as e:
    print(n, g, chi, "FAIL", type(e).__name__, str(e)[:100])
PY
done
