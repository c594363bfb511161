"""Time the truncated engine on the reference's `bench tfim` workload (tfim_workload)."""
import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import numpy as np
import torch
from paper_2112_10239_b200 import truncated as TR, chain as C
from paper_2112_10239_b200.report import tfim_workload
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import theta_sets
for (n, g, chi, B) in [(500, 5000, 16, 1), (500, 5000, 16, 148), (100, 3000, 32, 1), (100, 3000, 32, 148)]:
    c = tfim_workload(n, g)
    terms = C.normalize_terms(tfim(n))
    th = theta_sets(c.n_params, B, seed=0)
    for dt in ("complex128", "complex64"):
        TR.simulate_terms(c, terms, th[:1], 0.0, chi, dtype=dt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = TR.simulate_terms(c, terms, th, 0.0, chi, dtype=dt)
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t0
        print(f"n={n} gates={g} chi={chi} B={B} {dt}: {dt_s*1e3:.1f} ms  ({B/dt_s:.2f} sims/s) maxbond={r.bonds.max()} disc={r.discarded[0]:.3e}", flush=True)
