import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import torch
from paper_2112_10239_b200 import truncated as TR, chain as C
from paper_2112_10239_b200.report import tfim_workload
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import theta_sets
for (n, g, chi) in [(500, 5000, 16), (100, 3000, 32)]:
    c = tfim_workload(n, g); terms = C.normalize_terms(tfim(n)); th = theta_sets(c.n_params, 1, seed=0)
    tr = TR.simulate_train(c, th, 0.0, chi); tr.term_values(terms); torch.cuda.synchronize()
    t0 = time.perf_counter(); tr = TR.simulate_train(c, th, 0.0, chi); torch.cuda.synchronize(); t1 = time.perf_counter()
    v, _ = tr.term_values(terms); torch.cuda.synchronize(); t2 = time.perf_counter()
    trc = TR.compress(tr, 1e-6, chi); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"n={n} gates={g} chi={chi}: run {1e3*(t1-t0):.1f} ms, values {1e3*(t2-t1):.1f} ms, compress {1e3*(t3-t2):.1f} ms")
