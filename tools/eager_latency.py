"""Host-side latency of the eager API (grad_expval on cfg1 / cfg2 shapes), averaged."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10239_b200 import autodiff as AD
from paper_2112_10239_b200.workloads import CONFIGS, theta_sets
for name, B in (("cfg1", 1), ("cfg2", 1), ("cfg2", 256)):
    cfg = CONFIGS[name]; c, h = cfg.circuit(), cfg.hamiltonian()
    th = theta_sets(c.n_params, B, seed=0)
    for _ in range(3):
        AD.grad_expval(c, h, th)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); n = 20
    for _ in range(n):
        AD.grad_expval(c, h, th)
    torch.cuda.synchronize()
    print(f"{name} B={B}: {1e3 * (time.perf_counter() - t0) / n:.3f} ms per grad_expval call")
