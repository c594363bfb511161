import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_10239_b200 import autodiff as AD
from paper_2112_10239_b200.workloads import CONFIGS, theta_sets
cfg = CONFIGS["cfg1"]; c, h = cfg.circuit(), cfg.hamiltonian()
th = theta_sets(c.n_params, 1, seed=0)[0]
for _ in range(5):
    AD.grad_expval(c, h, th)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    AD.grad_expval(c, h, th)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
