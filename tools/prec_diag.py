"""Precision diagnostic: cfg4 bench-batch set 0 energy vs the tnsim golden for several segmentations."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2112_10239_b200 import autodiff as AD, engine as E, chain as C
from paper_2112_10239_b200.workloads import CONFIGS, theta_sets
cfg = CONFIGS["cfg4"]; c, h = cfg.circuit(), cfg.hamiltonian()
th = theta_sets(c.n_params, 64, seed=0)
g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden_bench.npz")))
ref = g["cfg4b_E"]
print("auto segments B=64:", C.choose_segments(c.n_qubits, C.normalize_terms(h), C.time_gates(c), 64))
for S in (1, 2, 3, 4, 8, 16, 37, 148):
    v = AD.evaluate_expval(c, h, th[[0, 31, 63]], segments=S)
    print(S, v, v - ref)
