"""Small engine calls for compute-sanitizer (one tool per gpurun call)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2112_10239_b200 import autodiff as AD
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets
for n, layers, ent in ((10, 4, "cnot"), (24, 10, "cz"), (20, 12, "cz"), (12, 20, "cz")):
    c = layered_circuit(n, layers, "ry", ent)
    th = theta_sets(c.n_params, 3, seed=1)
    v, g = AD.grad_expval(c, tfim(n), th, segments=2)
    vals = AD.expectation_values(c, th, [{0: "Z"}, {3: "X", 4: "Z"}])
    print(n, layers, float(v[0]), float(np.abs(g).max()))
print("sanitize case done")
