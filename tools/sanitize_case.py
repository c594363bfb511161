"""Small engine calls for compute-sanitizer (one tool per gpurun call): every sweep path.

chi <= 8 fused warp teams (rl/lr direct path, build_wct, warp adjoint), chi = 16 and 32 CTA
teams (matrix bracket, cp.async A/P prefetch, compact digit-tree adjoint), the values sweeps,
the inner-product sweep, and the truncated engine (simulate, taped record, frozen replay)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2112_10239_b200 import autodiff as AD  # noqa: E402
from paper_2112_10239_b200 import chain as C  # noqa: E402
from paper_2112_10239_b200 import truncated as TR  # noqa: E402
from paper_2112_10239_b200.hamiltonians import tfim  # noqa: E402
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets  # noqa: E402

for n, layers, ent, segs in ((10, 4, "cnot", None), (24, 10, "cz", 2), (20, 12, "cz", 2), (14, 20, "cz", 2),
                             (40, 20, "cz", None)):
    c = layered_circuit(n, layers, "ry", ent)
    th = theta_sets(c.n_params, 3, seed=1)
    v, g = AD.grad_expval(c, tfim(n), th, segments=segs)
    vals = AD.expectation_values(c, th, [{0: "Z"}, {3: "X", 4: "Z"}], segments=segs)
    mbe_like = AD.evaluate_expval(c, tfim(n), th[0])
    print(n, layers, "chi", C.factored_chi(n, C.time_gates(c)), float(v[0]), float(np.abs(g).max()))
c = layered_circuit(8, 4)
print("inner", AD.state_inner_product(c, theta_sets(c.n_params, 1, seed=2)[0], c, theta_sets(c.n_params, 1, seed=3)[0]))
c = layered_circuit(10, 8)
terms = C.normalize_terms(tfim(10))
th = theta_sets(c.n_params, 2, seed=4)
res = TR.simulate_terms(c, terms, th, 0.0, 4)
vals, grad = TR.straight_through(c, terms, th, 0.0, 2)
print("truncated", res.discarded, float(np.abs(grad).max()))
print("sanitize case done")
