import os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, "%s")
from paper_2112_10239_b200 import autodiff as AD, chain as C
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets
for n, L, segs in ((14, 20, None), (14, 20, 1), (20, 20, 1), (40, 20, 1), (40, 20, None)):
    c = layered_circuit(n, L, "ry", "cz")
    th = theta_sets(c.n_params, 2, seed=n)
    v = AD.evaluate_expval(c, tfim(n), th, dtype="complex64", segments=segs)
    p = C.compile_chain(c, C.normalize_terms(tfim(n)), "energy", segments=segs)
    s = p.sites
    n32 = int(((s["chi_l"] == 32) & (s["chi_r"] == 32)).sum())
    print(n, L, segs, p.n_segments, "sites32", n32, "E", v.tolist())
''' % R
for tc in ("0", "1"):
    env = dict(os.environ, TQ_TC=tc)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print("TQ_TC", tc); print(out.stdout[-3000:], out.stderr[-2000:])
