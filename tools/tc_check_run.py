import os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys
sys.path.insert(0, "%s")
from paper_2112_10239_b200 import _lib
_lib.load(os.path.join("%s", "paper_2112_10239_b200", "libtq_engine_check.so"))
from paper_2112_10239_b200 import autodiff as AD
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets
c = layered_circuit(14, 20, "ry", "cz")
th = theta_sets(c.n_params, 1, seed=14)
for segs in (14,):
    print("segs", segs, AD.evaluate_expval(c, tfim(14), th, dtype="complex64", segments=segs), flush=True)
''' % (R, R)
for tc in ("0", "1", "2", "3"):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, TQ_TC=tc), capture_output=True, text=True, timeout=200)
    print("TQ_TC", tc); print(out.stdout[-2500:]); print(out.stderr[-1500:])
