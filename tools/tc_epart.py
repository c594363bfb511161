import ctypes, os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import ctypes, sys, torch, numpy as np
sys.path.insert(0, "%s")
from paper_2112_10239_b200 import _lib, engine as E, chain as C
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets
c = layered_circuit(14, 20, "ry", "cz"); h = tfim(14)
terms = C.normalize_terms(h)
th = torch.tensor(theta_sets(c.n_params, 1, seed=14), dtype=torch.float32, device="cuda")
dp = E.device_plan(c, terms, "energy", 1, th.device, 14, dtype="complex64")
coef = torch.tensor([[t[0].real for t in terms]], dtype=torch.float32, device="cuda")
e, _ = E.energy_grad_raw(dp, th, coef, False, "complex64")
ws, nb = dp.workspace(1, 0, _lib.TQ_C64, torch.cuda.current_stream().cuda_stream)
base = (ws.data_ptr() + 255) // 256 * 256 - ws.data_ptr()
ep = ws[base: base + 14 * 8].view(torch.complex64).cpu().numpy()
print("E", e[0].tolist()); print("epart", np.round(ep.real, 5).tolist())
s = dp.plan.sites; sg = dp.plan.segs
for g in range(14):
    b0, cnt = int(sg["site_begin"][g]), int(sg["site_count"][g])
    m = [(int(s["chi_l"][k]), int(s["chi_r"][k]), int(s["rl_db"][k])) for k in range(b0, b0 + cnt)]
    n32 = sum(1 for a, bb, d in m if a == 32 and bb == 32)
    print(g, "sites", cnt, "n32", n32, "db32", sorted({d for a, bb, d in m if a == 32 and bb == 32}))
''' % R
for tc in ("0", "1"):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, TQ_TC=tc), capture_output=True, text=True, timeout=200)
    print("TQ_TC", tc); print(out.stdout[-3000:]); print(out.stderr[-1500:])
