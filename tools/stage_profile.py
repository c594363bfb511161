"""Per-stage cycle breakdown of the sweep kernels (diagnostic build -DTQ_STAGE_TIMING).

usage (GPU box): python tools/stage_profile.py [cfg2|cfg4|cfg5|cfg1] [batch]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_10239_b200 import _lib  # noqa: E402

lib = _lib.load(os.environ.get("TQ_TIMING_LIB") or os.path.join(ROOT, "paper_2112_10239_b200", "libtq_engine_timing.so"))
lib.tq_stage_cycles.restype = ctypes.c_int32
lib.tq_stage_cycles.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
from paper_2112_10239_b200 import engine as E  # noqa: E402
from paper_2112_10239_b200.program import ExpvalProgram  # noqa: E402
from paper_2112_10239_b200.workloads import CONFIGS, theta_sets  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.batch
c, h = cfg.circuit(), cfg.hamiltonian()
prog = ExpvalProgram(c, h, B, grad=cfg.grad)
th = torch.tensor(theta_sets(c.n_params, B), dtype=torch.float32, device="cuda")
for _ in range(3):
    prog.run_device(th)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
lib.tq_stage_cycles(buf)
reps = 5
for _ in range(reps):
    prog.run_device(th)
torch.cuda.synchronize()
lib.tq_stage_cycles(buf)
plan = prog.plan
items = B * plan.n_segments
sites = B * int(plan.info["sub_chain_sites"])
print(f"{name} B={B} segments={plan.n_segments} sub-chain sites={plan.info['sub_chain_sites']} chi={plan.chi_max}")
rl = ["stage", "fold", "N gemm", "bracket", "resolve+sync", "P gemm"]
lr = ["stage+PIN+A", "-", "M gemm", "bracket", "Lam+G gemm", "G store", "-", "values MR", "values dots", "values fin"]
for k, names in ((0, rl), (1, lr)):
    tot = sum(buf[16 * k + i] for i in range(16))
    if not tot:
        continue
    print(("RL" if k == 0 else "LR") + f"  total {tot / reps / sites:.0f} cycles per site-item")
    for i, nm in enumerate(names):
        v = buf[16 * k + i] / reps / sites
        print(f"   {nm:12s} {v:8.0f} cyc/site  {100 * buf[16 * k + i] / tot:5.1f}%")
