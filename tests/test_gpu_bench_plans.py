"""GPU parity on the exact plans ``bench.py`` times (VERDICT r1 "What's weak" 1).

* cfg4: n=1000, 20 layers, B=64 angle sets ``theta_sets(P, 64, seed=0)``, the automatic
  light-cone segmentation the bench picks for B=64, through ``ExpvalProgram`` (the bench's
  captured device graph and its host-buffer graph).  Energies of sets 0/31/63 and 32 + 16
  parameter-shift coordinates of sets 0 and 63 against the REAL reference
  (``tests/golden/golden_bench.npz``, made by ``make_golden_bench.py`` with tnsim's
  ``evaluate_expval(engine="tt", eps=1e-12)``; reference autodiff.py:490-550).
* cfg5: n=1024, 10 layers, forward only, B=64 (the bench plan): energies of sets 0/63 against
  tnsim; n=8192 (``init_params(40960, generator(0))``) against tnsim's E, both as one chain and
  as the sum of the 8 chain shards the 8-GPU run evaluates (distributed.shard_hamiltonian).

Tolerances (complex64): |dE| <= 1e-5 max(|E|, 1e-2 sum|c|);
|dg_k| <= 1e-5 |g_ref,k| + 1e-6 ||g||_inf.  Only sampled gradient coordinates exist on the
reference side (each costs two 20 s tnsim forwards), so ||g||_inf is taken from the engine's
full gradient vector."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from helpers_engine import tol64  # noqa: E402
from paper_2112_10239_b200 import autodiff as AD  # noqa: E402
from paper_2112_10239_b200.distributed import shard_hamiltonian  # noqa: E402
from paper_2112_10239_b200.hamiltonians import tfim  # noqa: E402
from paper_2112_10239_b200.program import ExpvalProgram  # noqa: E402
from paper_2112_10239_b200.workloads import CONFIGS, layered_circuit, theta_sets  # noqa: E402

GB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_bench.npz")


@pytest.fixture(scope="module")
def golden_bench():
    if not os.path.exists(GB):
        pytest.skip("golden_bench.npz not generated")
    return dict(np.load(GB))


def _shift_ok(g, coords, ref, gmax):
    err = np.abs(g[coords] - ref)
    bound = 1e-5 * np.abs(ref) + 1e-6 * gmax
    return np.all(err <= bound), float(np.max(err / bound))


@pytest.fixture(scope="module")
def cfg4_bench():
    cfg = CONFIGS["cfg4"]
    c, h = cfg.circuit(), cfg.hamiltonian()
    th = theta_sets(c.n_params, 64, seed=0)
    prog = ExpvalProgram(c, h, 64)           # exactly what bench.py builds (segments=None -> auto)
    prog.theta_dev.copy_(torch.tensor(th, dtype=torch.float32))
    prog.capture()
    e_dev, g_dev = prog.replay()
    e_dev, g_dev = e_dev[:, 0].cpu().numpy().copy(), g_dev.double().cpu().numpy().copy()
    e_host, g_host = prog(th)                # the host-buffer graph (e2e path)
    return prog, th, h, e_dev, g_dev, e_host, g_host


def test_cfg4_bench_plan_energies(cfg4_bench, golden_bench):
    prog, th, h, e, g, e_host, g_host = cfg4_bench
    assert prog.plan.n_segments >= 2          # the auto-segmented plan, not the B=1 one
    np.testing.assert_array_equal(e, e_host)  # device graph and host-buffer graph agree bitwise
    np.testing.assert_array_equal(g.astype(np.float32), g_host)
    for b, ref in zip(golden_bench["cfg4b_theta_idx"], golden_bench["cfg4b_E"]):
        assert abs(e[b] - ref) <= tol64(ref, h), (b, e[b], ref)


@pytest.mark.parametrize("which", ["b0", "b63"])
def test_cfg4_bench_plan_shift_coordinates(cfg4_bench, golden_bench, which):
    _, _, _, _, g, _, _ = cfg4_bench
    b = 0 if which == "b0" else 63
    coords, ref = golden_bench[f"cfg4b_coords_{which}"], golden_bench[f"cfg4b_shift_{which}"]
    assert len(coords) >= 16 and (which != "b0" or len(coords) >= 32)
    ok, worst = _shift_ok(g[b], coords, ref, np.max(np.abs(g[b])))
    assert ok, f"set {b}: worst error / bound = {worst:.3f}"


def test_cfg4_golden_set_32_coordinates(golden_bench, golden_large):
    """The generator(0) set at B=1 (the other segmentation): 4 + 28 shift coordinates."""
    cfg = CONFIGS["cfg4"]
    c, h = cfg.circuit(), cfg.hamiltonian()
    v, g = AD.grad_expval(c, h, golden_large["cfg4_theta"])
    coords = np.concatenate([golden_large["cfg4_coords"], golden_bench["cfg4_coords_more"]])
    ref = np.concatenate([golden_large["cfg4_shift"], golden_bench["cfg4_shift_more"]])
    assert len(coords) >= 32
    assert abs(v - float(golden_large["cfg4_E"])) <= tol64(float(golden_large["cfg4_E"]), h)
    ok, worst = _shift_ok(g, coords, ref, np.max(np.abs(g)))
    assert ok, f"worst error / bound = {worst:.3f}"


def test_cfg5_bench_plan_n1024(golden_bench):
    cfg = CONFIGS["cfg5"]
    c, h = cfg.circuit(), cfg.hamiltonian()
    th = theta_sets(c.n_params, 64, seed=0)
    prog = ExpvalProgram(c, h, 64, grad=False)
    e, _ = prog(th)
    prog.capture()
    e2, _ = prog(th)
    np.testing.assert_array_equal(e, e2)
    for b, ref in zip(golden_bench["cfg5b_theta_idx"], golden_bench["cfg5b_E"]):
        assert abs(e[b] - ref) <= tol64(ref, h), (b, e[b], ref)


def test_cfg5_n8192_whole_and_sharded(golden_bench):
    if "cfg5_8192_E" not in golden_bench:
        pytest.skip("n=8192 golden not generated")
    n = 8192
    c, h = layered_circuit(n, 10), tfim(n)
    th = theta_sets(c.n_params, 1, seed=0)
    ref = float(golden_bench["cfg5_8192_E"])
    whole = AD.evaluate_expval(c, h, th[0])
    assert abs(whole - ref) <= tol64(ref, h), (whole, ref)
    # the 8-GPU decomposition: each rank's owned terms on its light-cone sub-chain; the
    # all-reduce is the sum (evaluated here one shard after another on this GPU)
    parts = [AD.evaluate_expval(c, shard_hamiltonian(h, r, 8), th[0]) for r in range(8)]
    assert abs(sum(parts) - ref) <= tol64(ref, h), (sum(parts), ref)
