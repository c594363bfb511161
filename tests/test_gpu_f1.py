"""Row f1 parity: the on-device MBE MaxCut optimisation loop against the REAL reference's
``minimize`` (autodiff.py:614-659) on ``mbe_objective`` (maxcut.py:219-252) and its
``solve_maxcut`` (maxcut.py:273-319), same seeds (tests/golden/golden_f1.json, made by
make_golden_f1.py with tnsim).

* ``AdamGraph`` (one captured CUDA graph per iteration, restarts as the batch), complex128,
  replayed one iteration at a time: every iteration's loss within 1e-9 (relative) of the
  reference's for every restart, and the final angles within 1e-7.
* ``solve_maxcut`` (default dtype complex128): identical assignment, cut, restart index and
  iteration count; relaxed loss within 1e-9."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2112_10239_b200 import maxcut as MC  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_f1.json")


def _cases():
    with open(GOLD) as fh:
        return json.load(fh)["cases"]


def _graph(c):
    return MC.Graph(c["V"], tuple((int(u), int(v), float(w)) for u, v, w in c["edges"]))


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_adam_graph_trajectory_matches_reference(case):
    g = _graph(case)
    n, _ = MC.mbe_encode(g)
    circ = MC.brickwork_ansatz(n, case["depth"])
    R = case["restarts"]
    obj = MC.MBEObjective(circ, g, case["alpha"], dtype="complex128", batch=R)
    th0 = np.array([r["theta0"] for r in case["runs"]])
    ag = MC.AdamGraph(obj, th0, case["rate"], case["max_iters"], optimizer=case["optimizer"]).capture()
    traj = []
    for _ in range(case["max_iters"] + 1):
        ag.graph.replay()
        traj.append(ag.value.cpu().numpy().copy())
    assert int(ag.bad.item()) < 0
    traj = np.array(traj)                       # [iters + 1, R]
    for r, run in enumerate(case["runs"]):
        ref = np.array(run["loss"])
        got = traj[:len(ref), r]
        np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-11, err_msg=f"restart {r}")
        np.testing.assert_allclose(ag.theta[r].cpu().numpy(), run["theta_final"], atol=1e-7)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_solve_maxcut_matches_reference(case):
    g = _graph(case)
    res = MC.solve_maxcut(g, depth=case["depth"], optimizer=case["optimizer"], rate=case["rate"],
                          restarts=case["restarts"], max_iters=case["max_iters"], seed=case["seed"],
                          alpha=case["alpha"])
    ref = case["solve"]
    assert list(res.assignment) == ref["assignment"]
    assert res.cut_value == ref["cut"]
    assert res.restart_index == ref["restart_index"]
    assert res.iterations == ref["iters"]
    assert abs(res.relaxed_loss - ref["loss"]) <= 1e-9 * max(1.0, abs(ref["loss"]))
