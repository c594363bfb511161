"""Pin the CPU oracle (numpy restatement of tnsim) against the reference's golden
vectors and the closed forms of the reference's own tests."""

import numpy as np
import pytest

import oracle as O
from conftest import ocircuit, oterms


def test_oracle_matches_reference_golden_values(golden_small):
    for case in golden_small["cases"]:
        c = ocircuit(case["circuit"])
        h = oterms(case["ham"])
        th = np.array(case["theta"])
        if c.n > 12 and case["name"].startswith("cfg2") and case["name"] != "cfg2_b0":
            continue  # keep the CPU suite short; b0 covers cfg2
        v, g = O.grad_expval_tt(c, h, th, eps=0.0)
        assert abs(v - case["value"]) < 1e-10, case["name"]
        np.testing.assert_allclose(g, case["grad"], atol=1e-9, rtol=0, err_msg=case["name"])


def test_oracle_untaped_tt_and_dense_agree(golden_small):
    for case in golden_small["cases"]:
        c = ocircuit(case["circuit"])
        if c.n > 10:
            continue
        h = oterms(case["ham"])
        th = np.array(case["theta"])
        e_tt = O.evaluate_expval(c, h, th, eps=0.0)
        e_d = O.expval_dense(O.simulate_dense(c, th), h)
        assert abs(e_tt.real - case["value"]) < 1e-10
        assert abs(e_d.real - case["value"]) < 1e-10


def test_oracle_closed_forms():
    # rx/Z: value cos t, grad -sin t (reference test_autodiff.py:72-82)
    for t in (-1.3, 0.4, 2.9):
        c = O.OCircuit(1, [("rx", (0,), t)], [0])
        v, g = O.grad_expval_tt(c, [(1 + 0j, ((0, "Z"),))], [t])
        assert abs(v - np.cos(t)) < 1e-12 and abs(g[0] + np.sin(t)) < 1e-12
    # <0..0|TFIM|0..0> = -(n-1) (reference test_hamiltonians.py:59-61)
    for n in (2, 5, 9):
        c = O.OCircuit(n, [], [])
        v, _ = O.grad_expval_tt(c, O.tfim_terms(n), [])
        assert abs(v + (n - 1)) < 1e-12
    # crz: <X0> = cos(0.45), grad = -sin(0.45)/2 (reference test_autodiff.py:126-149)
    c = O.OCircuit(2, [("h", (0,), None), ("h", (1,), None), ("crz", (0, 1), 0.9)], [2])
    v, g = O.grad_expval_tt(c, [(1 + 0j, ((0, "X"),))], [0.9])
    assert abs(v - np.cos(0.45)) < 1e-12 and abs(g[0] + 0.5 * np.sin(0.45)) < 1e-12
    shift = O.parameter_shift_grad(c, [(1 + 0j, ((0, "X"),))], [0.9], engine="dense")
    assert abs(shift[0] - g[0]) < 1e-12


def test_oracle_mbe_matches_reference(golden_small):
    d = golden_small["mbe10"]
    c = O.brickwork(5, d["depth"])
    fun = O.mbe_objective(c, 10, [tuple(e) for e in d["edges"]], alpha=d["alpha"])
    loss, grad = fun(np.array(d["theta"]))
    assert abs(loss - d["loss"]) < 1e-10
    np.testing.assert_allclose(grad, d["grad"], atol=1e-9)
    ev = O.vertex_expectations(c, np.array(d["theta"]), 10)
    np.testing.assert_allclose(ev, d["vertex"], atol=1e-12)
    asg = O.round_cut(ev)
    assert list(asg) == d["assignment"]
    assert O.cut_value([tuple(e) for e in d["edges"]], asg) == d["cut"]


def test_oracle_inner(golden_small):
    d = golden_small["inner8"]
    c = ocircuit(d["circuit"])
    a = O.simulate_tt(c, d["theta_a"], eps=0.0)
    b = O.simulate_tt(c, d["theta_b"], eps=0.0)
    ip = O.tt_inner(a, b)
    assert abs(ip - complex(d["re"], d["im"])) < 1e-12


def test_reading_a_generator_counts():
    # SURVEY.md section 8 config shorthand: gate and parameter counts
    c = O.ry_cz_layers(10, 4, "ry", "cnot")
    assert c.n_params == 20 and len(c.gates) == 29
    c = O.ry_cz_layers(100, 10)
    assert c.n_params == 500 and len(c.gates) == 748
    c = O.brickwork(1024, 4)
    assert c.n_params == 8192 and len(c.gates) == 9727


def test_oracle_adam_matches_reference_minimize():
    """The oracle's Adam restatement (used by the f1 GPU checks) against the REAL reference's
    minimize on mbe_objective (tests/golden/golden_f1.json): every iteration's loss to 1e-10."""
    import json
    import os

    import oracle as O

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_f1.json")
    case = [c for c in json.load(open(path))["cases"] if c["optimizer"] == "adam"][0]
    n = (case["V"] + 1) // 2
    fun = O.mbe_objective(O.brickwork(n, case["depth"]), case["V"], [tuple(e) for e in case["edges"]],
                          alpha=case["alpha"])
    run = case["runs"][0]
    theta, values = O.adam_minimize(fun, np.array(run["theta0"]), rate=case["rate"], max_iters=case["max_iters"])
    np.testing.assert_allclose(values, run["loss"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(theta, run["theta_final"], atol=1e-9)
