"""Row f3 on CPU: the numpy mirror of the truncated kernel (tests/mirror_trunc.py) and the
host compiler (truncated.compile_gates) against the reference's own truncated simulation
(golden_trunc.json) and the oracle."""

import json
import os

import numpy as np
import pytest

import mirror_trunc as M
import oracle as O
from helpers_engine import to_circuit, to_ham
from paper_2112_10239_b200 import chain as C
from paper_2112_10239_b200 import truncated as TR
from paper_2112_10239_b200.errors import InputError

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden_trunc():
    with open(os.path.join(HERE, "golden", "golden_trunc.json")) as f:
        return json.load(f)


def test_mirror_matches_reference_golden(golden_trunc):
    ran = 0
    for case in golden_trunc["cases"]:
        c = to_circuit(case["circuit"])
        if c.n_qubits > 10:
            continue   # the pure-Python Jacobi is slow; the GPU test covers the rest
        h = to_ham(case["ham"], c.n_qubits)
        terms = C.normalize_terms(h)
        _, rows = TR.compile_gates(c)
        cores, disc = M.simulate(c.n_qubits, TR.resolved_gates(rows, np.array(case["theta"])), case["eps"],
                                 case["chi_max"])
        vals = M.term_values(cores, terms)
        e = sum(cf * v for (cf, _), v in zip(terms, vals))
        assert abs(e.real - case["value"]) < 1e-10, case["name"]
        assert abs(disc - case["discarded"]) < 1e-12, case["name"]
        assert [1] + [cc.shape[2] for cc in cores] == case["bonds"], case["name"]
        ran += 1
    assert ran >= 4


def test_swap_chain_expansion_matches_reference_order():
    from paper_2112_10239_b200.circuits import Circuit, standard_gate

    c = Circuit(6, (standard_gate("cnot", (4, 1)), standard_gate("crz", (0, 2), 0.4)), (1,))
    table, rows = TR.compile_gates(c)
    sites = [(int(r["kind"]), int(r["site"])) for r in table]
    # cnot(4,1): swaps (3,4),(2,3) bring 4 next to 1, gate on (1,2), swaps back (2,3),(3,4)
    assert sites[:5] == [(2, 3), (2, 2), (2, 1), (2, 2), (2, 3)]
    assert table[2]["flip"] == 0 and np.any(table[2]["m"])        # constant, pre-flipped matrix
    assert table[6]["rot"] == 4 and table[6]["slot"] == 0          # trainable crz stays symbolic
    th = np.array([0.4])
    res = TR.resolved_gates(rows, th)
    psi = np.zeros(64, complex)
    psi[0] = 1
    oc = O.OCircuit(6, [(g.name, tuple(g.wires), g.param) for g in c.gates], [1])
    ref = O.simulate_dense(oc, th).reshape(-1)
    cores, _ = M.simulate(6, res, 0.0, None)
    dense = cores[0].reshape(2, -1)
    for k in range(1, 6):
        dense = np.tensordot(dense, cores[k], axes=([-1], [0]))
    np.testing.assert_allclose(dense.reshape(-1), ref, atol=1e-12)


def test_truncation_argument_checks():
    with pytest.raises(InputError):
        TR.check_truncation_args(-1.0, None)
    with pytest.raises(InputError):
        TR.check_truncation_args(0.0, 0)
    assert TR.check_truncation_args(0.0, 8) == 8
    assert TR.check_truncation_args(1e-3, None) == TR.MAX_CHI_TRUNC
