"""Edge cases on the GPU (reference test strategy): empty and identity
operators, single-qubit registers, long Pauli strings, complex coefficients, maximum bond
dimensions per dtype, batch-size invariance and more segments than terms."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import oracle as O  # noqa: E402
from paper_2112_10239_b200 import autodiff as AD  # noqa: E402
from paper_2112_10239_b200.circuits import Circuit, standard_gate  # noqa: E402
from paper_2112_10239_b200.errors import BondTooLarge  # noqa: E402
from paper_2112_10239_b200.hamiltonians import PauliHamiltonian, term, tfim  # noqa: E402
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets  # noqa: E402


def _ocirc(c):
    return O.OCircuit(c.n_qubits, [(g.name, tuple(g.wires), g.param) for g in c.gates], list(c.trainable))


def _oterms(h):
    return [(t.coeff, tuple(t.ops)) for t in h.terms]


def test_empty_and_identity_operators():
    c = layered_circuit(6, 4)
    th = theta_sets(c.n_params, 3, seed=1)
    v, g = AD.grad_expval(c, PauliHamiltonian(6, ()), th, dtype="complex128")
    assert np.all(v == 0) and np.all(g == 0)
    v, g = AD.grad_expval(c, PauliHamiltonian(6, (term(2.5, {}),)), th, dtype="complex128")
    np.testing.assert_allclose(v, 2.5, atol=1e-12)
    np.testing.assert_allclose(g, 0.0, atol=1e-12)


def test_single_qubit_register():
    c = Circuit(1, (standard_gate("ry", (0,), 0.0), standard_gate("rz", (0,), 0.0), standard_gate("rx", (0,), 0.0)),
                (0, 1, 2))
    h = PauliHamiltonian(1, (term(0.3, {0: "X"}), term(-0.7, {0: "Y"}), term(1.1, {0: "Z"})))
    th = np.array([0.4, -1.2, 2.0])
    v, g = AD.grad_expval(c, h, th, dtype="complex128")
    ov, og = O.grad_expval_tt(_ocirc(c), _oterms(h), th)
    assert abs(v - ov) < 1e-12
    np.testing.assert_allclose(g, og, atol=1e-12)


def test_long_pauli_strings_and_complex_coefficients():
    n = 9
    c = layered_circuit(n, 6, "ry", "cnot")
    h = PauliHamiltonian(n, (term(0.5, {0: "X", 2: "Y", 5: "Z", 8: "X"}), term(-0.25, {1: "Y", 7: "Y"}),
                             term(0.75, {3: "Z", 4: "X", 5: "Y", 6: "Z"}), term(0.1, {})))
    th = theta_sets(c.n_params, 2, seed=4)
    v, g = AD.grad_expval(c, h, th, dtype="complex128")
    for b in range(2):
        ov, og = O.grad_expval_tt(_ocirc(c), _oterms(h), th[b])
        assert abs(v[b] - ov) < 1e-11
        np.testing.assert_allclose(g[b], og, atol=1e-11)
    # a Hermitian sum written with complex coefficients: c P + conj(c) P for a Hermitian P
    h2 = PauliHamiltonian(n, (term(0.3 + 0.2j, {0: "Z", 1: "Z"}), term(0.3 - 0.2j, {0: "Z", 1: "Z"})))
    v2 = AD.evaluate_expval(c, h2, th, dtype="complex128")
    v3 = AD.evaluate_expval(c, PauliHamiltonian(n, (term(0.6, {0: "Z", 1: "Z"}),)), th, dtype="complex128")
    np.testing.assert_allclose(v2, v3, atol=1e-12)


def test_bond_limits_per_dtype():
    # chi = 16 in both dtypes, chi = 32 only in complex64
    c16 = layered_circuit(12, 16, "ry", "cz")
    c32 = layered_circuit(14, 20, "ry", "cz")
    h16, h32 = tfim(12), tfim(14)
    th16 = theta_sets(c16.n_params, 1, seed=0)[0]
    th32 = theta_sets(c32.n_params, 1, seed=0)[0]
    ref16 = float(np.real(O.expval_dense(O.simulate_dense(_ocirc(c16), th16), _oterms(h16))))
    v = AD.evaluate_expval(c16, h16, th16, dtype="complex128")
    assert abs(v - ref16) < 1e-10
    v32 = AD.evaluate_expval(c32, h32, th32, dtype="complex64")
    ref32 = float(np.real(O.expval_dense(O.simulate_dense(_ocirc(c32), th32), _oterms(h32))))
    assert abs(v32 - ref32) < 1e-5 * max(1.0, abs(ref32)) + 1e-4
    with pytest.raises(BondTooLarge):
        AD.evaluate_expval(c32, h32, th32, dtype="complex128")
    with pytest.raises(BondTooLarge):
        AD.evaluate_expval(layered_circuit(16, 24, "ry", "cz"), tfim(16),
                           theta_sets(layered_circuit(16, 24).n_params, 1, seed=0)[0])


def test_batch_size_and_segment_invariance():
    c = layered_circuit(40, 8, "ry", "cz")
    h = tfim(40)
    th = theta_sets(c.n_params, 7, seed=9)
    vb, gb = AD.grad_expval(c, h, th, dtype="complex128")
    for b in (0, 6):
        v1, g1 = AD.grad_expval(c, h, th[b], dtype="complex128")
        assert abs(v1 - vb[b]) < 1e-12
        np.testing.assert_allclose(g1, gb[b], atol=1e-12)
    vs, gs = AD.grad_expval(c, h, th, dtype="complex128", segments=60)   # more segments than owned sites
    np.testing.assert_allclose(vs, vb, atol=1e-11)
    np.testing.assert_allclose(gs, gb, atol=1e-11)


def test_values_mode_at_large_bonds():
    """Per-term values (tq_term_values) on the unfused chi = 16 / 32 kernels against the dense
    oracle, including multi-site and Y strings."""
    for n, layers, dtype, tol in ((12, 16, "complex128", 1e-11), (14, 20, "complex64", 2e-5)):
        c = layered_circuit(n, layers, "ry", "cz")
        th = theta_sets(c.n_params, 2, seed=n)
        groups = [{0: "Z"}, {3: "X", 4: "Y"}, {1: "Y", 6: "Z", n - 1: "X"}, {n // 2: "X", n // 2 + 1: "X"}, {}]
        vals = AD.expectation_values(c, th, groups, dtype=dtype)
        for b in range(2):
            psi = O.simulate_dense(_ocirc(c), th[b])
            ref = O.dense_term_values(psi, [(1.0, tuple(sorted(g.items()))) for g in groups])
            np.testing.assert_allclose(vals[b], ref, atol=tol)
