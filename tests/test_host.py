"""CPU-only tests: chain compiler + numpy kernel mirror against the oracle, the
C-ABI library's exports and struct layouts (no compute calls without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

import mirror
import oracle as O
from helpers_engine import to_circuit, to_ham
from paper_2112_10239_b200 import chain as C
from paper_2112_10239_b200.circuits import Circuit, standard_gate
from paper_2112_10239_b200.errors import BondTooLarge
from paper_2112_10239_b200.hamiltonians import tfim
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mirror_matches_reference_golden(golden_small):
    ran = 0
    for case in golden_small["cases"]:
        c = to_circuit(case["circuit"])
        if c.n_qubits > 12:
            continue
        h = to_ham(case["ham"], c.n_qubits)
        terms = C.normalize_terms(h)
        for segs in (1, 3):
            try:
                plan = C.compile_chain(c, terms, "energy", segments=segs)
            except BondTooLarge:
                continue
            coef = np.array([t[0].real for t in terms])
            e, g = mirror.energy_grad(plan, np.array(case["theta"]), coef)
            assert abs(e.real - case["value"]) < 1e-12, case["name"]
            np.testing.assert_allclose(g, case["grad"], atol=1e-12)
            ran += 1
    assert ran >= 20


def test_mirror_values_and_segments_cfg2(golden_small):
    case = golden_small["cases"][1]
    c = to_circuit(case["circuit"])
    h = to_ham(case["ham"], c.n_qubits)
    terms = C.normalize_terms(h)
    plan = C.compile_chain(c, terms, "values", segments=4)
    vals = mirror.term_values(plan, np.array(case["theta"]))
    e = sum(t[0] * v for t, v in zip(terms, vals))
    assert abs(e.real - case["value"]) < 1e-12


def test_factored_bond_dimensions_match_survey():
    # SURVEY.md section 8 shorthand: chi per config under reading A
    for n, layers, ent, chi in ((10, 4, "cnot", 2), (100, 10, "cz", 8), (1000, 20, "cz", 32), (64, 10, "cz", 8)):
        c = layered_circuit(n, layers, "ry", ent)
        plan = C.compile_chain(c, C.normalize_terms(tfim(n)), "energy", segments=1)
        assert plan.chi_max == chi, (n, layers, plan.chi_max)


def test_light_cone_segments_cover_terms():
    c = layered_circuit(100, 10)
    terms = C.normalize_terms(tfim(100))
    plan = C.compile_chain(c, terms, "energy", segments=8)
    assert plan.n_segments == 8
    lo, hi = plan.segs["lo"], plan.segs["hi"]
    assert lo[0] == 0 and hi[-1] == 99
    # every trainable slot is covered by at least one segment
    assert np.all(np.diff(plan.gred_ptr) >= 1)


def test_operator_schmidt_split():
    for name in ("cz", "cnot", "swap"):
        g = standard_gate(name, (0, 1))
        bits, f0, f1 = C.split_two_qubit(g.matrix)
        rebuilt = sum(np.kron(a, b) for a, b in zip(f0, f1))
        np.testing.assert_allclose(rebuilt, g.matrix, atol=1e-14)
        assert bits == (2 if name == "swap" else 1)


def test_bond_limit_raises():
    wide = Circuit(8, tuple(standard_gate("cnot", (0, 7)) for _ in range(6)), ())
    with pytest.raises(BondTooLarge):
        C.compile_chain(wide, C.normalize_terms(tfim(8)), "energy")


def _lib_path():
    return os.path.join(ROOT, "paper_2112_10239_b200", "libtq_engine.so")


def test_library_exports_every_header_symbol():
    path = _lib_path()
    if not os.path.exists(path):
        pytest.skip("library not built")
    import torch  # noqa: F401  (provides libcudart.so.12 to the loader)
    from paper_2112_10239_b200 import _lib

    declared = set()
    for h in ("tq_engine.h", "tq_trunc.h"):
        header = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"\b(tq_[a-z_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    lib = ctypes.CDLL(path)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert _lib.abi_sizes() == _lib.NUMPY_SIZES
    assert b"sm_100a" in _lib.load().tq_build_info()


def test_theta_sets_are_float32_exact():
    th = theta_sets(500, 4, seed=0)
    np.testing.assert_array_equal(th, th.astype(np.float32).astype(np.float64))
    g = np.array(O.generator(0).uniform(-np.pi, np.pi, 500))
    np.testing.assert_array_equal(theta_sets(500, 1, seed=0)[0], g.astype(np.float32).astype(np.float64))


def test_every_module_imports_without_a_gpu():
    import importlib

    for m in ("autodiff", "chain", "circuits", "engine", "errors", "hamiltonians", "maxcut", "program",
              "roofline", "seeding", "tlq", "workloads", "_lib", "build"):
        importlib.import_module(f"paper_2112_10239_b200.{m}")


def test_reference_objects_compile_directly():
    """A tnsim maintainer passes tnsim.Circuit / PauliHamiltonian straight to the engine
    (INTEGRATION.md); the compiler duck-types them.  Build container only."""
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted")
    import sys

    sys.path.insert(0, ref)
    try:
        import tnsim
    finally:
        sys.path.remove(ref)
    import mirror

    c = tnsim.Circuit(6, tuple(tnsim.standard_gate(*g) for g in (("ry", (0,), 0.3), ("cnot", (0, 1)), ("rx", (2,), 0.1),
                                                                   ("cz", (1, 2)), ("ry", (5,), 0.7), ("crz", (4, 5), 0.2))),
                      trainable=(0, 2, 4, 5))
    h = tnsim.tfim(6)
    terms = C.normalize_terms(h)
    plan = C.compile_chain(c, terms, "energy", segments=2)
    th = np.array([0.3, 0.1, 0.7, 0.2])
    e, g = mirror.energy_grad(plan, th, np.array([t[0].real for t in terms]))
    v, gr = tnsim.grad_expval(c, h, th, engine="tt")
    assert abs(e.real - v) < 1e-12 and np.max(np.abs(g - gr)) < 1e-12
    assert C.structure_key(c) == C.structure_key(c)


def test_survey_work_model_matches_section_8d():
    """bench.py's roofline uses SURVEY.md section 8(d)'s official per-evaluation work; the survey
    quotes cfg4 F_eval = 1.765e10 flop and B_eval = 1.645e7 bytes, cfg2 1.21e7 / 6.78e4."""
    from paper_2112_10239_b200 import chain as C
    from paper_2112_10239_b200 import roofline
    from paper_2112_10239_b200.workloads import CONFIGS

    for name, f_eval, b_eval in (("cfg4", 1.765e10, 1.645e7), ("cfg2", 1.21e7, 6.78e4)):
        cfg = CONFIGS[name]
        terms = C.normalize_terms(cfg.hamiltonian())
        t1 = sum(1 for _, ops in terms if len(ops) == 1)
        t2 = sum(1 for _, ops in terms if len(ops) == 2)
        m = roofline.survey_model(C.compile_chain(cfg.circuit(), terms, "energy", segments=1), t1, t2,
                                  cfg.layers, cfg.grad)
        assert abs(m["F_eval"] / f_eval - 1) < 5e-3, (name, m)   # the survey rounds to 3-4 digits
        assert abs(m["B_eval"] / b_eval - 1) < 5e-3, (name, m)


def test_taped_truncation_rule():
    """The reference's taped path keeps every singular value at eps = 0 (zeros too), so its bond
    after a split is min(2 chi_l, 2 chi_r): a chi_max below that cuts the tape even when the
    factored bond fits (autodiff._taped_truncates)."""
    from paper_2112_10239_b200 import autodiff as AD
    from paper_2112_10239_b200.maxcut import brickwork_ansatz
    from paper_2112_10239_b200.workloads import layered_circuit

    bw = brickwork_ansatz(5, 3)                      # factored bond 2, taped bonds reach 4
    assert not AD._truncating(bw, 0.0, 2) and AD._taped_truncates(bw, 0.0, 2)
    assert not AD._taped_truncates(bw, 0.0, 4) and not AD._taped_truncates(bw, 0.0, None)
    assert AD._taped_truncates(bw, 1e-3, None)       # eps > 0 may cut anywhere
    c = layered_circuit(6, 2)                        # one entangler line: taped bonds stay 2
    assert not AD._taped_truncates(c, 0.0, 2)


def test_real_path_flag():
    """chain.real_path (tq_chain.real_path): real iff every factor, input vector and MPO edge is
    real -- ry + CZ/CNOT + X/Z terms yes; rx / rz rotations or a Y term no."""
    from paper_2112_10239_b200 import chain as C
    from paper_2112_10239_b200.hamiltonians import PauliHamiltonian, term, tfim
    from paper_2112_10239_b200.workloads import layered_circuit

    def flag(rot, ent, ham):
        return C.real_path(C.compile_chain(layered_circuit(10, 4, rot, ent), C.normalize_terms(ham), "energy"))

    assert flag("ry", "cz", tfim(10)) and flag("ry", "cnot", tfim(10))
    assert not flag("rx", "cz", tfim(10)) and not flag("rz", "cnot", tfim(10))
    ham_y = PauliHamiltonian(10, tfim(10).terms + (term(0.5, ((3, "Y"), (4, "Y"))),))
    assert not flag("ry", "cz", ham_y)


def test_executed_model_counts_real_fmas_on_real_path():
    """bench.py's executed-work model charges 2 flops per cMAC (one real FMA) when the plan runs
    the real-part instantiation, 8 otherwise; the cMAC count itself is unchanged."""
    import bench
    from paper_2112_10239_b200 import chain as C
    from paper_2112_10239_b200 import roofline
    from paper_2112_10239_b200.workloads import CONFIGS

    cfg = CONFIGS["cfg2"]
    _, e = bench.work_model(cfg, cfg.circuit(), cfg.hamiltonian(), cfg.batch)
    plan = C.compile_chain(cfg.circuit(), C.normalize_terms(cfg.hamiltonian()), "energy", segments=1)
    full = roofline.eval_model(plan, grad=True)
    assert e["real_path"] and e["flops_per_cmac"] == 2.0 and not full["real_path"]
    assert abs(e["flops_rl"] * 4 - full["flops_rl"]) < 1e-6 * full["flops_rl"]
    assert abs(e["flops_lr"] * 4 - full["flops_lr"]) < 1e-6 * full["flops_lr"]
    assert e["flops_adj"] == full["flops_adj"]          # chi 8: the warp adjoint stays complex
    c4 = CONFIGS["cfg4"]
    _, e4 = bench.work_model(c4, c4.circuit(), c4.hamiltonian(), c4.batch)
    assert e4["flops_per_cmac_adj"] == 2.0                 # chi 32: digit-tree adjoint, real
