"""Shared test helpers: golden documents -> product IR objects."""

import numpy as np

from paper_2112_10239_b200.circuits import Circuit, standard_gate
from paper_2112_10239_b200.hamiltonians import PauliHamiltonian, PauliTerm


def to_circuit(doc):
    gates = tuple(standard_gate(name, tuple(wires), param) for name, wires, param in doc["gates"])
    return Circuit(doc["n"], gates, tuple(doc["trainable"]))


def to_ham(doc, n):
    return PauliHamiltonian(n, tuple(PauliTerm(complex(re, im), tuple((int(q), l) for q, l in ops))
                                     for re, im, ops in doc))


def tol64(ref_val, ham):
    """complex64 energy tolerance: 1e-5 * max(|E|, 1e-2 * sum|c|)."""
    s = sum(abs(t.coeff) for t in ham.terms)
    return 1e-5 * max(abs(ref_val), 1e-2 * s, 1e-3)


def grad_ok64(g, ref, ham=None, energy=None):
    """complex64 gradient bar of SURVEY.md section 8c: |dg| <= 1e-5 |g_ref| + 1e-6 ||g_ref||_inf.
    For gradient vectors that vanish identically (goldens whose angles cannot move the energy,
    e.g. rz rotations on basis states) fp32 leaves ~eps * |E| of rounding, so the floor takes the
    energy bar's scale instead (tol64: max(|E|, 1e-2 sum|c|)):
    1e-6 max(||g_ref||_inf, |E|, 1e-2 sum|c|)."""
    ref = np.asarray(ref)
    scale = np.max(np.abs(ref), initial=0.0)
    if ham is not None:
        scale = max(scale, 1e-2 * sum(abs(t.coeff) for t in ham.terms))
    if energy is not None:
        scale = max(scale, abs(energy))
    return np.all(np.abs(g - ref) <= 1e-5 * np.abs(ref) + 1e-6 * scale + 1e-12)
