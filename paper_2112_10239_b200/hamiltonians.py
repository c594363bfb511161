"""Pauli-sum operators (mirrors reference ``tnsim/hamiltonians.py:26-107``).

A Hamiltonian is a weighted sum of Pauli strings; each string is a sparse map
qubit -> 'X' | 'Y' | 'Z'.  The B200 engine never forms any 2^n object: the
operator is compiled into a matrix-product-operator automaton
(:mod:`paper_2112_10239_b200.chain`) whose transfer channels are swept on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError, QubitOutOfRange

PAULI_MATRICES = {
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
}
PAULI_CODE = {"I": 0, "X": 1, "Y": 2, "Z": 3}
RESIDUE_TOL = 1e-8  # reference hamiltonians.py:34 (complex128); complex64 scales it, see engine


@dataclass(frozen=True)
class PauliTerm:
    """One weighted Pauli string; ``ops`` maps qubit -> letter (reference hamiltonians.py:37-61)."""

    coeff: complex
    ops: tuple

    def __post_init__(self):
        coeff = complex(self.coeff)
        if not (np.isfinite(coeff.real) and np.isfinite(coeff.imag)):
            raise InputError(f"coefficient {self.coeff!r} is not finite")
        items = tuple(sorted((int(q), str(op)) for q, op in dict(self.ops).items()))
        for q, op in items:
            if q < 0:
                raise QubitOutOfRange(f"negative qubit index {q}")
            if op not in PAULI_MATRICES:
                raise InputError(f"unknown Pauli letter {op!r}")
        object.__setattr__(self, "coeff", coeff)
        object.__setattr__(self, "ops", items)

    @property
    def support(self) -> tuple:
        return tuple(q for q, _ in self.ops)


def term(coeff, ops) -> PauliTerm:
    """Reference hamiltonians.py:64-66."""
    return PauliTerm(coeff, tuple(dict(ops).items()))


@dataclass(frozen=True)
class PauliHamiltonian:
    """Reference hamiltonians.py:69-90."""

    n_qubits: int
    terms: tuple

    def __post_init__(self):
        if self.n_qubits < 1:
            raise InputError(f"need at least one qubit, got {self.n_qubits}")
        object.__setattr__(self, "terms", tuple(self.terms))
        for t in self.terms:
            if not isinstance(t, PauliTerm):
                raise InputError(f"terms must be PauliTerm, got {type(t).__name__}")
            for q, _ in t.ops:
                if q >= self.n_qubits:
                    raise QubitOutOfRange(f"term acts on qubit {q} but n_qubits={self.n_qubits}")

    def __add__(self, other: "PauliHamiltonian") -> "PauliHamiltonian":
        if other.n_qubits != self.n_qubits:
            raise InputError("cannot add Hamiltonians on different qubit counts")
        return PauliHamiltonian(self.n_qubits, self.terms + other.terms)

    def structure_key(self):
        return (self.n_qubits, tuple(t.ops for t in self.terms))

    def coefficients(self) -> np.ndarray:
        return np.array([t.coeff for t in self.terms], dtype=complex)


def tfim(n_qubits: int, j: float = 1.0, h: float = 1.0, periodic: bool = False) -> PauliHamiltonian:
    """H = -j sum Z_k Z_{k+1} - h sum X_k; ZZ terms first (reference hamiltonians.py:93-107)."""
    n = int(n_qubits)
    if n < 1:
        raise InputError(f"need at least one qubit, got {n}")
    bonds = n if periodic and n > 1 else n - 1
    terms = [term(-float(j), {k: "Z", (k + 1) % n: "Z"}) for k in range(bonds)]
    terms += [term(-float(h), {k: "X"}) for k in range(n)]
    return PauliHamiltonian(n, tuple(terms))


# ---------------------------------------------------------------- JSON documents
# Reference document shape (hamiltonians.py:227-271): {"n_qubits", "terms": [{"coeff": real,
# "ops": {"<qubit>": "X"|"Y"|"Z"}}]}.

def hamiltonian_to_dict(ham: PauliHamiltonian) -> dict:
    return {"n_qubits": ham.n_qubits,
            "terms": [{"coeff": t.coeff.real, "ops": {str(q): op for q, op in t.ops}} for t in ham.terms]}


def hamiltonian_from_dict(doc) -> PauliHamiltonian:
    """Validating loader; every structural problem is a ``ParseError`` (an ``InputError``)."""
    from .errors import ParseError

    if not isinstance(doc, dict):
        raise ParseError(f"expected an object, got {type(doc).__name__}")
    try:
        n = int(doc["n_qubits"])
        entries = doc["terms"]
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(f"malformed Hamiltonian object: {exc}") from exc
    if not isinstance(entries, list):
        raise ParseError("'terms' must be a list")
    out = []
    for i, e in enumerate(entries):
        if not isinstance(e, dict) or "coeff" not in e or "ops" not in e:
            raise ParseError(f"term {i} must have 'coeff' and 'ops'")
        c = e["coeff"]
        if isinstance(c, bool) or not isinstance(c, (int, float)):
            raise ParseError(f"term {i} coefficient must be a real number")
        if not isinstance(e["ops"], dict):
            raise ParseError(f"term {i} 'ops' must be an object")
        ops = {}
        for key, letter in e["ops"].items():
            try:
                ops[int(key)] = letter
            except (TypeError, ValueError):
                raise ParseError(f"term {i} has non-integer qubit key {key!r}")
        try:
            out.append(term(float(c), ops))
        except InputError as exc:
            raise ParseError(f"term {i}: {exc}") from exc
    try:
        return PauliHamiltonian(n, tuple(out))
    except InputError as exc:
        raise ParseError(str(exc)) from exc
