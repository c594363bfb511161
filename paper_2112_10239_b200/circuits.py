"""Gate-level circuit IR with the reference's conventions and validation.

Mirrors ``tnsim.circuits`` (reference ``circuits.py:1-241``): qubit 0 is the most
significant bit; ``R_a(t) = exp(-i t sigma_a / 2)``; two-qubit matrices order
their wires as given (first wire most significant); controlled gates use the
first wire as control; ``Circuit.trainable`` lists gate positions whose params
form the gradient vector, in order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import (
    ArityMismatch,
    InputError,
    MissingParam,
    ParamCountMismatch,
    UnknownGate,
    WireOutOfRange,
)

_SQ2 = 1.0 / math.sqrt(2.0)

FIXED_MATRICES = {  # reference circuits.py:41-55
    "h": np.array([[_SQ2, _SQ2], [_SQ2, -_SQ2]], dtype=complex),
    "x": np.array([[0, 1], [1, 0]], dtype=complex),
    "y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "z": np.array([[1, 0], [0, -1]], dtype=complex),
    "s": np.array([[1, 0], [0, 1j]], dtype=complex),
    "t": np.array([[1, 0], [0, np.exp(1j * math.pi / 4)]], dtype=complex),
    "cnot": np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex),
    "cz": np.diag([1, 1, 1, -1]).astype(complex),
    "swap": np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex),
}
PARAM_GATES = frozenset({"rx", "ry", "rz", "crz"})
STANDARD_GATES = frozenset(FIXED_MATRICES) | PARAM_GATES
ARITY = {**{g: 1 for g in ("h", "x", "y", "z", "s", "t", "rx", "ry", "rz")},
         **{g: 2 for g in ("cnot", "cz", "crz", "swap")}}


def gate_matrix(name: str, param: float | None = None) -> np.ndarray:
    """Matrix of a standard gate (reference circuits.py:64-85)."""
    if name in FIXED_MATRICES:
        return FIXED_MATRICES[name].copy()
    if name not in PARAM_GATES:
        raise UnknownGate(f"unknown gate '{name}'")
    if param is None:
        raise MissingParam(f"gate '{name}' requires a parameter")
    t = float(param)
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    if name == "rx":
        return np.array([[c, -1j * s], [-1j * s, c]])
    if name == "ry":
        return np.array([[c, -s], [s, c]], dtype=complex)
    if name == "rz":
        return np.diag([np.exp(-0.5j * t), np.exp(0.5j * t)])
    return np.diag([1.0, 1.0, np.exp(-0.5j * t), np.exp(0.5j * t)])


def gate_matrix_derivative(name: str, param: float) -> np.ndarray:
    """d(matrix)/d(theta) (reference circuits.py:88-102)."""
    if name not in PARAM_GATES:
        raise UnknownGate(f"gate '{name}' has no parameter derivative")
    t = float(param)
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    if name == "rx":
        return 0.5 * np.array([[-s, -1j * c], [-1j * c, -s]])
    if name == "ry":
        return 0.5 * np.array([[-s, -c], [c, -s]], dtype=complex)
    if name == "rz":
        return np.diag([-0.5j * np.exp(-0.5j * t), 0.5j * np.exp(0.5j * t)])
    return np.diag([0.0, 0.0, -0.5j * np.exp(-0.5j * t), 0.5j * np.exp(0.5j * t)])


@dataclass(frozen=True)
class Gate:
    """A gate bound to wires (reference circuits.py:105-130)."""

    name: str
    wires: tuple
    matrix: np.ndarray
    param: float | None = None

    def __post_init__(self):
        wires = tuple(int(w) for w in self.wires)
        object.__setattr__(self, "wires", wires)
        if len(set(wires)) != len(wires):
            raise ArityMismatch(f"gate '{self.name}' repeats a wire: {wires}")
        if any(w < 0 for w in wires):
            raise WireOutOfRange(f"negative wire in {wires}")
        m = np.asarray(self.matrix, dtype=complex)
        dim = 2 ** len(wires)
        if m.shape != (dim, dim):
            raise ArityMismatch(f"gate '{self.name}' on {len(wires)} wires needs a {dim}x{dim} matrix")
        m = m.copy()
        m.flags.writeable = False
        object.__setattr__(self, "matrix", m)


def standard_gate(name: str, wires, param: float | None = None) -> Gate:
    """Reference circuits.py:150-170."""
    name = str(name)
    if name not in STANDARD_GATES:
        raise UnknownGate(f"unknown gate '{name}'")
    wires = (int(wires),) if isinstance(wires, (int, np.integer)) else tuple(int(w) for w in wires)
    if len(wires) != ARITY[name]:
        raise ArityMismatch(f"gate '{name}' acts on {ARITY[name]} wire(s), got {len(wires)}")
    if name in PARAM_GATES:
        if param is None:
            raise MissingParam(f"gate '{name}' requires a parameter")
        param = float(param)
    elif param is not None:
        raise MissingParam(f"gate '{name}' takes no parameter")
    return Gate(name, wires, gate_matrix(name, param), param)


def custom_gate(name: str, wires, matrix, *, tol: float = 1e-10) -> Gate:
    """Explicit (unitary) matrix gate (reference circuits.py:173-184)."""
    m = np.asarray(matrix, dtype=complex)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise InputError("custom gate matrix must be square")
    if np.max(np.abs(m.conj().T @ m - np.eye(m.shape[0]))) > tol:
        raise InputError(f"matrix for '{name}' is not unitary within {tol}")
    return Gate(str(name), tuple(int(w) for w in wires), m, None)


@dataclass(frozen=True)
class Circuit:
    """Ordered gate list + trainable slots (reference circuits.py:187-227)."""

    n_qubits: int
    gates: tuple
    trainable: tuple = ()

    def __post_init__(self):
        if self.n_qubits < 1:
            raise InputError(f"n_qubits must be >= 1, got {self.n_qubits}")
        object.__setattr__(self, "gates", tuple(self.gates))
        object.__setattr__(self, "trainable", tuple(int(i) for i in self.trainable))
        for g in self.gates:
            if max(g.wires) >= self.n_qubits:
                raise WireOutOfRange(f"gate '{g.name}' wires {g.wires} exceed register of {self.n_qubits}")
        seen = set()
        for idx in self.trainable:
            if not 0 <= idx < len(self.gates):
                raise InputError(f"trainable index {idx} out of range")
            if self.gates[idx].param is None:
                raise MissingParam(f"trainable index {idx} refers to '{self.gates[idx].name}' which has no parameter")
            if idx in seen:
                raise InputError(f"trainable index {idx} listed twice")
            seen.add(idx)

    @property
    def n_params(self) -> int:
        return len(self.trainable)

    def params(self) -> np.ndarray:
        return np.array([self.gates[i].param for i in self.trainable], dtype=float)

    def structure_key(self):
        """Hashable key of everything except trainable parameter values (for plan caching)."""
        cached = self.__dict__.get("_skey")
        if cached is not None:
            return cached
        tr = set(self.trainable)
        parts = []
        for i, g in enumerate(self.gates):
            if i in tr:
                parts.append((g.name, g.wires, "T"))
            else:
                parts.append((g.name, g.wires, g.matrix.tobytes()))
        key = (self.n_qubits, tuple(parts), self.trainable)
        object.__setattr__(self, "_skey", key)
        return key


def with_params(circuit: Circuit, theta) -> Circuit:
    """Reference circuits.py:230-241."""
    theta = np.asarray(theta, dtype=float)
    if theta.shape != (circuit.n_params,):
        raise ParamCountMismatch(f"expected {circuit.n_params} parameters, got shape {theta.shape}")
    gates = list(circuit.gates)
    for slot, idx in enumerate(circuit.trainable):
        g = gates[idx]
        gates[idx] = standard_gate(g.name, g.wires, float(theta[slot]))
    return Circuit(circuit.n_qubits, tuple(gates), circuit.trainable)


# ---------------------------------------------------------------- JSON documents
# Same document shape as the reference (circuits.py:344-372), so circuit files written by
# ``tnsim`` load here unchanged and vice versa: {"n_qubits", "gates": [{name, wires[, param]}],
# "trainable": [...]}.

def circuit_to_dict(circuit: Circuit) -> dict:
    out_gates = []
    for g in circuit.gates:
        if g.name not in STANDARD_GATES:
            raise UnknownGate(f"gate '{g.name}' has no JSON form (custom matrix)")
        doc = {"name": g.name, "wires": list(g.wires)}
        if g.param is not None:
            doc["param"] = g.param
        out_gates.append(doc)
    return {"n_qubits": circuit.n_qubits, "gates": out_gates, "trainable": list(circuit.trainable)}


def circuit_from_dict(doc: dict) -> Circuit:
    """Inverse of :func:`circuit_to_dict`; structural problems raise ``ParseError``."""
    from .errors import ParseError

    try:
        n = int(doc["n_qubits"])
        entries = doc["gates"]
        trainable = tuple(int(i) for i in doc.get("trainable", ()))
        gates = tuple(standard_gate(e["name"], e["wires"], e.get("param")) for e in entries)
    except (KeyError, TypeError) as exc:
        raise ParseError(f"malformed circuit document: {exc!r}") from exc
    return Circuit(n, gates, trainable)
