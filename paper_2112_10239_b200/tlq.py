"""tlquantum-style drop-in API (north_star: TTCircuit, Unary rotation layers,
BinaryGatesUnitary CNOT/CZ layers, forward_expectation_value, state_inner_product,
Pauli/Ising/MaxCut operators).

The names follow TensorLy-Quantum; their semantics are pinned to the reference
``tnsim``: a ``TTCircuit`` compiles to the gate list
R, L0, R, L1, ... (reading A) that ``tnsim.Circuit`` would hold, and every value
is checked against the oracle.  The tensor-contraction knobs of tlquantum
(``ncontraq``, ``ncontral``, contraction equations) are accepted and ignored:
the B200 engine always contracts the chain with its own fused sweeps.

Parameters are ``torch.nn.Parameter`` scalars owned by the rotation gates, so
``energy.backward()`` fills ``gate.theta.grad`` like a tlquantum model; the
gradient comes from the engine's reverse sweep, not from torch autograd over a
contraction graph.
"""

from __future__ import annotations

import math

import numpy as np
import torch
from torch import nn

from . import chain as C
from . import engine as E
from .autodiff import _device, state_inner_product as _inner
from .circuits import Circuit, custom_gate, standard_gate
from .errors import InputError, SizeMismatch
from .hamiltonians import PauliHamiltonian, PauliTerm

__all__ = ["RotX", "RotY", "RotZ", "cnot", "cz", "Unitary", "UnaryGatesUnitary", "BinaryGatesUnitary",
           "TTCircuit", "ProductState", "TTState", "spins_to_tt_state", "pauli_x", "pauli_y", "pauli_z",
           "unary_hamiltonian", "binary_hamiltonian", "ising_hamiltonian", "maxcut_readouts"]


# ----------------------------------------------------------------------------- gates
class _Rot(nn.Module):
    axis = "y"

    def __init__(self, theta: float | None = None, dtype=torch.float32, device=None, seed=None):
        super().__init__()
        if theta is None:
            g = np.random.default_rng(seed)
            theta = float(g.uniform(-math.pi, math.pi))
        self.theta = nn.Parameter(torch.tensor([float(theta)], dtype=dtype, device=device))

    @property
    def name(self) -> str:
        return "r" + self.axis


class RotX(_Rot):
    axis = "x"


class RotY(_Rot):
    axis = "y"


class RotZ(_Rot):
    axis = "z"


def cnot():
    """CNOT with the control on the lower qubit of the pair (reference circuits.py:48-50)."""
    return "cnot"


def cz():
    return "cz"


# ----------------------------------------------------------------------------- layers
class Unitary(nn.Module):
    """One layer of single-qubit gates, one per qubit (None = identity)."""

    def __init__(self, gates, nqubits: int, ncontraq: int = 1):
        super().__init__()
        if len(gates) != nqubits:
            raise SizeMismatch(f"{len(gates)} gates for {nqubits} qubits")
        self.nqubits = int(nqubits)
        self.gates = nn.ModuleList([g if g is not None else nn.Identity() for g in gates])
        self.ncontraq = ncontraq

    def ir(self, offset_params: int):
        gates, train, params = [], [], []
        for q, g in enumerate(self.gates):
            if isinstance(g, _Rot):
                gates.append(standard_gate(g.name, (q,), 0.0))
                train.append(len(gates) - 1)
                params.append(g.theta)
        return gates, train, params


class UnaryGatesUnitary(Unitary):
    """A row of trainable rotations (tlquantum's Unary layer); axis in {'x','y','z'}."""

    def __init__(self, nqubits: int, ncontraq: int = 1, axis: str = "y", seed=None, dtype=torch.float32, device=None):
        cls = {"x": RotX, "y": RotY, "z": RotZ}[axis]
        rng = np.random.default_rng(seed)
        gates = [cls(float(rng.uniform(-math.pi, math.pi)), dtype=dtype, device=device) for _ in range(nqubits)]
        super().__init__(gates, nqubits, ncontraq)


class BinaryGatesUnitary(nn.Module):
    """A line of two-qubit gates on (q, q+1), q = parity (mod 2)."""

    def __init__(self, nqubits: int, ncontraq: int = 1, q2gate="cz", parity: int = 0):
        super().__init__()
        self.nqubits, self.parity, self.ncontraq = int(nqubits), int(parity) % 2, ncontraq
        if isinstance(q2gate, str):
            if q2gate not in ("cz", "cnot", "swap"):
                raise InputError(f"unknown two-qubit gate {q2gate!r}")
            self.gate_name, self.matrix = q2gate, None
        else:
            self.gate_name, self.matrix = "custom", np.asarray(q2gate, dtype=complex).reshape(4, 4)

    def ir(self, offset_params: int):
        gates = []
        for q in range(self.parity, self.nqubits - 1, 2):
            if self.matrix is None:
                gates.append(standard_gate(self.gate_name, (q, q + 1)))
            else:
                gates.append(custom_gate("custom", (q, q + 1), self.matrix))
        return gates, [], []


# ----------------------------------------------------------------------------- states
class ProductState:
    """Product input state as per-qubit complex 2-vectors (tlquantum spins_to_tt_state)."""

    def __init__(self, vectors):
        v = np.asarray(vectors, dtype=complex)
        if v.ndim != 2 or v.shape[1] != 2:
            raise InputError("product state needs an [n, 2] array of single-qubit vectors")
        self.vectors = v

    @property
    def nqubits(self) -> int:
        return self.vectors.shape[0]

    def is_zero(self) -> bool:
        return bool(np.all(self.vectors[:, 0] == 1) and np.all(self.vectors[:, 1] == 0))


class TTState:
    """An arbitrary tensor-train input state: n cores of shape (chi_l, 2, chi_r) (the reference's
    TTState.cores, tt.py:38-76; bonds <= 32).  TTCircuit.forward_expectation_value on it is
    differentiable (exact gradient, autodiff.expval_state); state_inner_product accepts it too."""

    def __init__(self, cores):
        self.cores = [np.asarray(c, dtype=complex) for c in getattr(cores, "cores", cores)]
        if not self.cores or any(c.ndim != 3 or c.shape[1] != 2 for c in self.cores):
            raise InputError("a TT state needs cores of shape (chi_l, 2, chi_r)")

    @property
    def nqubits(self) -> int:
        return len(self.cores)

    @classmethod
    def from_product(cls, state: "ProductState") -> "TTState":
        return cls([v.reshape(1, 2, 1) for v in state.vectors])


class _TrainExpval(torch.autograd.Function):
    """E[b] on an arbitrary input train; gradient from the same engine calls (exact shift rule on
    frozen-constant replays, truncated.straight_through)."""

    @staticmethod
    def forward(ctx, theta, circuit, ham, state):
        from .autodiff import expval_state

        want = bool(ctx.needs_input_grad[0])
        e, g = expval_state(circuit, ham, theta.detach().double().cpu().numpy(), state.cores, want_grad=want,
                            device=theta.device if theta.is_cuda else None)
        if want:
            ctx.save_for_backward(torch.as_tensor(g, dtype=theta.dtype, device=theta.device))
        return torch.as_tensor(e, dtype=torch.float64, device=theta.device)

    @staticmethod
    def backward(ctx, g_e):
        (g,) = ctx.saved_tensors
        return (g_e.to(g.dtype)[:, None] * g), None, None, None


def spins_to_tt_state(spins) -> ProductState:
    """|s_0 s_1 ...> for bits s_i (qubit 0 most significant)."""
    vecs = np.zeros((len(spins), 2), dtype=complex)
    for i, s in enumerate(spins):
        vecs[i, int(s)] = 1.0
    return ProductState(vecs)


# ----------------------------------------------------------------------------- circuit
class TTCircuit(nn.Module):
    """A chain of unitaries (alternate rotation rows and entangler lines for the
    canonical ansatz) evaluated by the B200 TT engine."""

    def __init__(self, unitaries, ncontraq: int = 1, ncontral: int = 1, equations=None, contrsets=None,
                 dtype: str = "complex64", device=None):
        super().__init__()
        self.unitaries = nn.ModuleList(unitaries)
        if not unitaries:
            raise InputError("TTCircuit needs at least one unitary")
        self.nqubits = unitaries[0].nqubits
        for u in unitaries:
            if u.nqubits != self.nqubits:
                raise SizeMismatch("all unitaries must act on the same number of qubits")
        self.ncontraq, self.ncontral, self.dtype = ncontraq, ncontral, dtype
        self.device = device
        gates, train, params = [], [], []
        for u in unitaries:
            g, t, p = u.ir(len(params))
            base = len(gates)
            gates.extend(g)
            train.extend(base + i for i in t)
            params.extend(p)
        self._circuit = Circuit(self.nqubits, tuple(gates), tuple(train))
        self._params = params

    def to_circuit(self) -> Circuit:
        """The equivalent reference-convention Circuit (for tnsim parity)."""
        return self._circuit

    def theta(self) -> torch.Tensor:
        """All trainable angles, in circuit slot order (differentiable)."""
        if not self._params:
            return torch.zeros(0)
        return torch.cat([p.reshape(1) for p in self._params])

    def _dev(self):
        return _device(self.device)

    def forward_expectation_value(self, state: ProductState | None, operator: PauliHamiltonian,
                                  theta: torch.Tensor | None = None) -> torch.Tensor:
        """<state|U(theta)^H H U(theta)|state>, differentiable w.r.t. the gate parameters
        (or w.r.t. ``theta`` [B, P] if given: returns [B])."""
        if operator.n_qubits != self.nqubits:
            raise SizeMismatch(f"operator on {operator.n_qubits} qubits, circuit {self.nqubits}")
        dev = self._dev()
        if isinstance(state, TTState):   # an arbitrary train: the taped engine from that state
            if state.nqubits != self.nqubits:
                raise SizeMismatch("state and circuit qubit counts differ")
            single = theta is None
            th = self.theta().to(dev)[None] if single else theta.to(dev)
            val = _TrainExpval.apply(th, self._circuit, operator, state)
            return val[0] if single else val
        init = None if state is None or state.is_zero() else state.vectors
        if state is not None and state.nqubits != self.nqubits:
            raise SizeMismatch("state and circuit qubit counts differ")
        single = theta is None
        th = self.theta().to(dev)[None] if single else theta.to(dev)
        terms = C.normalize_terms(operator)
        dp = E.device_plan(self._circuit, terms, "energy", th.shape[0], dev, None, init=init, dtype=self.dtype)
        coef = torch.tensor([[c.real for c, _ in terms]], dtype=torch.float64, device=dev)
        val, full = E.ExpvalFunction.apply(th, dp, coef, self.dtype)
        E.check_finite(full)
        return val[0] if single else val

    def forward(self, state, operator):
        return self.forward_expectation_value(state, operator)

    def state_inner_product(self, state: ProductState | None, compare_state: ProductState | None) -> torch.Tensor:
        """<compare_state| U(theta) |state>: a complex scalar tensor whose gradient flows to the
        rotation parameters (exact shift rule, one batched launch; autodiff.InnerFunction)."""
        from .autodiff import inner

        if isinstance(state, TTState) or isinstance(compare_state, TTState):
            # arbitrary trains: the circuit applied to the ket train on the truncated engine (no
            # truncation), then the train-train transfer <compare|U|state> (forward only)
            from . import truncated as TR

            def train(s):
                if s is None:
                    s = spins_to_tt_state([0] * self.nqubits)
                s = s if isinstance(s, TTState) else TTState.from_product(s)
                return TR.GPUTrain.from_cores(s.cores, dtype="complex128", device=self._dev())

            ket = TR.apply_circuit(train(state), self._circuit, self.theta().detach().double().cpu().numpy())
            z = TR.tt_inner(train(compare_state), ket)[0]
            return torch.tensor(complex(z), dtype=torch.complex128, device=self._dev())
        ki = None if state is None else state.vectors
        bi = None if compare_state is None else compare_state.vectors
        th = self.theta().to(self._dev())
        return inner(self._circuit, th, None, None, ket_init=ki, bra_init=bi, dtype=self.dtype)[0]


# ----------------------------------------------------------------------------- operators
def pauli_x():
    return "X"


def pauli_y():
    return "Y"


def pauli_z():
    return "Z"


def unary_hamiltonian(op, nqubits: int, qubits=None, weights=None) -> PauliHamiltonian:
    """sum_i w_i op_{q_i} (default: every qubit, weight 1)."""
    qubits = list(range(nqubits)) if qubits is None else [int(q) for q in qubits]
    weights = [1.0] * len(qubits) if weights is None else list(weights)
    return PauliHamiltonian(nqubits, tuple(PauliTerm(w, ((q, op),)) for q, w in zip(qubits, weights)))


def binary_hamiltonian(op, nqubits: int, qubits1=None, qubits2=None, weights=None) -> PauliHamiltonian:
    """sum_i w_i op_{q1_i} op_{q2_i} (default: nearest-neighbour open chain)."""
    qubits1 = list(range(nqubits - 1)) if qubits1 is None else [int(q) for q in qubits1]
    qubits2 = [q + 1 for q in qubits1] if qubits2 is None else [int(q) for q in qubits2]
    weights = [1.0] * len(qubits1) if weights is None else list(weights)
    return PauliHamiltonian(nqubits, tuple(PauliTerm(w, {a: op, b: op}) for a, b, w in zip(qubits1, qubits2, weights)))


def ising_hamiltonian(nqubits: int, j: float = 1.0, h: float = 1.0) -> PauliHamiltonian:
    """Transverse-field Ising chain, ZZ terms first (same term order as tnsim.tfim)."""
    return binary_hamiltonian("Z", nqubits, weights=[-j] * (nqubits - 1)) + unary_hamiltonian("X", nqubits, weights=[-h] * nqubits)


def maxcut_readouts(num_vertices: int) -> PauliHamiltonian:
    """MBE readout operators: vertex 2k -> Z_k, 2k+1 -> X_k (reference maxcut.py:127-135)."""
    n = (num_vertices + 1) // 2
    return PauliHamiltonian(max(n, 1), tuple(PauliTerm(1.0, ((v // 2, "Z" if v % 2 == 0 else "X"),))
                                             for v in range(num_vertices)))


def ansatz(nqubits: int, layers: int, rot: str = "y", ent: str = "cz", seed=None, dtype: str = "complex64",
           device=None) -> TTCircuit:
    """Reading-A TTCircuit: even layers rotation rows, odd layers entangler lines with parity 0,1,0,..."""
    units = []
    for l in range(layers):
        if l % 2 == 0:
            units.append(UnaryGatesUnitary(nqubits, axis=rot, seed=None if seed is None else seed + l))
        else:
            units.append(BinaryGatesUnitary(nqubits, q2gate=ent, parity=(l // 2) % 2))
    return TTCircuit(units, dtype=dtype, device=device)
