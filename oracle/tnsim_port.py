"""numpy restatement of the reference ``tnsim`` hot path (test oracle, see package doc).

Conventions (reference ``circuits.py:1-12``): qubit 0 is the most significant
bit; ``R_a(t) = exp(-i t sigma_a / 2)``; two-qubit matrices order their wires as
given, first wire most significant.

Data model used here (plain Python, no reference classes):
  gate       = (name, wires tuple, param or None)
  circuit    = OCircuit(n, gates list, trainable list of gate indices)
  hamiltonian= list of (coeff complex, ops) with ops a sorted tuple ((q, 'X'|'Y'|'Z'), ...)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OCircuit", "gate_matrix", "gate_matrix_derivative", "with_params",
    "tfim_terms", "ry_cz_layers", "brickwork", "tfim_workload_gates",
    "simulate_dense", "expval_dense", "dense_term_values",
    "TT", "tt_zero", "apply_gate_tt", "simulate_tt", "canonicalize",
    "expval_tt", "tt_term_values", "tt_inner", "tt_to_dense", "tt_from_product",
    "grad_expval_tt", "taped_term_values", "evaluate_expval",
    "parameter_shift_grad", "finite_diff_grad",
    "mbe_encode", "mbe_objective", "vertex_expectations", "round_cut", "cut_value",
    "pairing_graph", "init_params", "generator", "spawn", "adam_minimize",
]

PAULI = {
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
}
_R2 = 1.0 / math.sqrt(2.0)
FIXED = {  # reference circuits.py:41-55
    "h": np.array([[_R2, _R2], [_R2, -_R2]], dtype=complex),
    "x": PAULI["X"].copy(),
    "y": PAULI["Y"].copy(),
    "z": PAULI["Z"].copy(),
    "s": np.diag([1, 1j]).astype(complex),
    "t": np.diag([1, np.exp(1j * math.pi / 4)]).astype(complex),
    "cnot": np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex),
    "cz": np.diag([1, 1, 1, -1]).astype(complex),
    "swap": np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex),
}
PARAMETRIC = ("rx", "ry", "rz", "crz")


# --------------------------------------------------------------------------- seeding
def generator(seed: int) -> np.random.Generator:
    """PCG64 stream (reference seeding.py:14-16)."""
    return np.random.Generator(np.random.PCG64(seed))


def spawn(seed: int, k: int):
    """Child streams via SeedSequence.spawn (reference seeding.py:19-22)."""
    return [np.random.Generator(np.random.PCG64(s)) for s in np.random.SeedSequence(seed).spawn(k)]


def init_params(p: int, rng) -> np.ndarray:
    """U[-pi, pi) angles (reference autodiff.py:609-611)."""
    return rng.uniform(-np.pi, np.pi, size=int(p))


# --------------------------------------------------------------------------- gates
def gate_matrix(name: str, param=None) -> np.ndarray:
    """Reference circuits.py:64-85."""
    if name in FIXED:
        return FIXED[name].copy()
    t = float(param)
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    if name == "rx":
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)
    if name == "ry":
        return np.array([[c, -s], [s, c]], dtype=complex)
    if name == "rz":
        return np.diag([np.exp(-0.5j * t), np.exp(0.5j * t)])
    if name == "crz":
        return np.diag([1.0, 1.0, np.exp(-0.5j * t), np.exp(0.5j * t)])
    raise ValueError(f"unknown gate {name!r}")


def gate_matrix_derivative(name: str, param) -> np.ndarray:
    """Reference circuits.py:88-102 (d/dtheta of the rotation matrices)."""
    t = float(param)
    c, s = math.cos(t / 2.0), math.sin(t / 2.0)
    if name == "rx":
        return 0.5 * np.array([[-s, -1j * c], [-1j * c, -s]])
    if name == "ry":
        return 0.5 * np.array([[-s, -c], [c, -s]], dtype=complex)
    if name == "rz":
        return np.diag([-0.5j * np.exp(-0.5j * t), 0.5j * np.exp(0.5j * t)])
    if name == "crz":
        return np.diag([0.0, 0.0, -0.5j * np.exp(-0.5j * t), 0.5j * np.exp(0.5j * t)])
    raise ValueError(f"gate {name!r} has no derivative")


@dataclass
class OCircuit:
    """Gate list + trainable slots (the reference Circuit, circuits.py:187-227)."""

    n: int
    gates: list
    trainable: list = field(default_factory=list)

    @property
    def n_params(self) -> int:
        return len(self.trainable)


def with_params(circ: OCircuit, theta) -> OCircuit:
    """Rebind trainable params in slot order (reference circuits.py:230-241)."""
    theta = np.asarray(theta, dtype=float).reshape(-1)
    if theta.shape[0] != circ.n_params:
        raise ValueError("parameter count mismatch")
    gates = list(circ.gates)
    for slot, gi in enumerate(circ.trainable):
        name, wires, _ = gates[gi]
        gates[gi] = (name, wires, float(theta[slot]))
    return OCircuit(circ.n, gates, list(circ.trainable))


# --------------------------------------------------------------------------- workloads
def tfim_terms(n: int, j: float = 1.0, h: float = 1.0, periodic: bool = False):
    """H = -j sum Z_k Z_k+1 - h sum X_k; ZZ terms first (reference hamiltonians.py:93-107)."""
    out = []
    bonds = n if periodic and n > 1 else n - 1
    for k in range(bonds):
        ops = {k: "Z", (k + 1) % n: "Z"}
        out.append((complex(-j), tuple(sorted(ops.items()))))
    for k in range(n):
        out.append((complex(-h), ((k, "X"),)))
    return out


def ry_cz_layers(n: int, layers: int, rot: str = "ry", ent: str = "cz") -> OCircuit:
    """Reading-A layer program: even layers are a trainable
    rotation row, odd layers an entangler line with parity alternating 0,1,0,..."""
    gates, train = [], []
    for l in range(layers):
        if l % 2 == 0:
            for q in range(n):
                train.append(len(gates))
                gates.append((rot, (q,), 0.0))
        else:
            p = (l // 2) % 2
            for q in range(p, n - 1, 2):
                gates.append((ent, (q, q + 1), None))
    return OCircuit(n, gates, train)


def brickwork(n: int, depth: int = 4) -> OCircuit:
    """ry+rz rows separated by cz lines (reference maxcut.py:186-203)."""
    gates, train = [], []
    for layer in range(depth):
        for name in ("ry", "rz"):
            for q in range(n):
                train.append(len(gates))
                gates.append((name, (q,), 0.0))
        if layer < depth - 1:
            for q in range(layer % 2, n - 1, 2):
                gates.append(("cz", (q, q + 1), None))
    return OCircuit(n, gates, train)


def tfim_workload_gates(n: int, n_gates: int) -> OCircuit:
    """Reference bench.py:70-96: brickwork stream cut to exactly n_gates."""
    gates, train = [], []
    layer = 0
    while len(gates) < n_gates:
        for name in ("ry", "rz"):
            for q in range(n):
                if len(gates) >= n_gates:
                    break
                train.append(len(gates))
                gates.append((name, (q,), 0.0))
        for q in range(layer % 2, n - 1, 2):
            if len(gates) >= n_gates:
                break
            gates.append(("cz", (q, q + 1), None))
        layer += 1
    return OCircuit(n, gates, train)


# --------------------------------------------------------------------------- dense engine
def simulate_dense(circ: OCircuit, theta=None) -> np.ndarray:
    """Statevector oracle (reference circuits.py:300-325); returns shape (2,)*n."""
    if theta is not None:
        circ = with_params(circ, theta)
    n = circ.n
    psi = np.zeros((2,) * n, dtype=complex)
    psi[(0,) * n] = 1.0
    for name, wires, param in circ.gates:
        k = len(wires)
        g = gate_matrix(name, param).reshape((2,) * (2 * k))
        psi = np.tensordot(g, psi, axes=(tuple(range(k, 2 * k)), tuple(wires)))
        psi = np.moveaxis(psi, tuple(range(k)), tuple(wires))
    return psi


def dense_term_values(psi: np.ndarray, terms) -> np.ndarray:
    """<psi|P_t|psi> per term (reference hamiltonians.py:110-126)."""
    flat = psi.reshape(-1)
    out = np.zeros(len(terms), dtype=complex)
    for i, (_, ops) in enumerate(terms):
        phi = psi
        for q, letter in ops:
            phi = np.moveaxis(np.tensordot(PAULI[letter], phi, axes=([1], [q])), 0, q)
        out[i] = np.vdot(flat, phi.reshape(-1))
    return out


def expval_dense(psi: np.ndarray, terms) -> complex:
    vals = dense_term_values(psi, terms)
    total = 0j
    for (c, _), v in zip(terms, vals):
        total += c * v
    return total


# --------------------------------------------------------------------------- TT engine
@dataclass
class TT:
    """Tensor train: cores (chi_l, 2, chi_r) + orthogonality centre (reference tt.py:38-76)."""

    cores: list
    center: int | None = None
    discarded: float = 0.0

    @property
    def n(self) -> int:
        return len(self.cores)

    @property
    def bonds(self):
        return (1,) + tuple(c.shape[2] for c in self.cores)


def tt_zero(n: int) -> TT:
    """|0...0> with bond 1 (reference tt.py:79-82)."""
    core = np.zeros((1, 2, 1), dtype=complex)
    core[0, 0, 0] = 1.0
    return TT([core.copy() for _ in range(n)], 0)


def tt_from_product(vectors) -> TT:
    """Product state from per-site 2-vectors (bond 1 everywhere)."""
    cores = [np.asarray(v, dtype=complex).reshape(1, 2, 1) for v in vectors]
    return TT(cores, None)


def _keep_count(s: np.ndarray, eps: float, chi_max):
    """Singular values kept, discarded weight, rescale (reference tt.py:85-100)."""
    total = float(s @ s)
    k = len(s)
    if eps > 0.0 and s[0] > 0.0:
        k = max(1, int(np.count_nonzero(s > eps * s[0])))
    if chi_max is not None:
        k = min(k, int(chi_max))
    kept = float(s[:k] @ s[:k])
    if total <= 0.0:
        return max(k, 1), 0.0, 1.0
    return k, max(0.0, 1.0 - kept / total), (math.sqrt(total / kept) if kept > 0 else 1.0)


def _svd_split(mat: np.ndarray, eps: float, chi_max):
    """Sigma to the thin side (reference tt.py:103-115)."""
    u, s, vh = np.linalg.svd(mat, full_matrices=False)
    k, disc, scale = _keep_count(s, eps, chi_max)
    sk = s[:k] * scale
    if mat.shape[0] <= mat.shape[1]:
        return u[:, :k], sk[:, None] * vh[:k], disc, True
    return u[:, :k] * sk[None, :], vh[:k], disc, False


def _qr_right(cores, c):
    """Reference tt.py:118-122."""
    cl, _, cr = cores[c].shape
    q, r = np.linalg.qr(cores[c].reshape(cl * 2, cr))
    cores[c] = q.reshape(cl, 2, q.shape[1])
    cores[c + 1] = np.tensordot(r, cores[c + 1], axes=([1], [0]))


def _qr_left(cores, c):
    """Reference tt.py:125-129."""
    cl, _, cr = cores[c].shape
    q, r = np.linalg.qr(cores[c].reshape(cl, 2 * cr).T)
    cores[c] = q.T.reshape(q.shape[1], 2, cr)
    cores[c - 1] = np.tensordot(cores[c - 1], r.T, axes=([2], [0]))


def _move_center(cores, center, target):
    """Reference tt.py:146-161."""
    if center is None:
        for c in range(target):
            _qr_right(cores, c)
        for c in range(len(cores) - 1, target, -1):
            _qr_left(cores, c)
        return target
    while center < target:
        _qr_right(cores, center)
        center += 1
    while center > target:
        _qr_left(cores, center)
        center -= 1
    return center


def canonicalize(tt: TT, center: int) -> TT:
    """Reference tt.py:132-143."""
    cores = [c.copy() for c in tt.cores]
    for c in range(center):
        _qr_right(cores, c)
    for c in range(len(cores) - 1, center, -1):
        _qr_left(cores, c)
    return TT(cores, center, tt.discarded)


def _two_site(cores, i, m4, eps, chi_max):
    """Merge, apply, split (reference tt.py:168-183)."""
    th = np.tensordot(cores[i], cores[i + 1], axes=([2], [0]))
    th = np.tensordot(m4.reshape(2, 2, 2, 2), th, axes=([2, 3], [1, 2])).transpose(2, 0, 1, 3)
    cl, _, _, cr = th.shape
    left, right, disc, on_right = _svd_split(th.reshape(cl * 2, 2 * cr), eps, chi_max)
    k = left.shape[1]
    cores[i] = left.reshape(cl, 2, k)
    cores[i + 1] = right.reshape(k, 2, cr)
    return (i + 1 if on_right else i), disc


def apply_gate_tt(tt: TT, gate, eps: float = 1e-12, chi_max=None) -> TT:
    """Reference tt.py:186-234 (SWAP chains for distant wires)."""
    name, wires, param = gate
    mat = gate_matrix(name, param)
    cores = list(tt.cores)
    center, disc = tt.center, tt.discarded
    if len(wires) == 1:
        k = wires[0]
        if center is not None:
            center = _move_center(cores, center, k)
        cores[k] = np.tensordot(mat, cores[k], axes=([1], [1])).transpose(1, 0, 2)
        return TT(cores, center, disc)
    lo, hi = min(wires), max(wires)
    if wires[0] > wires[1]:
        mat = mat.reshape(2, 2, 2, 2).transpose(1, 0, 3, 2).reshape(4, 4)
    sw = FIXED["swap"]

    def at(site, m):
        nonlocal center, disc
        center = _move_center(cores, center, site)
        center, d = _two_site(cores, site, m, eps, chi_max)
        disc += d

    for j in range(hi - 1, lo, -1):
        at(j, sw)
    at(lo, mat)
    for j in range(lo + 1, hi):
        at(j, sw)
    return TT(cores, center, disc)


def simulate_tt(circ: OCircuit, theta=None, eps: float = 1e-12, chi_max=None, init: TT | None = None) -> TT:
    """Reference tt.py:237-244."""
    if theta is not None:
        circ = with_params(circ, theta)
    state = tt_zero(circ.n) if init is None else init
    for g in circ.gates:
        state = apply_gate_tt(state, g, eps, chi_max)
    return state


def tt_term_values(tt: TT, terms) -> np.ndarray:
    """Per-term windows on a mixed-canonical copy (reference hamiltonians.py:129-160)."""
    if tt.center is None:
        tt = canonicalize(tt, 0)
    cores = list(tt.cores)
    center = tt.center
    vals = np.zeros(len(terms), dtype=complex)
    order = sorted(range(len(terms)), key=lambda i: (terms[i][1][0][0] if terms[i][1] else 0, i))
    for i in order:
        ops = dict(terms[i][1])
        if not ops:
            vals[i] = 1.0
            continue
        lo, hi = min(ops), max(ops)
        center = _move_center(cores, center, lo)
        env = np.eye(cores[lo].shape[0], dtype=complex)
        for k in range(lo, hi + 1):
            ket = np.tensordot(env, cores[k], axes=([1], [0]))
            if k in ops:
                ket = np.tensordot(PAULI[ops[k]], ket, axes=([1], [1])).transpose(1, 0, 2)
            env = np.tensordot(np.conj(cores[k]), ket, axes=([0, 1], [0, 1]))
        vals[i] = np.trace(env)
    return vals


def expval_tt(tt: TT, terms) -> complex:
    """Sum in original term order (reference hamiltonians.py:161-164)."""
    total = 0j
    for (c, _), v in zip(terms, tt_term_values(tt, terms)):
        total += c * v
    return total


def tt_inner(a: TT, b: TT) -> complex:
    """<a|b>, first argument conjugated (reference tt.py:247-255)."""
    env = np.ones((1, 1), dtype=complex)
    for ca, cb in zip(a.cores, b.cores):
        env = np.tensordot(env, np.conj(ca), axes=([0], [0]))
        env = np.tensordot(env, cb, axes=([0, 1], [0, 1]))
    return complex(env[0, 0])


def tt_to_dense(tt: TT) -> np.ndarray:
    """Reference tt.py:288-296."""
    acc = tt.cores[0].reshape(2, -1)
    for core in tt.cores[1:]:
        acc = np.tensordot(acc, core, axes=([-1], [0]))
    return acc.reshape((2,) * tt.n)


def evaluate_expval(circ: OCircuit, terms, theta, eps: float = 1e-12, chi_max=None) -> complex:
    """Untaped value (reference autodiff.py:490-503, engine='tt')."""
    return expval_tt(simulate_tt(circ, theta, eps, chi_max), terms)


# --------------------------------------------------------------------------- reverse mode
class _Var:
    """Node of a pullback graph.  Cotangent convention dL = Re sum(conj(g) dz)
    (reference autodiff.py:4-6)."""

    __slots__ = ("val", "parents", "uid")
    _counter = [0]

    def __init__(self, val, parents=()):
        self.val = val
        self.parents = parents  # tuple of (var, pullback(g) -> cotangent)
        _Var._counter[0] += 1
        self.uid = _Var._counter[0]


class _Graph:
    """Minimal reverse-mode recorder; nodes are visited in reverse creation order
    exactly like the reference tape (autodiff.py:190-247)."""

    def __init__(self):
        self.nodes = []
        self.leaves = {}  # uid -> (slot, dmat)

    def _node(self, val, parents=()):
        v = _Var(val, parents)
        self.nodes.append(v)
        return v

    def const(self, val):
        return self._node(np.asarray(val, dtype=complex))

    def leaf(self, val, slot, dmat):
        v = self._node(np.asarray(val, dtype=complex))
        self.leaves[v.uid] = (slot, np.asarray(dmat, dtype=complex))
        return v

    def dot(self, a, b, axes):
        """tensordot with its VJP written as einsum contractions."""
        ax_a, ax_b = list(axes[0]), list(axes[1])
        letters = iter("abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ")
        sa = [None] * a.val.ndim
        sb = [None] * b.val.ndim
        for i, j in zip(ax_a, ax_b):
            sa[i] = sb[j] = next(letters)
        for i in range(len(sa)):
            if sa[i] is None:
                sa[i] = next(letters)
        for j in range(len(sb)):
            if sb[j] is None:
                sb[j] = next(letters)
        out = [sa[i] for i in range(len(sa)) if i not in ax_a] + [sb[j] for j in range(len(sb)) if j not in ax_b]
        A, Bs, O = "".join(sa), "".join(sb), "".join(out)
        val = np.einsum(f"{A},{Bs}->{O}", a.val, b.val)
        av, bv = a.val, b.val
        return self._node(val, (
            (a, lambda g: np.einsum(f"{O},{Bs}->{A}", g, np.conj(bv))),
            (b, lambda g: np.einsum(f"{A},{O}->{Bs}", np.conj(av), g)),
        ))

    def conj(self, a):
        return self._node(np.conj(a.val), ((a, np.conj),))

    def transpose(self, a, perm):
        inv = np.argsort(perm)
        return self._node(a.val.transpose(perm), ((a, lambda g: g.transpose(inv)),))

    def reshape(self, a, shape):
        s0 = a.val.shape
        return self._node(a.val.reshape(shape), ((a, lambda g: g.reshape(s0)),))

    def add(self, a, b):
        return self._node(a.val + b.val, ((a, lambda g: g), (b, lambda g: g)))

    def scale(self, a, c):
        c = complex(c)
        return self._node(c * a.val, ((a, lambda g: np.conj(c) * g),))

    def mul(self, a, b):
        av, bv = a.val, b.val
        return self._node(av * bv, ((a, lambda g: g * np.conj(bv)), (b, lambda g: g * np.conj(av))))

    def tanh(self, a):
        t = np.tanh(a.val)
        return self._node(t, ((a, lambda g: g * np.conj(1.0 - t * t)),))

    def real(self, a):
        return self._node(np.asarray(a.val.real, dtype=complex), ((a, lambda g: np.asarray(complex(np.real(g)))),))

    def backward(self, out, n_slots):
        cot = {out.uid: np.asarray(1.0 + 0j)}
        grads = np.zeros(n_slots)
        for node in reversed(self.nodes):
            g = cot.pop(node.uid, None)
            if g is None:
                continue
            if node.uid in self.leaves:
                slot, dmat = self.leaves[node.uid]
                grads[slot] += float(np.sum(np.conj(g) * dmat).real)
                continue
            for parent, pull in node.parents:
                contrib = pull(g)
                if parent.uid in cot:
                    cot[parent.uid] = cot[parent.uid] + contrib
                else:
                    cot[parent.uid] = contrib
        return grads


def _taped_split(G, cores, i, g4, eps, chi_max):
    """Reference autodiff.py:315-336: SVD unitary factor recorded as a constant."""
    th = G.dot(cores[i], cores[i + 1], ([2], [0]))
    th = G.dot(g4, th, ([2, 3], [1, 2]))
    th = G.transpose(th, (2, 0, 1, 3))
    cl, _, _, cr = th.val.shape
    m, nn = cl * 2, 2 * cr
    mat = G.reshape(th, (m, nn))
    u, s, vh = np.linalg.svd(mat.val, full_matrices=False)
    k, _, scale = _keep_count(s, eps, chi_max)
    if m <= nn:
        left = G.const(u[:, :k])
        right = G.dot(G.const(u[:, :k].conj().T), mat, ([1], [0]))
        if scale != 1.0:
            right = G.scale(right, scale)
    else:
        right = G.const(vh[:k])
        left = G.dot(mat, G.const(vh[:k].conj().T), ([1], [0]))
        if scale != 1.0:
            left = G.scale(left, scale)
    cores[i] = G.reshape(left, (cl, 2, k))
    cores[i + 1] = G.reshape(right, (k, 2, cr))


def _taped_state(G, circ: OCircuit, theta, eps, chi_max, init_vectors=None):
    """Reference autodiff.py:267-283 (gate leaves) and 339-363 (taped state)."""
    n = circ.n
    cores = []
    for q in range(n):
        c = np.zeros((1, 2, 1), dtype=complex)
        if init_vectors is None:
            c[0, 0, 0] = 1.0
        else:
            c[0, :, 0] = init_vectors[q]
        cores.append(G.const(c))
    slot_of = {gi: s for s, gi in enumerate(circ.trainable)}
    swap4 = None
    for gi, (name, wires, param) in enumerate(circ.gates):
        if gi in slot_of:
            s = slot_of[gi]
            mid = G.leaf(gate_matrix(name, theta[s]), s, gate_matrix_derivative(name, theta[s]))
        else:
            mid = G.const(gate_matrix(name, param))
        if len(wires) == 1:
            k = wires[0]
            cores[k] = G.transpose(G.dot(mid, cores[k], ([1], [1])), (1, 0, 2))
            continue
        lo, hi = min(wires), max(wires)
        g4 = G.reshape(mid, (2, 2, 2, 2))
        if wires[0] > wires[1]:
            g4 = G.transpose(g4, (1, 0, 3, 2))
        if hi > lo + 1 and swap4 is None:
            swap4 = G.reshape(G.const(FIXED["swap"]), (2, 2, 2, 2))
        for j in range(hi - 1, lo, -1):
            _taped_split(G, cores, j, swap4, eps, chi_max)
        _taped_split(G, cores, lo, g4, eps, chi_max)
        for j in range(lo + 1, hi):
            _taped_split(G, cores, j, swap4, eps, chi_max)
    return cores


def _taped_terms(G, cores, op_groups):
    """Reference autodiff.py:366-402: shared prefix/suffix environments + windows."""
    n = len(cores)
    cc = [G.conj(c) for c in cores]
    left = [G.const(np.ones((1, 1)))]
    for k in range(n):
        t = G.dot(left[k], cc[k], ([0], [0]))
        left.append(G.dot(t, cores[k], ([0, 1], [0, 1])))
    right = [None] * (n + 1)
    right[n] = G.const(np.ones((1, 1)))
    for k in range(n - 1, -1, -1):
        t = G.dot(cc[k], right[k + 1], ([2], [0]))
        right[k] = G.dot(t, cores[k], ([1, 2], [1, 2]))
    cache = {}

    def opc(k, letter):
        if (k, letter) not in cache:
            t = G.dot(G.const(PAULI[letter]), cores[k], ([1], [1]))
            cache[(k, letter)] = G.transpose(t, (1, 0, 2))
        return cache[(k, letter)]

    out = []
    for ops in op_groups:
        if not ops:
            out.append(G.reshape(left[n], ()))
            continue
        sites = sorted(ops)
        env = left[sites[0]]
        for k in range(sites[0], sites[-1] + 1):
            ket = opc(k, ops[k]) if k in ops else cores[k]
            env = G.dot(G.dot(env, cc[k], ([0], [0])), ket, ([0, 1], [0, 1]))
        out.append(G.dot(env, right[sites[-1] + 1], ([0, 1], [0, 1])))
    return out


def grad_expval_tt(circ: OCircuit, terms, theta, eps: float = 0.0, chi_max=None, init_vectors=None):
    """Value + gradient, taped TT engine (reference autodiff.py:428-442, 471-487).

    Exact at eps=0 without a bond cap; returns (float value, float64[P])."""
    theta = np.asarray(theta, dtype=float).reshape(-1)
    G = _Graph()
    cores = _taped_state(G, circ, theta, eps, chi_max, init_vectors)
    vals = _taped_terms(G, cores, [dict(ops) for _, ops in terms])
    acc = None
    for (c, _), v in zip(terms, vals):
        sv = G.scale(v, c)
        acc = sv if acc is None else G.add(acc, sv)
    if acc is None:
        acc = G.const(np.asarray(0j))
    out = G.real(acc)
    return float(out.val.real), G.backward(out, circ.n_params)


def taped_term_values(circ: OCircuit, theta, op_groups, eps: float = 0.0, chi_max=None) -> np.ndarray:
    """Complex <P_t> per op-group sharing one state (reference autodiff.py:405-425)."""
    G = _Graph()
    cores = _taped_state(G, circ, np.asarray(theta, dtype=float), eps, chi_max)
    return np.array([complex(v.val) for v in _taped_terms(G, cores, [dict(o) for o in op_groups])])


_CRZ_A = (math.sqrt(2.0) + 1.0) / (4.0 * math.sqrt(2.0))
_CRZ_B = (math.sqrt(2.0) - 1.0) / (4.0 * math.sqrt(2.0))


def parameter_shift_grad(circ: OCircuit, terms, theta, eps: float = 1e-12, coords=None, engine: str = "tt"):
    """Two-term shift (four-term for crz), reference autodiff.py:509-550.
    ``coords`` restricts the evaluation to a subset of slots (others left 0)."""
    theta = np.asarray(theta, dtype=float).reshape(-1)

    def e(t):
        if engine == "dense":
            return expval_dense(simulate_dense(circ, t), terms).real
        return evaluate_expval(circ, terms, t, eps).real

    grad = np.zeros(len(theta))
    for k in (range(len(theta)) if coords is None else coords):
        name = circ.gates[circ.trainable[k]][0]

        def sh(d, k=k):
            t = theta.copy()
            t[k] += d
            return e(t)

        if name == "crz":
            grad[k] = _CRZ_A * (sh(np.pi / 2) - sh(-np.pi / 2)) - _CRZ_B * (sh(3 * np.pi / 2) - sh(-3 * np.pi / 2))
        else:
            grad[k] = 0.5 * (sh(np.pi / 2) - sh(-np.pi / 2))
    return grad


def finite_diff_grad(circ: OCircuit, terms, theta, step: float = 1e-5, eps: float = 1e-12):
    """Central differences (reference autodiff.py:553-576)."""
    theta = np.asarray(theta, dtype=float).reshape(-1)
    g = np.zeros(len(theta))
    for k in range(len(theta)):
        up, dn = theta.copy(), theta.copy()
        up[k] += step
        dn[k] -= step
        g[k] = (evaluate_expval(circ, terms, up, eps).real - evaluate_expval(circ, terms, dn, eps).real) / (2 * step)
    return g


# --------------------------------------------------------------------------- MBE MaxCut
def mbe_encode(num_vertices: int):
    """Vertex 2k -> (k, Z), 2k+1 -> (k, X) (reference maxcut.py:127-135)."""
    return (num_vertices + 1) // 2, [(v // 2, "Z" if v % 2 == 0 else "X") for v in range(num_vertices)]


def vertex_expectations(circ: OCircuit, theta, num_vertices: int) -> np.ndarray:
    """Reference maxcut.py:206-216 (eps=0 taped values)."""
    _, mapping = mbe_encode(num_vertices)
    vals = taped_term_values(circ, theta, [((q, l),) for q, l in mapping])
    return vals.real.copy()


def mbe_objective(circ: OCircuit, num_vertices: int, edges, alpha: float = 1.0):
    """fun(theta) -> (loss, grad) through one tape (reference maxcut.py:219-252)."""
    _, mapping = mbe_encode(num_vertices)
    groups = [{q: l} for q, l in mapping]

    def fun(theta):
        theta = np.asarray(theta, dtype=float)
        G = _Graph()
        cores = _taped_state(G, circ, theta, 0.0, None)
        nodes = _taped_terms(G, cores, groups)
        tn = [G.tanh(G.scale(G.real(v), alpha)) for v in nodes]
        acc = None
        for u, v, w in edges:
            e = G.scale(G.mul(tn[u], tn[v]), w)
            acc = e if acc is None else G.add(acc, e)
        if acc is None:
            acc = G.const(np.asarray(0j))
        out = G.real(acc)
        return float(out.val.real), G.backward(out, circ.n_params)

    return fun


def round_cut(x):
    """Sign rounding, 0 -> +1 (reference maxcut.py:148-153)."""
    return tuple(1 if v >= 0 else -1 for v in np.asarray(x, dtype=float).reshape(-1))


def cut_value(edges, assignment) -> float:
    """Reference maxcut.py:156-164."""
    a = list(assignment)
    return float(sum(w * (1 - int(a[u]) * int(a[v])) / 2 for u, v, w in edges))


def pairing_graph(num_vertices: int, degree: int, rng):
    """Random d-regular multigraph-free pairing model (SURVEY.md section 8d cfg3 spec):
    shuffle repeated stubs, pair consecutive entries, retry until simple."""
    while True:
        stubs = np.repeat(np.arange(num_vertices), degree)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        seen = set()
        ok = True
        for u, v in pairs:
            key = (min(u, v), max(u, v))
            if u == v or key in seen:
                ok = False
                break
            seen.add(key)
        if ok:
            return [(int(u), int(v), 1.0) for u, v in pairs]


def adam_minimize(fun, theta0, rate=0.1, max_iters=10, betas=(0.9, 0.999), adam_eps=1e-8, tol=1e-8):
    """Adam branch of reference autodiff.py:614-659; returns (theta_final, values)."""
    theta = np.asarray(theta0, dtype=float).copy()
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    values = []
    for it in range(max_iters + 1):
        val, g = fun(theta)
        values.append(val)
        if float(np.linalg.norm(g)) < tol or it == max_iters:
            break
        b1, b2 = betas
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        mh = m / (1 - b1 ** (it + 1))
        vh = v / (1 - b2 ** (it + 1))
        theta = theta - rate * mh / (np.sqrt(vh) + adam_eps)
    return theta, values
