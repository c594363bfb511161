"""Truncated tensor-train engine: TEBD-style simulation with SVD
truncation by (eps, chi_max), discarded weight and per-term expectation values, batched over
theta-sets on the GPU (``csrc/tq_trunc.cu``, C ABI ``include/tq_trunc.h``).

Semantics follow the reference ``simulate_tt`` / ``apply_gate_tt`` (``tt.py:85-244``):
- gates are applied in circuit order;
- a non-adjacent two-qubit gate becomes the reference's SWAP chain (``tt.py:229-233``), and
  every SWAP is truncated by the same rule;
- each two-site split keeps ``sigma_i / sigma_max > eps`` up to ``chi_max``, renormalises by
  the retained weight, and puts sigma on the thin side;
- the discarded weight accumulates per theta-set.

Gradients through truncated splits follow the reference's straight-through tape
(``autodiff.py:10-13,315-363``): :func:`straight_through` records the taped construction's
constant SVD factors and differentiates the frozen-constant value exactly by batched replays.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from .circuits import Circuit, gate_matrix
from .errors import BondTooLarge, InputError, UnsupportedArity, WireOutOfRange

TGATE_DTYPE = np.dtype([("kind", "<i4"), ("site", "<i4"), ("rot", "<i4"), ("slot", "<i4"),
                        ("flip", "<i4"), ("pad", "<i4", (3,)), ("m", "<f8", (32,))])   # 288 bytes
ROT_CODE = {"rx": 1, "ry": 2, "rz": 3, "crz": 4}
MAX_CHI_TRUNC = 32          # bond capacity of the kernel (shared-memory split of 2chi x 2chi)
_SWAP = gate_matrix("swap")


def _flip4(m: np.ndarray) -> np.ndarray:
    return m.reshape(2, 2, 2, 2).transpose(1, 0, 3, 2).reshape(4, 4)


def compile_gates(circuit: Circuit):
    """Circuit -> (gate table [G] TGATE_DTYPE, python list [(matrix-or-None, sites, rot, slot, flip)]).

    Trainable rotations keep their theta slot (the kernel evaluates the matrix per theta-set);
    everything else is stored as a constant matrix with axes in site order."""
    n = circuit.n_qubits
    slot_of = {g: s for s, g in enumerate(circuit.trainable)}
    rows = []
    for gi, g in enumerate(circuit.gates):
        w = tuple(int(x) for x in g.wires)
        if any(not 0 <= x < n for x in w):
            raise WireOutOfRange(f"gate '{g.name}' wires {w} exceed n={n}")
        slot = slot_of.get(gi, -1)
        rot = ROT_CODE.get(g.name, 0) if slot >= 0 else 0
        mat = np.asarray(g.matrix, dtype=complex)
        if len(w) == 1:
            rows.append((None if rot else mat, (w[0],), rot, slot, 0))
            continue
        if len(w) != 2:
            raise UnsupportedArity(f"TT engine handles 1- and 2-qubit gates, got {len(w)} wires")
        lo, hi = min(w), max(w)
        flip = 1 if w[0] > w[1] else 0
        m4 = None if rot else (_flip4(mat) if flip else mat)
        for j in range(hi - 1, lo, -1):      # bring hi next to lo (reference tt.py:229-231)
            rows.append((_SWAP, (j, j + 1), 0, -1, 0))
        rows.append((m4, (lo, lo + 1), rot, slot, flip if rot else 0))   # constants are pre-flipped
        for j in range(lo + 1, hi):          # and back
            rows.append((_SWAP, (j, j + 1), 0, -1, 0))
    table = np.zeros(len(rows), dtype=TGATE_DTYPE)
    for r, (m, sites, rot, slot, flip) in enumerate(rows):
        table[r]["kind"] = len(sites)
        table[r]["site"] = sites[0]
        table[r]["rot"] = rot
        table[r]["slot"] = slot
        table[r]["flip"] = flip
        if m is not None:
            flat = np.asarray(m, dtype=complex).reshape(-1)
            table[r]["m"][: 2 * flat.size: 2] = flat.real
            table[r]["m"][1: 2 * flat.size: 2] = flat.imag
    return table, rows


def resolved_gates(rows, theta: np.ndarray):
    """[(matrix, sites)] for one theta-set (the mirror's input; the kernel does this on device)."""
    out = []
    for m, sites, rot, slot, flip in rows:
        if m is None:
            name = {1: "rx", 2: "ry", 3: "rz", 4: "crz"}[rot]
            m = gate_matrix(name, float(theta[slot]))
            if flip:
                m = _flip4(m)
        out.append((m, sites))
    return out


def term_table(terms, n: int):
    """Normalised terms -> (lo [T], hi [T], code offsets [T+1], codes [sum window] int8)."""
    code = {"X": 1, "Y": 2, "Z": 3, 1: 1, 2: 2, 3: 3}
    lo = np.zeros(len(terms), np.int32)
    hi = np.full(len(terms), -1, np.int32)
    offs = np.zeros(len(terms) + 1, np.int32)
    codes = []
    for t, (_, ops) in enumerate(terms):
        ops = dict(ops)
        if ops:
            lo[t], hi[t] = min(ops), max(ops)
            codes += [code[ops[k]] if k in ops else 0 for k in range(lo[t], hi[t] + 1)]
        offs[t + 1] = len(codes)
    return lo, hi, offs, np.array(codes if codes else [0], np.int8)


def check_truncation_args(eps: float, chi_max) -> int:
    if eps < 0:
        raise InputError(f"eps must be >= 0, got {eps}")
    if chi_max is not None and int(chi_max) < 1:
        raise InputError(f"chi_max must be >= 1, got {chi_max}")
    # a larger chi_max is accepted; a bond that actually outgrows the capacity raises BondTooLarge
    return MAX_CHI_TRUNC if chi_max is None else min(int(chi_max), MAX_CHI_TRUNC)


class TruncatedResult:
    """Per-theta-set results of one truncated simulation."""

    def __init__(self, values, discarded, bonds, norm2):
        self.values = values          # complex128 [B, T]
        self.discarded = discarded    # float64 [B]
        self.bonds = bonds            # int32 [B, n+1] final bond dimensions
        self.norm2 = norm2            # float64 [B] <psi|psi>

    def energy(self, coeffs) -> np.ndarray:
        """sum_t coeff_t v_t in term order (reference hamiltonians.py:161-164)."""
        out = np.zeros(self.values.shape[0], dtype=complex)
        for t, c in enumerate(coeffs):
            out = out + c * self.values[:, t]
        return out


_GATE_CACHE: dict = {}
_TERM_CACHE: dict = {}
_CACHE_MAX = 8


def _device_gates(circuit: Circuit, dev):
    """Compiled gate table of a (frozen) circuit on ``dev``, cached per circuit object: a
    serving loop that evaluates one circuit at many angle batches compiles and uploads it once."""
    import torch

    key = (id(circuit), str(dev))
    hit = _GATE_CACHE.get(key)
    if hit is not None and hit[0]() is circuit:
        return hit[1], hit[2]
    table, _ = compile_gates(circuit)
    d_gates = torch.from_numpy(np.ascontiguousarray(table.view(np.uint8))).to(dev)
    if len(_GATE_CACHE) >= _CACHE_MAX:
        _GATE_CACHE.pop(next(iter(_GATE_CACHE)))
    _GATE_CACHE[key] = (weakref.ref(circuit), table, d_gates)
    return table, d_gates


def _device_terms(terms, n: int, dev):
    """term_table(terms, n) uploaded to ``dev``, cached on the (hashable) normalised terms."""
    import torch

    key = (tuple(terms), n, str(dev))
    hit = _TERM_CACHE.get(key)
    if hit is not None:
        return hit
    arrs = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in term_table(terms, n))
    if len(_TERM_CACHE) >= _CACHE_MAX:
        _TERM_CACHE.pop(next(iter(_TERM_CACHE)))
    _TERM_CACHE[key] = arrs
    return arrs


def simulate_terms(circuit: Circuit, terms, theta, eps: float = 0.0, chi_max=None, *,
                   dtype: str = "complex128", device=None) -> TruncatedResult:
    """Truncated evolution of every theta-set [B, P] and <P_t> for each normalised term."""
    import torch

    from . import _lib
    from .engine import _stream

    cap = check_truncation_args(eps, chi_max)
    theta = np.atleast_2d(np.asarray(theta, dtype=float))
    if theta.shape[1] != circuit.n_params:
        from .errors import ParamCountMismatch
        raise ParamCountMismatch(f"{theta.shape[1]} parameters supplied, circuit has {circuit.n_params} slots")
    B, n = theta.shape[0], circuit.n_qubits
    from .autodiff import _device

    dev = _device(device)   # EngineUnavailable without a GPU: there is no CPU fallback
    table, d_gates = _device_gates(circuit, dev)
    d_lo, d_hi, d_offs, d_codes = _device_terms(terms, n, dev)
    code = _lib.TQ_C128 if dtype == "complex128" else _lib.TQ_C64
    tdt = torch.float64 if dtype == "complex128" else torch.float32
    lib = _lib.load()
    th = torch.tensor(theta, dtype=tdt, device=dev)
    T = len(terms)
    values = torch.zeros(B, max(T, 1), 2, dtype=torch.float64, device=dev)
    disc = torch.zeros(B, dtype=torch.float64, device=dev)
    norm2 = torch.zeros(B, dtype=torch.float64, device=dev)
    bonds = torch.zeros(B, n + 1, dtype=torch.int32, device=dev)
    flags = torch.zeros(B, dtype=torch.int32, device=dev)
    ws_bytes = lib.tq_tt_workspace_bytes(n, B, cap, code)
    ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device=dev)
    st = lib.tq_tt_simulate(n, d_gates.data_ptr(), len(table), code, B, th.data_ptr(), th.stride(0),
                            ctypes.c_double(eps), cap, -1 if chi_max is None else int(chi_max),
                            d_lo.data_ptr(), d_hi.data_ptr(), d_offs.data_ptr(), d_codes.data_ptr(), T,
                            values.data_ptr(), disc.data_ptr(), norm2.data_ptr(), bonds.data_ptr(), flags.data_ptr(),
                            ws.data_ptr(), ctypes.c_size_t(int(ws_bytes)), _stream())
    _lib.check(st)
    f = flags.cpu().numpy()
    if np.any(f == 2):
        from .errors import NotFinite
        raise NotFinite("truncated engine produced NaN")
    if np.any(f):
        raise BondTooLarge(f"a bond exceeded the truncated engine's capacity chi={cap}; pass chi_max <= {cap}")
    vals = torch.view_as_complex(values).cpu().numpy()[:, :T]
    return TruncatedResult(vals, disc.cpu().numpy(), bonds.cpu().numpy(), norm2.cpu().numpy())


def work_model(circuit: Circuit, terms, chi_max) -> dict:
    """Algorithmic real flops of one truncated simulation (eps = 0, bonds capped by chi_max),
    by replaying the bond-dimension rules on the host:
    - one-site gate: 4 chi_l chi_r complex MACs;
    - centre move (Householder QR of m x n, k = min): (2 m n k - 2/3 k^3) for R plus the same
      for Q, and k n (2 chi') for the fold into the neighbour;
    - two-site gate: merge + gate chi_l chi_r (4 chi_m + 16), and a complex SVD of the
      m x n block costed as a LAPACK R-SVD: 4 (4 M^2 N + 8 M N^2 + 9 N^3) real flops
      (M >= N), the standard count a CPU reference pays;
    - norm environments and term windows: the transfer-step GEMMs.
    One complex MAC = 8 real flops."""
    table, _ = compile_gates(circuit)
    n = circuit.n_qubits
    cap = MAX_CHI_TRUNC if chi_max is None else min(int(chi_max), MAX_CHI_TRUNC)
    dims = [1] * (n + 1)
    center = 0
    cmac = 0.0
    svd = 0.0

    def move_right(c):
        nonlocal cmac
        m, nn = 2 * dims[c], dims[c + 1]
        k = min(m, nn)
        cmac += 2 * (m * nn * k - k ** 3 / 3.0) + k * nn * 2 * dims[c + 2]
        dims[c + 1] = k

    def move_left(c):
        nonlocal cmac
        m, nn = 2 * dims[c + 1], dims[c]
        k = min(m, nn)
        cmac += 2 * (m * nn * k - k ** 3 / 3.0) + 2 * dims[c - 1] * nn * k
        dims[c] = k

    for g in table:
        site = int(g["site"])
        if g["kind"] == 1:
            cmac += 4 * dims[site] * dims[site + 1]
            continue
        while center < site:
            move_right(center)
            center += 1
        while center > site:
            move_left(center)
            center -= 1
        cl, cm, cr = dims[site], dims[site + 1], dims[site + 2]
        cmac += cl * cr * (4 * cm + 16)
        M, N = max(2 * cl, 2 * cr), min(2 * cl, 2 * cr)
        svd += 4.0 * (4 * M * M * N + 8 * M * N * N + 9 * N ** 3)
        dims[site + 1] = min(N, cap)
        center = site + 1 if 2 * cl <= 2 * cr else site
    env = sum(2 * dims[k] ** 2 * dims[k + 1] + 2 * dims[k] * dims[k + 1] ** 2 for k in range(n))
    cmac += 2 * env
    for _, ops in terms:
        ops = dict(ops)
        if ops:
            lo, hi = min(ops), max(ops)
            cmac += sum(2 * dims[k] ** 2 * dims[k + 1] + 2 * dims[k] * dims[k + 1] ** 2 for k in range(lo, hi + 1))
    return {"flops": 8.0 * cmac + svd, "svd_flops": svd, "bonds": dims}


class GPUTrain:
    """Device-resident truncated trains of a theta-set batch: the reference's ``TTState``
    (tt.py:38-76) for B states at once.  ``cores_host(b)`` returns the reference layout
    (chi_l, 2, chi_r) per site."""

    def __init__(self, n, batch, cap, dtype, device):
        import torch

        from . import _lib

        self.n, self.batch, self.cap, self.dtype, self.device = n, batch, cap, dtype, device
        self.code = _lib.TQ_C128 if dtype == "complex128" else _lib.TQ_C64
        lib = _lib.load()
        self.cores = torch.zeros(int(lib.tq_tt_state_bytes(n, batch, cap, self.code)), dtype=torch.uint8, device=device)
        self.bonds = torch.ones(batch, n + 1, dtype=torch.int32, device=device)
        self.centers = torch.zeros(batch, dtype=torch.int32, device=device)
        self.discarded = torch.zeros(batch, dtype=torch.float64, device=device)
        self.flags = torch.zeros(batch, dtype=torch.int32, device=device)

    def _slot(self):
        c = 4
        while c < self.cap:
            c <<= 1
        return 2 * c * c

    @classmethod
    def from_cores(cls, trains, *, dtype: str = "complex128", device=None, cap: int | None = None) -> "GPUTrain":
        """Device trains from reference-layout cores: ``trains`` is one list of (chi_l, 2, chi_r)
        arrays (a reference TTState's ``cores``, tt.py:38-76) or a list of such lists (a batch)."""
        import torch

        from .autodiff import _device

        if trains and isinstance(trains[0], np.ndarray) and np.asarray(trains[0]).ndim == 3:
            trains = [trains]
        trains = [[np.asarray(c, dtype=complex) for c in tr] for tr in trains]
        n = len(trains[0])
        if n < 1 or any(len(tr) != n for tr in trains):
            raise InputError("trains must be non-empty and of equal length")
        chi = 1
        for tr in trains:
            for k, c in enumerate(tr):
                if c.ndim != 3 or c.shape[1] != 2:
                    raise InputError(f"core {k} must have shape (chi_l, 2, chi_r), got {c.shape}")
                if k and tr[k - 1].shape[2] != c.shape[0]:
                    raise InputError(f"bond mismatch between cores {k - 1} and {k}")
                chi = max(chi, c.shape[0], c.shape[2])
            if tr[0].shape[0] != 1 or tr[-1].shape[2] != 1:
                raise InputError("the boundary bonds of a train must be 1")
        cap = max(int(cap or 1), chi)
        if cap > MAX_CHI_TRUNC:
            raise BondTooLarge(f"a train bond of {chi} exceeds the engine's capacity {MAX_CHI_TRUNC}")
        out = cls(n, len(trains), cap, dtype, _device(device))
        cdt = torch.complex128 if dtype == "complex128" else torch.complex64
        slot = out._slot()
        host = np.zeros((len(trains), n, slot), dtype=np.complex128)
        bonds = np.ones((len(trains), n + 1), dtype=np.int32)
        for b, tr in enumerate(trains):
            for k, c in enumerate(tr):
                host[b, k, : c.size] = c.reshape(-1)
                bonds[b, k], bonds[b, k + 1] = c.shape[0], c.shape[2]
        out.cores.view(cdt).copy_(torch.from_numpy(host.reshape(-1)).to(cdt))
        out.bonds.copy_(torch.from_numpy(bonds))
        return out

    def row(self, b: int) -> "GPUTrain":
        """Train b alone (a copy with batch 1)."""
        out = GPUTrain.__new__(GPUTrain)
        out.__dict__.update(self.__dict__)
        nbytes = self.cores.numel() // self.batch
        out.batch = 1
        out.cores = self.cores[b * nbytes:(b + 1) * nbytes].clone()
        out.bonds = self.bonds[b:b + 1].clone()
        out.centers = self.centers[b:b + 1].clone()
        out.discarded = self.discarded[b:b + 1].clone()
        out.flags = self.flags[b:b + 1].clone()
        return out

    def clone(self) -> "GPUTrain":
        out = GPUTrain.__new__(GPUTrain)
        out.__dict__.update(self.__dict__)
        for k in ("cores", "bonds", "centers", "discarded", "flags"):
            setattr(out, k, getattr(self, k).clone())
        return out

    def check(self):
        f = self.flags.cpu().numpy()
        if np.any(f == 2):
            from .errors import NotFinite
            raise NotFinite("truncated engine produced NaN")
        if np.any(f):
            raise BondTooLarge(f"a bond exceeded the truncated engine's capacity chi={self.cap}")
        return self

    @property
    def bond_dims(self) -> np.ndarray:
        return self.bonds.cpu().numpy()

    def cores_host(self, b: int = 0) -> list:
        """Cores of train b as numpy arrays (chi_l, 2, chi_r), the reference layout."""
        import torch

        cdt = torch.complex128 if self.dtype == "complex128" else torch.complex64
        flat = self.cores.view(cdt).view(self.batch, self.n, self._slot())[b].cpu().numpy()
        dims = self.bond_dims[b]
        return [flat[k, : dims[k] * 2 * dims[k + 1]].reshape(dims[k], 2, dims[k + 1]).astype(complex)
                for k in range(self.n)]

    def term_values(self, terms):
        """<P_t> per normalised term for every train: (complex [B, T], <psi|psi> [B])."""
        import torch

        from . import _lib
        from .engine import _stream

        lo, hi, offs, codes = term_table(terms, self.n)
        dev = self.device

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        T = len(terms)
        values = torch.zeros(self.batch, max(T, 1), 2, dtype=torch.float64, device=dev)
        norm2 = torch.zeros(self.batch, dtype=torch.float64, device=dev)
        lib = _lib.load()
        wsb = int(lib.tq_tt_values_workspace_bytes(self.n, self.batch, self.cap, self.code))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        d_lo, d_hi, d_offs, d_codes = up(lo), up(hi), up(offs), up(codes)
        _lib.check(lib.tq_tt_values(self.n, self.code, self.batch, self.cap, self.cores.data_ptr(),
                                    self.bonds.data_ptr(), d_lo.data_ptr(), d_hi.data_ptr(), d_offs.data_ptr(),
                                    d_codes.data_ptr(), T, values.data_ptr(), norm2.data_ptr(), ws.data_ptr(),
                                    ctypes.c_size_t(wsb), _stream()))
        return torch.view_as_complex(values).cpu().numpy()[:, :T], norm2.cpu().numpy()


def simulate_train(circuit: Circuit, theta, eps: float = 0.0, chi_max=None, *, dtype: str = "complex128",
                   device=None) -> GPUTrain:
    """Truncated evolution of every theta-set [B, P] into device trains (reference simulate_tt)."""
    import torch

    from . import _lib
    from .autodiff import _device
    from .engine import _stream

    cap = check_truncation_args(eps, chi_max)
    theta = np.atleast_2d(np.asarray(theta, dtype=float))
    if theta.shape[1] != circuit.n_params:
        from .errors import ParamCountMismatch
        raise ParamCountMismatch(f"{theta.shape[1]} parameters supplied, circuit has {circuit.n_params} slots")
    dev = _device(device)
    train = GPUTrain(circuit.n_qubits, theta.shape[0], cap, dtype, dev)
    table, d_gates = _device_gates(circuit, dev)
    th = torch.tensor(theta, dtype=torch.float64 if dtype == "complex128" else torch.float32, device=dev)
    lib = _lib.load()
    _lib.check(lib.tq_tt_run(circuit.n_qubits, d_gates.data_ptr(), len(table), train.code, train.batch,
                             th.data_ptr(), th.stride(0), ctypes.c_double(eps), cap,
                             -1 if chi_max is None else int(chi_max), train.cores.data_ptr(), train.bonds.data_ptr(),
                             train.centers.data_ptr(), train.discarded.data_ptr(), train.flags.data_ptr(), _stream()))
    return train.check()


def apply_circuit(train: GPUTrain, circuit: Circuit, theta, eps: float = 0.0, chi_max=None) -> GPUTrain:
    """Run ``circuit`` on trains the caller already holds (the reference's apply_gate_tt over every
    gate, tt.py:186-234): a new train per row; the discarded weight accumulates onto the input's.
    theta [B, P] (or [P] for every row)."""
    import torch

    from . import _lib
    from .engine import _stream

    if circuit.n_qubits != train.n:
        from .errors import SizeMismatch
        raise SizeMismatch(f"circuit on {circuit.n_qubits} qubits, train on {train.n}")
    check_truncation_args(eps, chi_max)
    theta = np.atleast_2d(np.asarray(theta, dtype=float))
    if theta.shape[1] != circuit.n_params:
        from .errors import ParamCountMismatch
        raise ParamCountMismatch(f"{theta.shape[1]} parameters supplied, circuit has {circuit.n_params} slots")
    if theta.shape[0] == 1 and train.batch > 1:
        theta = np.repeat(theta, train.batch, axis=0)
    cap = MAX_CHI_TRUNC if chi_max is None else max(int(chi_max), train.cap)
    if cap > train.cap:   # room for the bonds the circuit grows (re-laid at the larger slot)
        out = GPUTrain.from_cores([train.cores_host(r) for r in range(train.batch)], dtype=train.dtype,
                                  device=train.device, cap=cap)
        out.centers.copy_(train.centers)
        out.discarded.copy_(train.discarded)
    else:
        out = train.clone()
    table, d_gates = _device_gates(circuit, out.device)
    th = torch.tensor(theta, dtype=torch.float64 if out.dtype == "complex128" else torch.float32, device=out.device)
    _lib.check(_lib.load().tq_tt_apply(out.n, d_gates.data_ptr(), len(table), out.code, out.batch, th.data_ptr(),
                                       th.stride(0), ctypes.c_double(eps), out.cap,
                                       -1 if chi_max is None else int(chi_max), out.cores.data_ptr(),
                                       out.bonds.data_ptr(), out.centers.data_ptr(), out.discarded.data_ptr(),
                                       out.flags.data_ptr(), _stream()))
    return out.check()


def tt_inner(a: GPUTrain, b: GPUTrain) -> np.ndarray:
    """<a_r|b_r> for every row of two train batches (reference tt_inner, tt.py:247-255), complex [B]."""
    import torch

    from . import _lib
    from .engine import _stream

    if a.n != b.n:
        from .errors import SizeMismatch
        raise SizeMismatch(f"{a.n} vs {b.n} qubits")
    if a.batch != b.batch or a.dtype != b.dtype:
        raise InputError("inner product needs trains of equal batch and dtype")
    if a._slot() != b._slot():   # one slot layout for both (re-laid at the larger capacity)
        cap = max(a.cap, b.cap)
        a = GPUTrain.from_cores([a.cores_host(r) for r in range(a.batch)], dtype=a.dtype, device=a.device, cap=cap)
        b = GPUTrain.from_cores([b.cores_host(r) for r in range(b.batch)], dtype=b.dtype, device=b.device, cap=cap)
    out = torch.zeros(a.batch, 2, dtype=torch.float64, device=a.device)
    _lib.check(_lib.load().tq_tt_inner(a.n, a.code, a.batch, a.cap, a.cores.data_ptr(), a.bonds.data_ptr(),
                                       b.cores.data_ptr(), b.bonds.data_ptr(), out.data_ptr(), _stream()))
    return torch.view_as_complex(out).cpu().numpy()


def compress(train: GPUTrain, eps: float, chi_max=None) -> GPUTrain:
    """Re-truncate every bond of every train (reference compress, tt.py:299-320): a new train;
    the discarded weight accumulates onto the input's."""
    from . import _lib
    from .engine import _stream

    check_truncation_args(eps, chi_max)
    out = train.clone()
    out.flags.zero_()
    lib = _lib.load()
    _lib.check(lib.tq_tt_compress(out.n, out.code, out.batch, ctypes.c_double(eps), out.cap,
                                  -1 if chi_max is None else int(chi_max), out.cores.data_ptr(), out.bonds.data_ptr(),
                                  out.centers.data_ptr(), out.discarded.data_ptr(), out.flags.data_ptr(), _stream()))
    return out.check()


# ----------------------------------------------------------------------------- straight-through gradient
def _check_flags(flags, cap):
    f = flags.cpu().numpy()
    if np.any(f == 2):
        from .errors import NotFinite
        raise NotFinite("truncated engine produced NaN")
    if np.any(f):
        raise BondTooLarge(f"a bond exceeded the truncated engine's capacity chi={cap}; pass chi_max <= {cap}")


def straight_through(circuit: Circuit, terms, theta, eps: float = 0.0, chi_max=None, *, dtype: str = "complex128",
                     device=None, want_grad: bool = True, rows_per_launch: int | None = None,
                     init: "GPUTrain | None" = None, weights=None):
    """The reference's gradient through truncated splits (``grad_expval`` with eps > 0 or a binding
    chi_max, autodiff.py:315-363,471-487): value and straight-through gradient for every theta-set.

    1. ``tq_tt_taped`` builds the TAPED state of each theta-set (no centre moves; every two-site
       split keeps U_k, or Vh_k, as a constant and the other factor as the differentiable
       projection) and records those constants;
    2. ``tq_tt_replay`` re-runs the construction for every shifted angle set with the constants of
       its theta-set frozen.  Frozen, each gate enters linearly and each angle as
       c + a cos(t/2) + b sin(t/2), so the reference's reverse-mode result equals the exact shift
       rule on the replayed values: (E(t + pi/2) - E(t - pi/2)) / 2, and crz's four-term rule
       (autodiff.py:509-550).  Shifted rows are batched over the SMs, one CTA per row.

    ``init``: an input train (batch 1, shared by every theta-set) instead of |0...0>.  With eps = 0
    and no binding chi_max every split keeps a square unitary factor, so the result is the EXACT
    gradient of <init|U^H H U|init> (the differentiable path for arbitrary input trains).
    ``weights``: callable(values [B, T]) -> [B, T] cotangent weights w; the gradient is then that
    of Re sum_t w_t v_t with w frozen at the unshifted values (the chain rule through a function
    of the readouts, e.g. the MBE loss).  Default: the terms' coefficients (the energy).

    Returns (values [B, T] complex128 of the taped state, grad [B, P] float64)."""
    import torch

    from . import _lib
    from .autodiff import _CRZ_Y1, _CRZ_Y2, _device
    from .engine import _stream

    cap = check_truncation_args(eps, chi_max)
    theta = np.atleast_2d(np.asarray(theta, dtype=float))
    if theta.shape[1] != circuit.n_params:
        from .errors import ParamCountMismatch
        raise ParamCountMismatch(f"{theta.shape[1]} parameters supplied, circuit has {circuit.n_params} slots")
    B, n, P = theta.shape[0], circuit.n_qubits, circuit.n_params
    dev = _device(device)
    table, d_gates = _device_gates(circuit, dev)
    n2 = int(np.sum(table["kind"] == 2))
    d_lo, d_hi, d_offs, d_codes = _device_terms(terms, n, dev)
    code = _lib.TQ_C128 if dtype == "complex128" else _lib.TQ_C64
    tdt = torch.float64 if dtype == "complex128" else torch.float32
    lib = _lib.load()
    T = len(terms)
    coef = np.array([c for c, _ in terms], dtype=complex)
    if init is not None:
        if init.n != n or init.dtype != dtype:
            raise InputError("the input train must match the circuit width and dtype")
        cap = max(cap, init.cap) if chi_max is None else cap
        if init._slot() != 2 * (1 << max(2, (cap - 1).bit_length())) ** 2 or init.batch != 1:
            init = GPUTrain.from_cores(init.cores_host(0), dtype=dtype, device=dev, cap=cap)
        init_ptrs = (init.cores.data_ptr(), init.bonds.data_ptr())
    else:
        init_ptrs = (None, None)
    tape = torch.empty(int(lib.tq_tt_tape_bytes(n2, B, cap, code)), dtype=torch.uint8, device=dev)

    def run(rows_theta, parent=None):
        R_ = rows_theta.shape[0]
        th = torch.tensor(rows_theta, dtype=tdt, device=dev)
        values = torch.zeros(R_, max(T, 1), 2, dtype=torch.float64, device=dev)
        norm2 = torch.zeros(R_, dtype=torch.float64, device=dev)
        bonds = torch.zeros(R_, n + 1, dtype=torch.int32, device=dev)
        flags = torch.zeros(R_, dtype=torch.int32, device=dev)
        wsb = int(lib.tq_tt_workspace_bytes(n, R_, cap, code))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        if parent is None:
            st = lib.tq_tt_taped(n, d_gates.data_ptr(), len(table), n2, code, R_, th.data_ptr(), th.stride(0),
                                 ctypes.c_double(eps), cap, -1 if chi_max is None else int(chi_max),
                                 d_lo.data_ptr(), d_hi.data_ptr(), d_offs.data_ptr(), d_codes.data_ptr(), T,
                                 values.data_ptr(), norm2.data_ptr(), bonds.data_ptr(), flags.data_ptr(),
                                 tape.data_ptr(), *init_ptrs, ws.data_ptr(), ctypes.c_size_t(wsb), _stream())
        else:
            par = torch.tensor(parent, dtype=torch.int32, device=dev)
            st = lib.tq_tt_replay(n, d_gates.data_ptr(), len(table), n2, code, R_, th.data_ptr(), th.stride(0), cap,
                                  par.data_ptr(), B, tape.data_ptr(), d_lo.data_ptr(), d_hi.data_ptr(),
                                  d_offs.data_ptr(), d_codes.data_ptr(), T, values.data_ptr(), norm2.data_ptr(),
                                  bonds.data_ptr(), flags.data_ptr(), *init_ptrs, ws.data_ptr(), ctypes.c_size_t(wsb),
                                  _stream())
        _lib.check(st)
        _check_flags(flags, cap)
        return torch.view_as_complex(values).cpu().numpy()[:, :T]

    vals = run(theta)
    if not want_grad:
        return vals, None
    W = np.broadcast_to(coef[None, :], vals.shape) if weights is None else np.asarray(weights(vals))
    names = [circuit.gates[g].name for g in circuit.trainable]
    rows, plan = [], []
    for b in range(B):
        for k in range(P):
            shifts = (np.pi / 2, -np.pi / 2, 3 * np.pi / 2, -3 * np.pi / 2) if names[k] == "crz" else (np.pi / 2, -np.pi / 2)
            idx = []
            for d in shifts:
                t = theta[b].copy()
                t[k] += d
                idx.append(len(rows))
                rows.append((b, t))
            plan.append((b, k, idx))
    grad = np.zeros((B, P))
    if not rows:
        return vals, grad
    if rows_per_launch is None:
        # one full wave per launch: four 128-thread CTAs resident per SM (csrc/tq_trunc.cu NT),
        # within a 16 GB workspace budget (HBM is 180 GB; a row at n=500, cap 16 takes ~8 MB)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        per_row = int(lib.tq_tt_workspace_bytes(n, 1, cap, code))
        rows_per_launch = int(max(sms, min(6 * sms, (16 << 30) // max(per_row, 1))))
    e = np.zeros(len(rows))
    for c0 in range(0, len(rows), rows_per_launch):
        chunk = rows[c0:c0 + rows_per_launch]
        v = run(np.stack([t for _, t in chunk]), [b for b, _ in chunk])
        par = np.array([b for b, _ in chunk])
        e[c0:c0 + len(chunk)] = np.einsum("rt,rt->r", v, W[par]).real
    for b, k, idx in plan:
        if names[k] == "crz":
            grad[b, k] = _CRZ_Y1 * (e[idx[0]] - e[idx[1]]) - _CRZ_Y2 * (e[idx[2]] - e[idx[3]])
        else:
            grad[b, k] = 0.5 * (e[idx[0]] - e[idx[1]])
    return vals, grad
