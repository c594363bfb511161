"""Chain compiler: circuit + Pauli operator -> the flat tables the sm_100a kernels sweep.

What it replaces.  The reference simulates gate by gate with SVD/QR re-factoring
(``tt.py:186-244``) and evaluates terms with per-term windows
(``hamiltonians.py:129-164``, taped ``autodiff.py:339-402``).  Here nothing is
re-factorised.  Every two-qubit gate is split once on the host into its operator
Schmidt form ``G = sum_a F0_a (x) F1_a`` (CZ = sum_a |a><a| (x) Z^a,
CNOT = sum_a |a><a| (x) X^a, generic gates by SVD); the digit ``a`` becomes a bond
leg across every cut the gate spans.  The MPS core of site k is then
``A_k[s]_{alpha,beta} = <s| O_L ... O_1 |init_k>``: the column of 2x2 operators
acting on qubit k, where digit-carrying ops select their factor by the digit of
alpha (gate whose right end is k) or beta (left end is k).  Bond dimensions are
exactly ``chi_c = 2^(bits crossing cut c)`` and depend only on the gate
sequence, like the reference's eps=0 mode (``tt.py:9-12``).

The Pauli sum becomes a finite-automaton MPO with channels START / DONE /
one in-flight channel per open multi-site term; the kernels sweep its transfer
environments (right-to-left for the energy, left-to-right for the gradient).

Light cone.  ``<P>`` only depends on gates in P's backward light cone, so the
chain is split into segments that own contiguous term ranges; each segment runs
on the sub-chain spanned by its owned terms' cone (all gates fully inside that
interval), exactly, with trivial boundaries.  Segments are independent CTAs.

Every table below is a numpy structured array whose layout is the C struct of
the same name in ``include/tq_engine.h``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import BondTooLarge, InputError, UnsupportedArity, WireOutOfRange
from .hamiltonians import PAULI_CODE

# ----------------------------------------------------------------------------- C layouts
SITE_DTYPE = np.dtype([
    ("op_begin", "<i4"), ("op_count", "<i4"), ("lmat_count", "<i4"), ("chi_l", "<i4"), ("chi_r", "<i4"),
    ("pass_begin", "<i4"), ("pass_count", "<i4"),
    ("rl_edge_begin", "<i4"), ("rl_edge_count", "<i4"), ("lr_edge_begin", "<i4"), ("lr_edge_count", "<i4"),
    ("fin_begin", "<i4"), ("fin_count", "<i4"),
    ("rl_da", "<i4"), ("rl_db", "<i4"), ("lr_da", "<i4"), ("lr_db", "<i4"),
    ("n_train", "<i4"), ("ent_begin", "<i4"),
    ("env_in", "<i8"), ("env_out", "<i8"),
    ("init", "<f8", (4,)),
    ("a_off", "<i8"), ("g_off", "<i8"),
], align=True)
OP_DTYPE = np.dtype([("mat", "<i4"), ("lmat", "<i4"), ("src", "<i4"), ("shift", "<i4"), ("bits", "<i4"),
                     ("tidx", "<i4"), ("gidx", "<i4"), ("toff", "<i4"), ("tbase", "<i4"), ("pad", "<i4")],
                    align=True)
MAT_DTYPE = np.dtype([("kind", "<i4"), ("slot", "<i4"), ("cls", "<i4"), ("pad", "<i4"),
                      ("angle", "<f8"), ("pscale", "<f8"), ("m", "<f8", (8,))], align=True)
EDGE_DTYPE = np.dtype([("a", "<i4"), ("b", "<i4"), ("op", "<i4"), ("coef", "<i4")], align=True)
PASS_DTYPE = np.dtype([("sa", "<i4"), ("sb", "<i4"), ("bits", "<i4"), ("pad", "<i4")], align=True)
SEG_DTYPE = np.dtype([("site_begin", "<i4"), ("site_count", "<i4"), ("gslot_begin", "<i4"), ("gslot_count", "<i4"),
                      ("lo", "<i4"), ("hi", "<i4"), ("env_base", "<i8"), ("env_elems", "<i8")], align=True)

SRC_NONE, SRC_ALPHA, SRC_BETA = 0, 1, 2
KIND_CONST, KIND_RX, KIND_RY, KIND_RZ = 0, 1, 2, 3
CLS_UNITARY, CLS_PROJ0, CLS_PROJ1, CLS_GENERAL = 0, 1, 2, 3
ROT_KIND = {"rx": KIND_RX, "ry": KIND_RY, "rz": KIND_RZ}
MAX_CHI = 32            # complex64 kernels
MAX_CHI_F64 = 16        # complex128 parity kernels
MAX_OPS = 64            # ops per column
MAX_TRAIN = 32          # trainable ops per column

_I2 = np.eye(2, dtype=complex)
_P0 = np.array([[1, 0], [0, 0]], dtype=complex)
_P1 = np.array([[0, 0], [0, 1]], dtype=complex)
_SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)


# ----------------------------------------------------------------------------- factor specs
@dataclass(frozen=True)
class MatSpec:
    """One 2x2 factor: a constant matrix or a rotation exp(-i t sigma/2) on a theta slot."""

    kind: int
    slot: int = -1
    const: tuple | None = None  # flattened complex 2x2 for KIND_CONST

    @staticmethod
    def of(matrix) -> "MatSpec":
        m = np.asarray(matrix, dtype=complex).reshape(2, 2)
        return MatSpec(KIND_CONST, -1, tuple(m.reshape(-1).tolist()))

    def matrix(self) -> np.ndarray:
        return np.array(self.const, dtype=complex).reshape(2, 2)


@dataclass
class TimeGate:
    """A gate in time order, already split into per-site factor lists."""

    lo: int
    hi: int
    bits: int                   # digit width carried across lo+1..hi (0 for 1q / product gates)
    fac_lo: list                # MatSpec per digit value on site lo
    fac_hi: list                # MatSpec per digit value on site hi (empty for 1q)


def _classify(m: np.ndarray):
    """(cls, pscale) of a constant 2x2 factor (kernel needs it to rebuild forward vectors)."""
    if np.max(np.abs(m.conj().T @ m - np.eye(2))) < 1e-12:
        return CLS_UNITARY, 1.0
    for cls, a in ((CLS_PROJ0, 0), (CLS_PROJ1, 1)):
        s = m[a, a]
        other = m.copy()
        other[a, a] = 0
        if np.max(np.abs(other)) < 1e-14 and abs(s) > 1e-12 and abs(s.imag) < 1e-15:
            return cls, float(s.real)
    return CLS_GENERAL, 1.0


def split_two_qubit(matrix: np.ndarray):
    """Operator-Schmidt split of a 4x4 gate in (w0, w1) order -> (bits, F0 list, F1 list).

    Controlled structure is detected first so CZ/CNOT get the exact |a><a| (x) U_a
    factors (projectors on the control, unitaries on the target); everything else
    goes through an SVD of the reshuffled matrix."""
    m = np.asarray(matrix, dtype=complex).reshape(4, 4)
    for swapped in (False, True):
        mm = _SWAP @ m @ _SWAP if swapped else m
        if np.max(np.abs(mm[0:2, 2:4])) < 1e-14 and np.max(np.abs(mm[2:4, 0:2])) < 1e-14:
            u0, u1 = mm[0:2, 0:2], mm[2:4, 2:4]
            if np.max(np.abs(u0 - u1)) < 1e-14:
                ctrl, targ = [_I2], [u0]
                bits = 0
            else:
                ctrl, targ = [_P0, _P1], [u0, u1]
                bits = 1
            return (bits, targ, ctrl) if swapped else (bits, ctrl, targ)
    r = m.reshape(2, 2, 2, 2).transpose(0, 2, 1, 3).reshape(4, 4)
    u, s, vh = np.linalg.svd(r)
    rank = int(np.count_nonzero(s > 1e-12 * s[0]))
    f0 = [math.sqrt(s[a]) * u[:, a].reshape(2, 2) for a in range(rank)]
    f1 = [math.sqrt(s[a]) * vh[a, :].reshape(2, 2) for a in range(rank)]
    if rank == 1:
        return 0, f0, f1
    bits = 1 if rank <= 2 else 2
    while len(f0) < (1 << bits):
        f0.append(np.zeros((2, 2), dtype=complex))
        f1.append(np.zeros((2, 2), dtype=complex))
    return bits, f0, f1


def gate_array(g) -> np.ndarray:
    """A gate's matrix as ndarray (this package's Gate or tnsim's DenseTensor-backed Gate)."""
    m = g.matrix
    return np.asarray(m.array if hasattr(m, "array") else m, dtype=complex)


def structure_key(circuit):
    """Hashable key of everything but trainable angle values (plan cache key); works for
    this package's Circuit and for reference tnsim.Circuit objects."""
    if hasattr(circuit, "structure_key"):
        return circuit.structure_key()
    tr = set(circuit.trainable)
    parts = tuple((g.name, tuple(g.wires), "T" if i in tr else gate_array(g).tobytes())
                  for i, g in enumerate(circuit.gates))
    return (circuit.n_qubits, parts, tuple(circuit.trainable))


def time_gates(circuit) -> list:
    """Circuit (reference-compatible object) -> list[TimeGate] in gate order."""
    slot_of = {gi: s for s, gi in enumerate(circuit.trainable)}
    out = []
    n = circuit.n_qubits
    for gi, g in enumerate(circuit.gates):
        wires = tuple(int(w) for w in g.wires)
        if any(not 0 <= w < n for w in wires):
            raise WireOutOfRange(f"gate '{g.name}' wires {wires} exceed n={n}")
        trainable = gi in slot_of
        if len(wires) == 1:
            if trainable:
                if g.name not in ROT_KIND:
                    raise InputError(f"trainable gate '{g.name}' is not a rotation")
                spec = MatSpec(ROT_KIND[g.name], slot_of[gi])
            else:
                spec = MatSpec.of(gate_array(g))
            out.append(TimeGate(wires[0], wires[0], 0, [spec], []))
            continue
        if len(wires) != 2:
            raise UnsupportedArity(f"TT engine handles 1- and 2-qubit gates, got {len(wires)} wires")
        w0, w1 = wires
        if trainable:
            if g.name != "crz":
                raise InputError(f"trainable gate '{g.name}' has no factored form")
            bits, f0 = 1, [MatSpec.of(_P0), MatSpec.of(_P1)]
            f1 = [MatSpec.of(_I2), MatSpec(KIND_RZ, slot_of[gi])]
        else:
            bits, m0, m1 = split_two_qubit(gate_array(g))
            f0 = [MatSpec.of(x) for x in m0]
            f1 = [MatSpec.of(x) for x in m1]
        if bits == 0:  # product gate: two single-site factors
            out.append(TimeGate(w0, w0, 0, [f0[0]], []))
            out.append(TimeGate(w1, w1, 0, [f1[0]], []))
            continue
        if w0 < w1:
            out.append(TimeGate(w0, w1, bits, f0, f1))
        else:
            out.append(TimeGate(w1, w0, bits, f1, f0))
    return out


# ----------------------------------------------------------------------------- operator
def normalize_terms(ham):
    """PauliHamiltonian-like -> list of (coeff complex, tuple((q, code)))."""
    terms = []
    for t in ham.terms:
        ops = tuple((int(q), PAULI_CODE[l]) for q, l in sorted(t.ops))
        terms.append((complex(t.coeff), ops))
    return terms


# ----------------------------------------------------------------------------- segments
def light_cone(tgates, lo, hi):
    """Interval hull of the backward light cone of sites [lo, hi] (exact for the
    engine: every gate touching the hull is absorbed, reference-free)."""
    for g in reversed(tgates):
        if g.bits and g.lo <= hi and g.hi >= lo:
            lo, hi = min(lo, g.lo), max(hi, g.hi)
    return lo, hi


def _cones_vectorized(tgates, los, his):
    los = np.array(los, dtype=np.int64)
    his = np.array(his, dtype=np.int64)
    two = [(g.lo, g.hi) for g in tgates if g.bits]
    for glo, ghi in reversed(two):
        m = (glo <= his) & (ghi >= los)
        if m.any():
            los = np.where(m, np.minimum(los, glo), los)
            his = np.where(m, np.maximum(his, ghi), his)
    return los, his


def factored_chi(n, tgates) -> int:
    """Largest factored bond 2^(bits crossing a cut) of the whole chain."""
    bits = np.zeros(n + 1, dtype=np.int64)
    for g in tgates:
        if g.bits:
            bits[g.lo + 1: g.hi + 1] += g.bits
    return int(1 << int(bits.max())) if n else 1


def resident_teams(chi: int, d: int = 3) -> int:
    """Work items resident per SM, from the kernels' shared-memory layout (lr sweep,
    complex64): 4 + 4D matrix slots of (chi+1)^2 complex for the fused small-chi path,
    2 + 6D otherwise, plus descriptors.  Warp teams (chi <= 8) come 4 per CTA; chi 16/32
    teams are whole CTAs."""
    b = 2
    while b < chi:
        b <<= 1
    slots = 2 + 3 * d if b <= 8 else 2 + 6 * d      # fused small-chi (direct-G) layout vs unfused (gradient sweep)
    team_bytes = slots * (b + 1) ** 2 * 8 + 4096
    smem = 227 * 1024
    if b <= 8:
        # 128-thread CTAs; the gradient kernel needs ~128 registers/thread -> at most 4 CTAs/SM
        # (a 5-CTA register cap was measured slower: more segments add light-cone halo work)
        ctas = max(1, min(smem // (4 * team_bytes), 4))
        return int(ctas * 4)
    return int(max(1, min(smem // team_bytes, 2048 // (128 if b == 16 else 256))))


def choose_segments(n, terms, tgates, batch, n_sm=148, requested=None):
    """Segments per theta-set.  Minimises waves x sites-per-item, where a segment
    costs its owned sites plus the light-cone halo, and a wave is one resident item
    per team slot on every SM."""
    if requested is not None:
        return max(1, int(requested))
    firsts = sorted({ops[0][0] for _, ops in terms if ops})
    if not firsts:
        return 1
    mid = firsts[len(firsts) // 2]
    clo, chi_ = light_cone(tgates, mid, mid + 1 if mid + 1 < n else mid)
    width = max(1, chi_ - clo + 1)
    chi = factored_chi(n, tgates)
    res = resident_teams(min(chi, 32))
    slots = n_sm * res
    nf = len(firsts)
    best, best_cost = 1, None
    for S in range(1, min(nf, 1024) + 1):
        waves = math.ceil(batch * S / slots)
        cost = waves * (nf / S + width)
        if best_cost is None or cost < best_cost - 1e-9:
            best, best_cost = S, cost
    return best


# ----------------------------------------------------------------------------- plan
@dataclass
class ChainPlan:
    n: int
    n_params: int
    n_terms: int
    mode: str
    sites: np.ndarray
    ops: np.ndarray
    mats: np.ndarray
    edges: np.ndarray
    fins: np.ndarray
    passes: np.ndarray
    segs: np.ndarray
    gred_ptr: np.ndarray
    gred_idx: np.ndarray
    chi_max: int
    d_max: int
    max_edges: int
    max_tree: int
    max_ttree: int        # largest sum of trainable-op tree levels of any column (compact adjoint tree)
    max_ops: int
    max_lmat: int
    max_train: int
    n_gslots: int
    env_total: int
    e_const: complex
    term_active: np.ndarray
    info: dict = field(default_factory=dict)

    @property
    def n_segments(self) -> int:
        return len(self.segs)


def _segment_ranges(n_terms_first, n_seg):
    """Split the sorted distinct first-sites into n_seg contiguous groups."""
    firsts = np.array(n_terms_first)
    groups = np.array_split(firsts, n_seg)
    return [(int(g[0]), int(g[-1])) for g in groups if len(g)]


def compile_chain(circuit, ham_terms, mode="energy", batch=1, segments=None, init=None,
                  chi_limit=MAX_CHI, n_sm=148) -> ChainPlan:
    """Compile (circuit, normalized terms) into a ChainPlan.

    mode="energy": MPO with coefficient indices (per-theta-set coefficients supported).
    mode="values": per-term values (windows finalised against the right environment).
    ``init``: optional per-qubit complex 2-vectors of the input product state (default |0>)."""
    n = int(circuit.n_qubits)
    tg = time_gates(circuit)
    T = len(ham_terms)
    e_const = sum((c for c, ops in ham_terms if not ops), 0j)
    active = np.array([1 if ops else 0 for _, ops in ham_terms], dtype=np.int32)
    for _, ops in ham_terms:
        for q, _ in ops:
            if not 0 <= q < n:
                raise WireOutOfRange(f"term acts on qubit {q} but n_qubits={n}")
    if mode == "state":   # the whole chain, no operator (inner products)
        owned, clos, chis = [[]], np.array([0]), np.array([n - 1])
    else:
        S = choose_segments(n, ham_terms, tg, batch, n_sm, segments)
        firsts = sorted({ops[0][0] for _, ops in ham_terms if ops})
        ranges = _segment_ranges(firsts, min(S, max(1, len(firsts)))) if firsts else []
        # owned terms per range
        owned = [[] for _ in ranges]
        starts = [r[0] for r in ranges]
        for t, (_, ops) in enumerate(ham_terms):
            if not ops:
                continue
            f = ops[0][0]
            gi = int(np.searchsorted(starts, f, side="right") - 1)
            owned[gi].append(t)
        los = [min(ham_terms[t][1][0][0] for t in ow) for ow in owned]
        his = [max(ham_terms[t][1][-1][0] for t in ow) for ow in owned]
        clos, chis = _cones_vectorized(tg, los, his)

    sites, ops, mats, edges, fins, passes, segs = [], [], [], [], [], [], []
    mat_index = {}
    gred = {}  # theta slot -> list of absolute partial indices
    chi_max, d_max, max_ops, max_lmat, max_train, max_tree, max_ttree = 1, 1, 0, 1, 0, 1, 1
    env_total = 0
    gslot_total = 0
    init_vecs = None if init is None else np.asarray(init, dtype=complex).reshape(n, 2)

    def make_rec(spec: MatSpec):
        rec = np.zeros((), dtype=MAT_DTYPE)
        rec["kind"], rec["slot"] = spec.kind, spec.slot
        if spec.kind == KIND_CONST:
            m = spec.matrix()
            cls, ps = _classify(m)
            rec["cls"], rec["pscale"] = cls, ps
            rec["m"] = np.stack([m.reshape(-1).real, m.reshape(-1).imag], axis=1).reshape(-1)
        else:
            rec["cls"], rec["pscale"] = CLS_UNITARY, 1.0
        return rec

    def mat_block(specs):
        """Table entries for one op (entry = base + digit), appended in op order so every
        site's entries are contiguous (the kernel resolves entry e of a site at ent_begin + e)."""
        base = len(mats)
        for spec in specs:
            key = (spec.kind, spec.slot, spec.const)
            if key not in mat_index:
                mat_index[key] = make_rec(spec)
            mats.append(mat_index[key])
        return base

    for gi_seg, (ow, c_lo, c_hi) in enumerate(zip(owned, clos.tolist(), chis.tolist())):
        # ---- columns of the sub-chain [c_lo, c_hi]
        nsite = c_hi - c_lo + 1
        cut_bits = np.zeros(nsite + 1, dtype=np.int64)   # local cut c = left of local site c
        col = [[] for _ in range(nsite)]                 # (src, shift, bits, [MatSpec])
        pas = [[] for _ in range(nsite)]
        for g in tg:
            if g.lo < c_lo or g.hi > c_hi:
                continue
            if g.bits == 0:
                col[g.lo - c_lo].append((SRC_NONE, 0, 0, g.fac_lo))
                continue
            a, b = g.lo - c_lo, g.hi - c_lo
            shifts = {}
            for c in range(a + 1, b + 1):
                shifts[c] = int(cut_bits[c])
                cut_bits[c] += g.bits
            col[a].append((SRC_BETA, shifts[a + 1], g.bits, g.fac_lo))
            col[b].append((SRC_ALPHA, shifts[b], g.bits, g.fac_hi))
            for q in range(a + 1, b):
                pas[q].append((shifts[q], shifts[q + 1], g.bits))
        if cut_bits.max() > int(math.log2(chi_limit)):
            raise BondTooLarge(f"factored bond dimension 2^{int(cut_bits.max())} exceeds the engine limit {chi_limit}")
        chis_cut = (1 << cut_bits).astype(np.int64)
        chi_max = max(chi_max, int(chis_cut.max()))

        # ---- MPO channels
        ow_terms = [(t, ham_terms[t][1]) for t in ow]
        rl_ch, lr_ch, rl_edges, lr_edges, fin_list = _build_mpo(ow_terms, c_lo, nsite, mode)
        d_max = max(d_max, max(len(x) for x in rl_ch), max(len(x) for x in lr_ch), 1)

        # ---- env offsets (RL channel envs stored at cuts 1..nsite)
        env_off = np.full(nsite + 1, -1, dtype=np.int64)
        off = 0
        for c in range(1, nsite + 1):
            env_off[c] = off
            off += len(rl_ch[c]) * int(chis_cut[c]) ** 2
        a_off = np.zeros(nsite, dtype=np.int64)      # folded cores A_k[s], stored by RL for LR
        for q in range(nsite):
            a_off[q] = off
            off += 2 * int(chis_cut[q]) * int(chis_cut[q + 1])
        g_off = np.zeros(nsite, dtype=np.int64)      # core cotangents G_k[s], LR sweep -> adjoint kernel
        if mode == "energy":
            for q in range(nsite):
                g_off[q] = off
                off += 2 * int(chis_cut[q]) * int(chis_cut[q + 1])
        seg_env = off

        # ---- emit site records
        site_begin = len(sites)
        gslot_begin = gslot_total
        g_local = 0
        for q in range(nsite):
            rec = np.zeros((), dtype=SITE_DTYPE)
            rec["op_begin"] = len(ops)
            rec["ent_begin"] = len(mats)
            lmat = 0
            ntrain = 0
            toff = 0      # digit bits introduced before this op (digit-tree level index width)
            tbase = 0     # entries of all previous tree levels
            ttb = 0       # entries of the previous trainable ops' levels (compact adjoint tree)
            for (src, shift, bits, specs) in col[q]:
                o = np.zeros((), dtype=OP_DTYPE)
                base = mat_block(specs)
                o["mat"], o["lmat"], o["src"], o["shift"], o["bits"] = base, lmat, src, shift, bits
                slots = {s.slot for s in specs if s.slot >= 0}
                if slots:
                    if len(slots) > 1:
                        raise InputError("one column op may carry only one trainable angle")
                    o["tidx"] = ntrain
                    o["gidx"] = g_local
                    gred.setdefault(slots.pop(), []).append(gslot_begin + g_local)
                    ntrain += 1
                    g_local += 1
                else:
                    o["tidx"], o["gidx"] = -1, -1
                o["toff"], o["tbase"] = toff, tbase
                tbase += 1 << (toff + bits)
                if o["tidx"] >= 0:
                    ttb += 1 << (toff + bits)
                toff += bits
                lmat += 1 << bits
                ops.append(o)
            max_tree = max(max_tree, tbase)
            max_ttree = max(max_ttree, ttb)
            rec["op_count"] = len(col[q])
            rec["lmat_count"] = lmat
            rec["n_train"] = ntrain
            max_ops = max(max_ops, len(col[q]))
            max_lmat = max(max_lmat, lmat)
            max_train = max(max_train, ntrain)
            rec["chi_l"], rec["chi_r"] = chis_cut[q], chis_cut[q + 1]
            rec["pass_begin"], rec["pass_count"] = len(passes), len(pas[q])
            for sa, sb, bits in pas[q]:
                p = np.zeros((), dtype=PASS_DTYPE)
                p["sa"], p["sb"], p["bits"] = sa, sb, bits
                passes.append(p)
            rec["rl_edge_begin"], rec["rl_edge_count"] = len(edges), len(rl_edges[q])
            edges.extend(rl_edges[q])
            rec["lr_edge_begin"], rec["lr_edge_count"] = len(edges), len(lr_edges[q])
            edges.extend(lr_edges[q])
            rec["fin_begin"], rec["fin_count"] = len(fins), len(fin_list[q])
            fins.extend(fin_list[q])
            rec["rl_da"], rec["rl_db"] = len(rl_ch[q]), len(rl_ch[q + 1])
            rec["lr_da"], rec["lr_db"] = len(lr_ch[q]), len(lr_ch[q + 1])
            rec["env_in"], rec["env_out"] = env_off[q + 1], env_off[q]
            rec["a_off"] = a_off[q]
            rec["g_off"] = g_off[q]
            v = np.array([1, 0], dtype=complex) if init_vecs is None else init_vecs[c_lo + q]
            rec["init"] = [v[0].real, v[0].imag, v[1].real, v[1].imag]
            sites.append(rec)
        if max_ops > MAX_OPS:
            raise InputError(f"a column holds {max_ops} operators; the engine limit is {MAX_OPS}")
        if max_train > MAX_TRAIN:
            raise InputError(f"a column holds {max_train} trainable angles; the engine limit is {MAX_TRAIN}")
        s = np.zeros((), dtype=SEG_DTYPE)
        s["site_begin"], s["site_count"] = site_begin, nsite
        s["gslot_begin"], s["gslot_count"] = gslot_begin, g_local
        s["lo"], s["hi"] = c_lo, c_hi
        s["env_base"], s["env_elems"] = env_total, seg_env
        segs.append(s)
        env_total += seg_env
        gslot_total += g_local

    P = int(circuit.n_params)
    ptr = np.zeros(P + 1, dtype=np.int32)
    idx = []
    for p in range(P):
        lst = gred.get(p, [])
        idx.extend(lst)
        ptr[p + 1] = ptr[p] + len(lst)

    def arr(lst, dt):
        return np.array(lst, dtype=dt) if lst else np.zeros(0, dtype=dt)

    plan = ChainPlan(
        n=n, n_params=P, n_terms=T, mode=mode,
        sites=arr(sites, SITE_DTYPE), ops=arr(ops, OP_DTYPE), mats=arr(mats, MAT_DTYPE),
        edges=arr(edges, EDGE_DTYPE), fins=arr(fins, EDGE_DTYPE), passes=arr(passes, PASS_DTYPE),
        segs=arr(segs, SEG_DTYPE), gred_ptr=ptr, gred_idx=np.array(idx, dtype=np.int32),
        chi_max=chi_max, d_max=d_max, max_edges=_max_edges(sites), max_tree=max_tree, max_ttree=max_ttree, max_ops=max_ops, max_lmat=max_lmat, max_train=max_train,
        n_gslots=gslot_total, env_total=env_total, e_const=e_const, term_active=active,
    )
    plan.info = {"segments": len(segs), "sub_chain_sites": int(sum(int(s["site_count"]) for s in segs)),
                 "chi_max": chi_max, "d_max": d_max}
    return plan


def _max_edges(sites):
    m = 1
    for r in sites:
        m = max(m, int(r["rl_edge_count"]), int(r["lr_edge_count"]), int(r["fin_count"]))
    return m


def real_path(plan) -> bool:
    """True when every factor matrix, input vector and MPO edge of the plan is real (ry
    rotations, real constant factors such as the CZ / CNOT projector splits, Paulis I/X/Z with
    real coefficients): the energy sweeps' complex arithmetic then has exactly-zero imaginary
    parts, and the engine runs its real-part instantiation (tq_chain.real_path)."""
    mats = plan.mats
    if len(mats):
        kind = mats["kind"]
        if not np.all((kind == 0) | (kind == 2)):
            return False
        const = mats["m"][kind == 0]
        if const.size and np.any(const.reshape(len(const), -1)[:, 1::2] != 0):
            return False
    if len(plan.sites) and np.any(plan.sites["init"][:, [1, 3]] != 0):
        return False
    if len(plan.edges) and np.any(plan.edges["op"] == 2):
        return False
    return True


def _edge(a, b, op, coef):
    e = np.zeros((), dtype=EDGE_DTYPE)
    e["a"], e["b"], e["op"], e["coef"] = a, b, op, coef
    return e


def _build_mpo(ow_terms, c_lo, nsite, mode):
    """Channels per local cut and per-site edge lists.

    energy mode (same automaton for both sweeps):
      START live at cut c iff an owned term starts at local site >= c,
      DONE  live at cut c iff an owned term ends at local site < c,
      INF(t) live for first(t) < c <= last(t).
    values mode: RL sweep carries only the identity environment (DONE);
      LR carries START + INF(t) and finalises each term against it."""
    terms = [(t, [(q - c_lo, code) for q, code in ops]) for t, ops in ow_terms]
    first = {t: ops[0][0] for t, ops in terms}
    last = {t: ops[-1][0] for t, ops in terms}
    max_first = max(first.values()) if terms else -1
    min_last = min(last.values()) if terms else nsite + 1

    def channels(c, with_done, with_start=True):
        ch = {}
        if with_start and max_first >= c:
            ch["S"] = len(ch)
        if with_done and min_last < c:
            ch["D"] = len(ch)
        for t, _ in terms:
            if first[t] < c <= last[t]:
                ch[t] = len(ch)
        return ch

    rl_edges = [[] for _ in range(nsite)]
    lr_edges = [[] for _ in range(nsite)]
    fins = [[] for _ in range(nsite)]
    if mode == "energy":
        ch = [channels(c, True) for c in range(nsite + 1)]
        for k in range(nsite):
            L, R = ch[k], ch[k + 1]
            el = []
            if "S" in L and "S" in R:
                el.append(_edge(L["S"], R["S"], 0, -1))
            if "D" in L and "D" in R:
                el.append(_edge(L["D"], R["D"], 0, -1))
            for t, ops in terms:
                sites = dict(ops)
                f, l = first[t], last[t]
                if not f <= k <= l:
                    continue
                op = sites.get(k, 0)
                src = L["S"] if k == f else L[t]
                if k == l:
                    el.append(_edge(src, R["D"], op, t))
                else:
                    el.append(_edge(src, R[t], op, -1))
            rl_edges[k] = el
            lr_edges[k] = el
        return ch, ch, rl_edges, lr_edges, fins
    if mode == "state":
        empty = [{} for _ in range(nsite + 1)]
        return empty, empty, rl_edges, lr_edges, fins
    if mode != "values":
        raise InputError(f"unknown plan mode {mode!r}")
    rl_ch = [{"D": 0} for _ in range(nsite + 1)]
    lr_ch = [channels(c, False) for c in range(nsite + 1)]
    for k in range(nsite):
        rl_edges[k] = [_edge(0, 0, 0, -1)]
        L, R = lr_ch[k], lr_ch[k + 1]
        el = []
        if "S" in L and "S" in R:
            el.append(_edge(L["S"], R["S"], 0, -1))
        fl = []
        for t, ops in terms:
            sites = dict(ops)
            f, l = first[t], last[t]
            if not f <= k <= l:
                continue
            op = sites.get(k, 0)
            src = L["S"] if k == f else L[t]
            if k == l:
                fl.append(_edge(src, t, op, -1))
            else:
                el.append(_edge(src, R[t], op, -1))
        lr_edges[k] = el
        fins[k] = fl
    return rl_ch, lr_ch, rl_edges, lr_edges, fins
