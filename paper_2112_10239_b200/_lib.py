"""ctypes binding of the C-ABI engine library ``libtq_engine.so`` (include/tq_engine.h).

The library is built in-tree by :func:`paper_2112_10239_b200.build.build_library`
(nvcc, ``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback:
if the library or a CUDA device is missing every engine call raises
:class:`EngineUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import chain as C
from .errors import BondTooLarge, EngineError, EngineUnavailable, InputError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TQ_ENGINE_LIB") or os.path.join(HERE, "libtq_engine.so")

TQ_OK, TQ_ERR_INPUT, TQ_ERR_UNSUPPORTED, TQ_ERR_CUDA, TQ_ERR_WORKSPACE = 0, 1, 2, 3, 4
TQ_C64, TQ_C128 = 0, 1
TQ_FLAG_GRAD, TQ_FLAG_VALUES = 1, 2


class TqChain(ctypes.Structure):
    """Mirror of ``tq_chain`` (include/tq_engine.h)."""

    _fields_ = [
        ("n_segments", ctypes.c_int32), ("n_sites", ctypes.c_int32), ("n_params", ctypes.c_int32),
        ("n_terms", ctypes.c_int32), ("chi_max", ctypes.c_int32), ("d_max", ctypes.c_int32),
        ("max_ops", ctypes.c_int32), ("max_lmat", ctypes.c_int32), ("max_train", ctypes.c_int32),
        ("n_gslots", ctypes.c_int32), ("max_edges", ctypes.c_int32), ("max_tree", ctypes.c_int32),
        ("env_total", ctypes.c_int64),
        ("e_const_re", ctypes.c_double), ("e_const_im", ctypes.c_double),
        ("sites", ctypes.c_void_p), ("ops", ctypes.c_void_p), ("mats", ctypes.c_void_p),
        ("edges", ctypes.c_void_p), ("fins", ctypes.c_void_p), ("passes", ctypes.c_void_p),
        ("segs", ctypes.c_void_p), ("gred_ptr", ctypes.c_void_p), ("gred_idx", ctypes.c_void_p),
        ("term_active", ctypes.c_void_p),
        ("blob", ctypes.c_void_p), ("blob_off", ctypes.c_void_p),
        ("blob_max", ctypes.c_int32), ("blob_dtype", ctypes.c_int32),
        ("max_pairs", ctypes.c_int32), ("max_ttree", ctypes.c_int32),
        ("real_path", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the engine library; raises EngineUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise EngineUnavailable(
                f"engine library {p} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            import torch  # noqa: F401  (loads libcudart first so the shared runtime is reused)
        except Exception:  # pragma: no cover - torch is always present in this image
            pass
        lib = ctypes.CDLL(p)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        pc = ctypes.POINTER(TqChain)
        lib.tq_workspace_bytes.restype = sz
        lib.tq_workspace_bytes.argtypes = [pc, i32, i32, i32]
        lib.tq_energy_grad.restype = i32
        lib.tq_energy_grad.argtypes = [pc, i32, i32, vp, i64, vp, i64, vp, vp, vp, sz, vp]
        lib.tq_energy_grad_timed.restype = i32
        lib.tq_energy_grad_timed.argtypes = [pc, i32, i32, vp, i64, vp, i64, vp, vp, vp, sz, vp, ctypes.POINTER(ctypes.c_float)]
        lib.tq_ffma_peak.restype = i32
        lib.tq_ffma_peak.argtypes = [i32, vp, ctypes.POINTER(ctypes.c_double)]
        lib.tq_term_values.restype = i32
        lib.tq_term_values.argtypes = [pc, i32, i32, vp, i64, vp, vp, sz, vp]
        lib.tq_inner.restype = i32
        lib.tq_inner.argtypes = [pc, vp, i64, pc, vp, i64, i32, i32, vp, vp]
        lib.tq_status_string.restype = ctypes.c_char_p
        lib.tq_status_string.argtypes = [i32]
        lib.tq_last_error.restype = ctypes.c_char_p
        lib.tq_last_error.argtypes = []
        lib.tq_abi_layout.restype = i32
        lib.tq_abi_layout.argtypes = [ctypes.POINTER(i32), i32]
        lib.tq_build_info.restype = ctypes.c_char_p
        lib.tq_build_info.argtypes = []
        lib.tq_tt_workspace_bytes.restype = sz
        lib.tq_tt_workspace_bytes.argtypes = [i32, i32, i32, i32]
        lib.tq_tt_simulate.restype = i32
        lib.tq_tt_simulate.argtypes = [i32, vp, i32, i32, i32, vp, i64, ctypes.c_double, i32, i32,
                                       vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, sz, vp]
        lib.tq_tt_state_bytes.restype = sz
        lib.tq_tt_state_bytes.argtypes = [i32, i32, i32, i32]
        lib.tq_tt_values_workspace_bytes.restype = sz
        lib.tq_tt_values_workspace_bytes.argtypes = [i32, i32, i32, i32]
        lib.tq_tt_run.restype = i32
        lib.tq_tt_run.argtypes = [i32, vp, i32, i32, i32, vp, i64, ctypes.c_double, i32, i32, vp, vp, vp, vp, vp, vp]
        lib.tq_tt_compress.restype = i32
        lib.tq_tt_compress.argtypes = [i32, i32, i32, ctypes.c_double, i32, i32, vp, vp, vp, vp, vp, vp]
        lib.tq_tt_values.restype = i32
        lib.tq_tt_values.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, sz, vp]
        lib.tq_tt_tape_bytes.restype = sz
        lib.tq_tt_tape_bytes.argtypes = [i32, i32, i32, i32]
        lib.tq_tt_taped.restype = i32
        lib.tq_tt_taped.argtypes = [i32, vp, i32, i32, i32, i32, vp, i64, ctypes.c_double, i32, i32,
                                    vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        lib.tq_tt_replay.restype = i32
        lib.tq_tt_replay.argtypes = [i32, vp, i32, i32, i32, i32, vp, i64, i32, vp, i32, vp,
                                     vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        lib.tq_tt_apply.restype = i32
        lib.tq_tt_apply.argtypes = [i32, vp, i32, i32, i32, vp, i64, ctypes.c_double, i32, i32, vp, vp, vp, vp, vp, vp]
        lib.tq_tt_inner.restype = i32
        lib.tq_tt_inner.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]
        lib.tq_tt_dfma_peak.restype = i32
        lib.tq_tt_dfma_peak.argtypes = [i32, vp, ctypes.POINTER(ctypes.c_double)]
        _lib = lib
        return lib


EXPORTED_SYMBOLS = ("tq_workspace_bytes", "tq_energy_grad", "tq_energy_grad_timed", "tq_ffma_peak",
                    "tq_term_values", "tq_inner",
                    "tq_status_string", "tq_last_error", "tq_abi_layout", "tq_build_info",
                    "tq_tt_workspace_bytes", "tq_tt_simulate", "tq_tt_dfma_peak", "tq_tt_state_bytes",
                    "tq_tt_values_workspace_bytes", "tq_tt_run", "tq_tt_compress", "tq_tt_values",
                    "tq_tt_tape_bytes", "tq_tt_taped", "tq_tt_replay", "tq_tt_inner", "tq_tt_apply")


def check(status: int):
    """Map a tq_status onto the reference exception taxonomy."""
    if status == TQ_OK:
        return
    msg = load().tq_last_error().decode(errors="replace")
    if status == TQ_ERR_UNSUPPORTED:
        raise BondTooLarge(msg)
    if status in (TQ_ERR_INPUT, TQ_ERR_WORKSPACE):
        raise InputError(msg)
    raise EngineError(msg)


def abi_sizes():
    lib = load()
    arr = (ctypes.c_int32 * 7)()
    lib.tq_abi_layout(arr, 7)
    return list(arr)


NUMPY_SIZES = [C.SITE_DTYPE.itemsize, C.OP_DTYPE.itemsize, C.MAT_DTYPE.itemsize, C.EDGE_DTYPE.itemsize,
               C.PASS_DTYPE.itemsize, C.SEG_DTYPE.itemsize, ctypes.sizeof(TqChain)]


def pack_opcode(ops: np.ndarray) -> np.ndarray:
    """Kernel op code: lmat[0:9] src[9:11] kshift[11:16] bits[16:18] tidx+1[18:24] toff[24:29];
    kshift = the digit's position in the pair key alpha | beta << 8 (csrc oc_digit)."""
    ksh = ops["shift"] + np.where(ops["src"] == 2, 8, 0)
    bits = np.where(ops["src"] == 0, 0, ops["bits"])
    return (ops["lmat"] | (ops["src"] << 9) | (ksh << 11) | (bits << 16)
            | ((ops["tidx"] + 1) << 18) | (ops["toff"] << 24)).astype(np.int32)


SITE_UNITS = C.SITE_DTYPE.itemsize // 16


def build_blobs(plan: C.ChainPlan, dtype_code: int):
    """Per-site descriptor blobs (layout in include/tq_engine.h); returns (bytes, offsets, max)."""
    eu = 3 if dtype_code == TQ_C64 else 6
    rdt = np.float32 if dtype_code == TQ_C64 else np.float64
    sites, ops, mats, edges = plan.sites, plan.ops, plan.mats, plan.edges
    nsite = len(sites)
    lens = np.zeros(nsite, dtype=np.int64)
    for i in range(nsite):
        st = sites[i]
        lens[i] = 1 + SITE_UNITS + int(st["op_count"]) + eu * int(st["lmat_count"]) + int(st["rl_edge_count"]) + int(st["lr_edge_count"])
    offs = np.zeros(nsite, dtype=np.int64)
    offs[1:] = np.cumsum(lens)[:-1]
    total = int(lens.sum()) if nsite else 1
    bmax = int(lens.max()) if nsite else 1
    buf = np.zeros((total + bmax) * 16, dtype=np.uint8)   # tail padding: prefetches copy bmax units
    seg_of = np.zeros(nsite, dtype=np.int64)
    nxt_rl = np.full(nsite, -1, dtype=np.int64)
    nxt_lr = np.full(nsite, -1, dtype=np.int64)
    for si, sg in enumerate(plan.segs):
        b0, cnt = int(sg["site_begin"]), int(sg["site_count"])
        for k in range(cnt):
            i = b0 + k
            seg_of[i] = si
            if k > 0:
                nxt_rl[i] = offs[i - 1]
            if k + 1 < cnt:
                nxt_lr[i] = offs[i + 1]
    opc = pack_opcode(ops) if len(ops) else np.zeros(0, np.int32)
    for i in range(nsite):
        st = sites[i]
        base = int(offs[i]) * 16
        hdr = np.array([lens[i], nxt_rl[i], nxt_lr[i], seg_of[i]], dtype=np.int32)
        buf[base:base + 16] = hdr.view(np.uint8)
        buf[base + 16:base + 16 + 16 * SITE_UNITS] = np.frombuffer(st.tobytes(), dtype=np.uint8)
        o = base + 16 + 16 * SITE_UNITS
        ob, oc = int(st["op_begin"]), int(st["op_count"])
        if oc:
            rec = np.zeros((oc, 4), dtype=np.int32)
            rec[:, 0] = opc[ob:ob + oc]
            rec[:, 1] = ops["gidx"][ob:ob + oc]
            rec[:, 2] = ops["tbase"][ob:ob + oc]
            rec[:, 3] = ops["tidx"][ob:ob + oc]
            buf[o:o + 16 * oc] = rec.view(np.uint8).reshape(-1)
            o += 16 * oc
        eb, ec = int(st["ent_begin"]), int(st["lmat_count"])
        if ec:
            m = mats[eb:eb + ec]
            if dtype_code == TQ_C64:
                rec = np.zeros((ec, 12), dtype=np.int32)
                rec[:, 0] = m["kind"] | (m["cls"] << 8)
                rec[:, 1] = m["slot"]
                f = rec.view(np.float32)
                f[:, 2] = (1.0 / m["pscale"]).astype(np.float32)
                f[:, 3] = m["angle"].astype(np.float32)
                f[:, 4:12] = m["m"].astype(np.float32)
            else:
                rec = np.zeros((ec, 24), dtype=np.int32)
                rec[:, 0] = m["kind"] | (m["cls"] << 8)
                rec[:, 1] = m["slot"]
                f = rec.view(np.float64)
                f[:, 1] = 1.0 / m["pscale"]
                f[:, 2] = m["angle"]
                f[:, 3:11] = m["m"]
            buf[o:o + 16 * eu * ec] = rec.view(np.uint8).reshape(-1)
            o += 16 * eu * ec
        for key in ("rl", "lr"):
            b, c = int(st[f"{key}_edge_begin"]), int(st[f"{key}_edge_count"])
            if c:
                buf[o:o + 16 * c] = np.frombuffer(edges[b:b + c].tobytes(), dtype=np.uint8)
                o += 16 * c
    return buf, offs.astype(np.int32), bmax


class DevicePlan:
    """A ChainPlan uploaded to one CUDA device (tables live in torch uint8 tensors)."""

    def __init__(self, plan: C.ChainPlan, device, dtype: str = "complex64"):
        import torch

        if not torch.cuda.is_available():
            raise EngineUnavailable("no CUDA device is available; the B200 engine has no CPU fallback")
        load()
        self.plan = plan
        self.device = torch.device(device)
        self._keep = {}

        def up(name, arr):
            a = np.ascontiguousarray(arr)
            if a.nbytes == 0:
                a = np.zeros(16, dtype=np.uint8)
            t = torch.from_numpy(a.view(np.uint8).copy()).to(self.device)
            self._keep[name] = t
            return t.data_ptr()

        ch = TqChain()
        ch.n_segments = plan.n_segments
        ch.n_sites = len(plan.sites)
        ch.n_params = plan.n_params
        ch.n_terms = plan.n_terms
        ch.chi_max = plan.chi_max
        ch.d_max = plan.d_max
        ch.max_ops = plan.max_ops
        ch.max_lmat = plan.max_lmat
        ch.max_train = plan.max_train
        ch.n_gslots = plan.n_gslots
        ch.max_edges = plan.max_edges
        ch.max_tree = plan.max_tree
        ch.env_total = plan.env_total
        ch.e_const_re = plan.e_const.real
        ch.e_const_im = plan.e_const.imag
        ch.sites = up("sites", plan.sites)
        ch.ops = up("ops", plan.ops)
        ch.mats = up("mats", plan.mats)
        ch.edges = up("edges", plan.edges)
        ch.fins = up("fins", plan.fins)
        ch.passes = up("passes", plan.passes)
        ch.segs = up("segs", plan.segs)
        ch.gred_ptr = up("gred_ptr", plan.gred_ptr)
        ch.gred_idx = up("gred_idx", plan.gred_idx)
        ch.term_active = up("term_active", plan.term_active)
        code = TQ_C64 if dtype == "complex64" else TQ_C128
        blob, boff, bmax = build_blobs(plan, code)
        ch.blob = up("blob", blob)
        ch.blob_off = up("blob_off", boff)
        ch.blob_max = bmax
        ch.blob_dtype = code
        ch.max_pairs = int((plan.sites["chi_l"] * plan.sites["chi_r"]).max()) if len(plan.sites) else 1
        ch.max_ttree = int(plan.max_ttree)
        ch.real_path = int(C.real_path(plan))
        self.chain = ch
        self._ws = {}

    def workspace(self, batch: int, flags: int, dtype: int, stream_ptr: int = 0):
        """Cached device workspace, one buffer per (flags, dtype, stream) so concurrent
        callers on different streams never share scratch."""
        import torch

        need = int(load().tq_workspace_bytes(ctypes.byref(self.chain), batch, flags, dtype))
        key = (flags, dtype, stream_ptr)
        buf = self._ws.get(key)
        if buf is None or buf.numel() < need:
            buf = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._ws[key] = buf
        return buf, need
