"""Engine entry points: compiled-plan cache, raw C-ABI calls, autograd Functions.

``ExpvalFunction``  E_b = sum_t c_t <P_t>  with dE/dtheta computed in the same call
                    (replaces grad_expval / evaluate_expval, reference autodiff.py:471-503).
``ValuesFunction``  v_{b,t} = <P_t> per term; its backward runs the energy sweep with
                    per-theta-set coefficients = the incoming cotangents, which is exactly
                    the gradient of the reference's tape through its readouts
                    (taped_expectations autodiff.py:405-425 as used by mbe_objective
                    maxcut.py:219-252).

Both go through ``libtq_engine.so``; nothing here computes physics on the CPU.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from . import chain as C
from .errors import InputError, NonHermitianResidue, NotFinite

_PLANS: "OrderedDict[tuple, _lib.DevicePlan]" = OrderedDict()
_MAX_PLANS = 32
_SEGS: dict = {}

DTYPES = {"complex64": (_lib.TQ_C64, torch.float32), "complex128": (_lib.TQ_C128, torch.float64)}


def residue_tol(dtype: str, coeff_abs_sum: float) -> float:
    """Imaginary-residue tolerance.  complex128 keeps the reference's 1e-8
    (hamiltonians.py:34); complex64 scales with the operator norm bound."""
    if dtype == "complex128":
        return 1e-8
    return max(1e-6, 1e-5 * coeff_abs_sum)


def _dtype(dtype: str):
    if dtype not in DTYPES:
        raise InputError(f"dtype must be 'complex64' or 'complex128', got {dtype!r}")
    return DTYPES[dtype]


def _stream():
    return torch.cuda.current_stream().cuda_stream


def device_plan(circuit, terms, mode: str, batch: int, device, segments=None, init=None, dtype="complex64"):
    """Compiled + uploaded plan for (circuit structure, term supports, mode, segmentation)."""
    dev = torch.device(device)
    if dev.type != "cuda":
        raise InputError("the B200 engine runs on CUDA devices only")
    supports = tuple(ops for _, ops in terms)
    if segments is None:
        skey = (C.structure_key(circuit), supports, int(batch))
        seg_key = _SEGS.get(skey)
        if seg_key is None:
            seg_key = C.choose_segments(circuit.n_qubits, terms, C.time_gates(circuit), batch)
            _SEGS[skey] = seg_key
    else:
        seg_key = segments
    init_key = None if init is None else np.asarray(init, dtype=complex).tobytes()
    key = (C.structure_key(circuit), supports, mode, seg_key, init_key,
           dev.index if dev.index is not None else torch.cuda.current_device(), dtype)
    dp = _PLANS.get(key)
    if dp is None:
        limit = C.MAX_CHI if dtype == "complex64" else C.MAX_CHI_F64
        plan = C.compile_chain(circuit, terms, mode=mode, batch=batch, segments=seg_key, init=init,
                               chi_limit=limit)
        dp = _lib.DevicePlan(plan, dev, dtype)
        _PLANS[key] = dp
        while len(_PLANS) > _MAX_PLANS:
            _PLANS.popitem(last=False)
    else:
        _PLANS.move_to_end(key)
    return dp


def _workspace(dp, ws, batch, flags, code, stream):
    """Caller-owned scratch (a uint8 device tensor, e.g. one per captured graph) or the plan's
    per-stream cache."""
    if ws is None:
        return dp.workspace(batch, flags, code, stream)
    need = int(_lib.load().tq_workspace_bytes(ctypes.byref(dp.chain), batch, flags, code))
    if ws.numel() < need or ws.device != dp.device:
        raise InputError(f"workspace must be a uint8 tensor of >= {need} bytes on {dp.device}")
    return ws, need


def workspace_bytes(dp: _lib.DevicePlan, batch: int, want_grad: bool, dtype: str, values: bool = False) -> int:
    code, _ = _dtype(dtype)
    flags = _lib.TQ_FLAG_VALUES if values else (_lib.TQ_FLAG_GRAD if want_grad else 0)
    return int(_lib.load().tq_workspace_bytes(ctypes.byref(dp.chain), batch, flags, code))


def energy_grad_raw(dp: _lib.DevicePlan, theta: torch.Tensor, coef: torch.Tensor, want_grad: bool, dtype: str,
                    out=None, ws=None):
    """theta [B,P], coef [B or 1, T] on the plan's device -> (E [B,2] float64, grad [B,P] | None).

    ``out = (energy, grad)`` supplies the output buffers instead: device tensors, or pinned host
    tensors, which the reduction kernels then write directly over the bus (the serving
    program's host-buffer graph uses this in place of separate device-to-host copies).
    ``ws`` is a caller-owned workspace: a captured graph bakes its scratch pointer in, so every
    graph that may replay concurrently with another owns its own."""
    code, tdt = _dtype(dtype)
    theta = theta.to(device=dp.device, dtype=tdt).contiguous()
    coef = coef.to(device=dp.device, dtype=tdt).contiguous()
    B = theta.shape[0]
    if theta.dim() != 2 or theta.shape[1] != dp.plan.n_params:
        raise InputError(f"theta must be [B, {dp.plan.n_params}], got {tuple(theta.shape)}")
    if coef.shape[-1] != dp.plan.n_terms or coef.shape[0] not in (1, B):
        raise InputError("coefficient array shape mismatch")
    if out is None:
        energy = torch.empty(B, 2, dtype=torch.float64, device=dp.device)
        grad = torch.empty(B, dp.plan.n_params, dtype=tdt, device=dp.device) if want_grad else None
    else:
        energy, grad = out
        for t, shape, dt in ((energy, (B, 2), torch.float64), (grad, (B, dp.plan.n_params), tdt)):
            if t is None:
                continue
            if tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous():
                raise InputError(f"output buffer must be a contiguous {dt} tensor of shape {shape}")
            if t.device.type == "cpu" and not t.is_pinned():
                raise InputError("host output buffers must be pinned")
        if want_grad and grad is None:
            raise InputError("want_grad needs a gradient output buffer")
    stream = _stream()
    ws, nbytes = _workspace(dp, ws, B, _lib.TQ_FLAG_GRAD if want_grad else 0, code, stream)
    st = _lib.load().tq_energy_grad(
        ctypes.byref(dp.chain), code, B, theta.data_ptr(), theta.stride(0) if B else 0,
        coef.data_ptr(), coef.stride(0) if coef.shape[0] > 1 else 0,
        energy.data_ptr(), grad.data_ptr() if grad is not None else None,
        ws.data_ptr(), nbytes, stream)
    _lib.check(st)
    return energy, grad


def values_raw(dp: _lib.DevicePlan, theta: torch.Tensor, dtype: str, ws=None) -> torch.Tensor:
    """theta [B,P] -> complex128 [B,T] term values (``ws``: optional caller-owned workspace)."""
    code, tdt = _dtype(dtype)
    theta = theta.to(device=dp.device, dtype=tdt).contiguous()
    B = theta.shape[0]
    vals = torch.zeros(B, dp.plan.n_terms, 2, dtype=torch.float64, device=dp.device)
    stream = _stream()
    ws, nbytes = _workspace(dp, ws, B, _lib.TQ_FLAG_VALUES, code, stream)
    st = _lib.load().tq_term_values(ctypes.byref(dp.chain), code, B, theta.data_ptr(),
                                    theta.stride(0) if B else 0, vals.data_ptr(), ws.data_ptr(), nbytes, stream)
    _lib.check(st)
    return torch.view_as_complex(vals)


class ExpvalFunction(torch.autograd.Function):
    """E[b] = Re sum_t coef[t] <psi(theta_b)|P_t|psi(theta_b)>; gradient from the same launch."""

    @staticmethod
    def forward(ctx, theta, dp, coef, dtype):
        want = bool(ctx.needs_input_grad[0])
        energy, grad = energy_grad_raw(dp, theta.detach(), coef, want, dtype)
        if want:
            ctx.save_for_backward(grad)
        ctx.in_dtype = theta.dtype
        ctx.mark_non_differentiable(energy)
        return energy[:, 0].clone(), energy

    @staticmethod
    def backward(ctx, g_e, _g_full):
        (grad,) = ctx.saved_tensors
        return (g_e.to(grad.dtype)[:, None] * grad).to(ctx.in_dtype), None, None, None


class ValuesFunction(torch.autograd.Function):
    """Re <P_t> for every term; backward = energy sweep with per-theta-set coefficients."""

    @staticmethod
    def forward(ctx, theta, dp_values, dp_energy, dtype):
        vals = values_raw(dp_values, theta.detach(), dtype)
        ctx.dp_energy, ctx.dtype = dp_energy, dtype
        ctx.in_dtype = theta.dtype
        ctx.save_for_backward(theta.detach())
        return vals.real.clone(), vals.imag.clone()

    @staticmethod
    def backward(ctx, g_re, _g_im):
        (theta,) = ctx.saved_tensors
        _, grad = energy_grad_raw(ctx.dp_energy, theta, g_re.contiguous(), True, ctx.dtype)
        return grad.to(ctx.in_dtype), None, None, None


def check_finite(*tensors):
    for t in tensors:
        if t is not None and not bool(torch.isfinite(t).all()):
            raise NotFinite("engine produced NaN or Inf")


def check_residue(energy_full: torch.Tensor, im_extra, tol: float):
    im = energy_full[:, 1]
    if im_extra is not None:
        im = im + im_extra
    worst = float(im.abs().max()) if im.numel() else 0.0
    if worst > tol:
        raise NonHermitianResidue(f"imaginary residue {worst:.3e} exceeds {tol:.0e}")


def inner_raw(dp_bra: _lib.DevicePlan, theta_bra: torch.Tensor, dp_ket: _lib.DevicePlan, theta_ket: torch.Tensor,
              dtype: str) -> torch.Tensor:
    """<bra_b|ket_b> for b in the batch (complex128 [B]); plans compiled in 'state' mode."""
    code, tdt = _dtype(dtype)
    tb = theta_bra.to(device=dp_ket.device, dtype=tdt).contiguous()
    tk = theta_ket.to(device=dp_ket.device, dtype=tdt).contiguous()
    B = tk.shape[0]
    if tb.shape[0] != B:
        raise InputError("bra and ket batches differ")
    out = torch.zeros(B, 2, dtype=torch.float64, device=dp_ket.device)
    st = _lib.load().tq_inner(ctypes.byref(dp_bra.chain), tb.data_ptr(), tb.stride(0) if tb.numel() else 0,
                              ctypes.byref(dp_ket.chain), tk.data_ptr(), tk.stride(0) if tk.numel() else 0,
                              code, B, out.data_ptr(), _stream())
    _lib.check(st)
    return torch.view_as_complex(out)
