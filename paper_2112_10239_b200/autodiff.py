"""Reference-compatible value/gradient API on the B200 engine.

Same names, argument meaning and error behaviour as ``tnsim.autodiff``
(reference ``autodiff.py:445-659``) for the TT engine.  Differences:

* ``engine`` accepts ``"tt"`` / ``"b200"`` (both mean this engine); the reference's
  ``"dense"`` oracle engine is not part of the product and raises ``InputError``.
* The engine is exact (the reference's ``eps=0`` semantics) for any ``eps``;
  ``chi_max`` below the exact factored bond raises ``InputError`` (truncated
  straight-through mode is a later row).
* ``theta`` may be 2-D ``[B, P]``: B independent parameter sets in one launch.
* ``dtype="complex64"`` (default, the B200 fast path) or ``"complex128"`` (parity mode).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import chain as C
from . import engine as E
from .circuits import Circuit
from .errors import (
    DivergenceDetected,
    InputError,
    ParamCountMismatch,
    TooManyQubits,
    UnsupportedGateForShift,
    WireOutOfRange,
)
from .hamiltonians import PAULI_MATRICES, PauliHamiltonian

SHIFTABLE_GATES = ("rx", "ry", "rz", "crz")
_CRZ_Y1 = (np.sqrt(2.0) + 1.0) / (4.0 * np.sqrt(2.0))
_CRZ_Y2 = (np.sqrt(2.0) - 1.0) / (4.0 * np.sqrt(2.0))


MAX_DENSE_QUBITS = 26   # the reference dense engine's width guard (circuits.py:36, autodiff.py:288)


def _check_engine(engine: str) -> str:
    """Reference autodiff.py:456-459 (engine seam).  'tt' / 'b200' and the reference's default
    'dense' all run on the B200 engine; see :func:`_engine_args` for what 'dense' means."""
    if engine in ("tt", "b200", "dense"):
        return engine
    raise InputError(f"unknown engine {engine!r}; expected 'dense', 'tt' or 'b200'")


def _engine_args(engine: str, circuit, eps: float, chi_max):
    """(eps, chi_max) the engine runs with.  engine='dense' is the reference's exact state-vector
    path: exact results, eps/chi_max ignored, and the same width guard (TooManyQubits above 26
    qubits).  The B200 engine computes those exact values without a state vector (the factored
    chain at eps=0), so callers relying on the reference's default engine get its numbers."""
    _check_engine(engine)
    if engine == "dense":
        if circuit.n_qubits > MAX_DENSE_QUBITS:
            raise TooManyQubits(f"n={circuit.n_qubits} exceeds the dense guard for the dense engine")
        return 0.0, None
    return eps, chi_max


def _check_theta(circuit: Circuit, theta):
    """Reference autodiff.py:445-453; returns float64 [B, P] and whether input was 1-D."""
    if isinstance(theta, torch.Tensor):
        theta = theta.detach().cpu().double().numpy()
    arr = np.asarray(theta, dtype=float)
    single = arr.ndim <= 1
    arr = arr.reshape(1, -1) if single else arr
    if arr.ndim != 2 or arr.shape[1] != circuit.n_params:
        raise ParamCountMismatch(f"{arr.shape[-1] if arr.ndim else arr.size} parameters supplied, "
                                 f"circuit has {circuit.n_params} slots")
    if arr.size and not np.all(np.isfinite(arr)):
        raise InputError("parameters must be finite")
    return arr, single


def _check_chi(plan, chi_max):
    if chi_max is not None and int(chi_max) < plan.chi_max:
        raise InputError(f"chi_max={chi_max} would truncate the exact factored bond {plan.chi_max}; "
                         "the B200 engine is exact (eps=0 semantics)")


def _truncating(circuit: Circuit, eps: float, chi_max) -> bool:
    """True when (eps, chi_max) can change the state: the truncated engine (row f3) runs.
    eps = 0 with chi_max at or above the exact factored bond truncates nothing."""
    if eps < 0:
        raise InputError(f"eps must be >= 0, got {eps}")
    if eps > 0:
        return True
    if chi_max is None:
        return False
    if int(chi_max) < 1:
        raise InputError(f"chi_max must be >= 1, got {chi_max}")
    return int(chi_max) < C.factored_chi(circuit.n_qubits, C.time_gates(circuit))


def _taped_truncates(circuit: Circuit, eps: float, chi_max) -> bool:
    """True when the reference's TAPED path (grad_expval / taped_expectations with eps, chi_max)
    would cut a split: it keeps every singular value at eps = 0, zeros included, so its bonds are
    min(2 chi_l, 2 chi_r) per split (no centre moves, _tt_taped_split autodiff.py:315-336) and can
    exceed both the true Schmidt rank and the factored bond.  A cut that only drops zero singular
    values leaves the state (and value) exact but freezes a non-square factor, so the gradient is
    then the straight-through one, not the exact one.  eps > 0 may cut anywhere: True."""
    if eps > 0:
        return True
    if chi_max is None:
        return False
    from . import truncated as TR

    table, _ = TR.compile_gates(circuit)
    dims = [1] * (circuit.n_qubits + 1)
    cap = int(chi_max)
    for g in table:
        if g["kind"] != 2:
            continue
        i = int(g["site"])
        k = min(2 * dims[i], 2 * dims[i + 2])
        if k > cap:
            return True
        dims[i + 1] = k
    return False


def _truncated_expval(circuit, ham, arr, eps, chi_max, dtype, device):
    """Forward value through the truncated TT engine (reference simulate_tt + expval,
    tt.py:237-244 / hamiltonians.py:167-187), every theta-set of arr [B, P] in one launch."""
    from . import truncated as TR

    terms = _terms(ham, circuit.n_qubits)
    res = TR.simulate_terms(circuit, terms, arr, eps, chi_max, dtype=dtype, device=device)
    e = res.energy([c for c, _ in terms])
    tol = E.residue_tol(dtype, sum(abs(c) for c, _ in terms))
    worst = float(np.max(np.abs(e.imag))) if e.size else 0.0
    if not np.all(np.isfinite(e)):
        from .errors import NotFinite
        raise NotFinite("engine produced NaN or Inf")
    if worst > tol:
        from .errors import NonHermitianResidue
        raise NonHermitianResidue(f"imaginary residue {worst:.3e} exceeds {tol:.0e}")
    return e.real


def _straight_through(circuit, ham, arr, eps, chi_max, dtype, device):
    """(E [B], grad [B, P]) of the reference's taped truncated evaluation (truncated.straight_through);
    the taped value gets the same residue and finiteness checks as every energy."""
    from . import truncated as TR

    terms = _terms(ham, circuit.n_qubits)
    vals, grad = TR.straight_through(circuit, terms, arr, eps, chi_max, dtype=dtype, device=device)
    e = vals @ np.array([c for c, _ in terms], dtype=complex) if terms else np.zeros(arr.shape[0], complex)
    if not (np.all(np.isfinite(e)) and np.all(np.isfinite(grad))):
        from .errors import NotFinite
        raise NotFinite("engine produced NaN or Inf")
    tol = E.residue_tol(dtype, sum(abs(c) for c, _ in terms))
    worst = float(np.max(np.abs(e.imag))) if e.size else 0.0
    if worst > tol:
        from .errors import NonHermitianResidue
        raise NonHermitianResidue(f"imaginary residue {worst:.3e} exceeds {tol:.0e}")
    return e.real, grad


def _device(device):
    if device is None:
        if not torch.cuda.is_available():
            from .errors import EngineUnavailable
            raise EngineUnavailable("no CUDA device is available; the B200 engine has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _terms(ham: PauliHamiltonian, n: int):
    if ham.n_qubits != n:
        raise InputError(f"state has {n} qubits, Hamiltonian {ham.n_qubits}")
    return C.normalize_terms(ham)


def energy(circuit: Circuit, ham: PauliHamiltonian, theta: torch.Tensor, *, dtype: str = "complex64",
           segments=None, check: bool = True) -> torch.Tensor:
    """Torch-native, differentiable: theta [B,P] (device tensor) -> Re<H> [B] (float64).

    Gradients are produced by the same engine call (the reference's one-tape
    value+gradient, autodiff.py:471-487) and flow through ``torch.autograd``."""
    terms = _terms(ham, circuit.n_qubits)
    if theta.dim() == 1:
        theta = theta[None]
    dev = theta.device
    dp = E.device_plan(circuit, terms, "energy", theta.shape[0], dev, segments, dtype=dtype)
    coef = torch.tensor([[c.real for c, _ in terms]], dtype=torch.float64, device=dev)
    val, full = E.ExpvalFunction.apply(theta, dp, coef, dtype)
    if check:
        E.check_finite(full)
        im_extra = None
        if any(c.imag != 0 for c, _ in terms):
            cim = torch.tensor([[c.imag for c, _ in terms]], dtype=torch.float64, device=dev)
            e_im, _ = E.energy_grad_raw(dp, theta.detach(), cim, False, dtype)
            im_extra = e_im[:, 0]
        E.check_residue(full, im_extra, E.residue_tol(dtype, sum(abs(c) for c, _ in terms)))
    return val


def grad_expval(circuit: Circuit, ham: PauliHamiltonian, theta, engine: str = "tt", eps: float = 0.0,
                chi_max=None, *, dtype: str = "complex64", device=None, segments=None):
    """Value and gradient of <H> (reference autodiff.py:471-487).

    1-D theta -> (float, float64[P]); 2-D theta [B,P] -> (float64[B], float64[B,P])."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    arr, single = _check_theta(circuit, theta)
    if _truncating(circuit, eps, chi_max) or _taped_truncates(circuit, eps, chi_max):
        # the reference's straight-through gradient of its taped truncated state (autodiff.py:10-13,
        # 315-363): value of the taped construction and the gradient with the split constants frozen
        v, g = _straight_through(circuit, ham, arr, eps, chi_max, dtype if dtype != "complex64" else "complex128",
                                 device)
        return (float(v[0]), g[0]) if single else (v, g)
    dev = _device(device)
    terms = _terms(ham, circuit.n_qubits)
    dp = E.device_plan(circuit, terms, "energy", arr.shape[0], dev, segments, dtype=dtype)
    _check_chi(dp.plan, chi_max)
    tdt = E.DTYPES[dtype][1]
    th = torch.tensor(arr, dtype=tdt, device=dev, requires_grad=True)
    val = energy(circuit, ham, th, dtype=dtype, segments=segments)
    (g,) = torch.autograd.grad(val.sum(), th)
    v = val.detach().cpu().numpy()
    gg = g.detach().double().cpu().numpy()
    if single:
        return float(v[0]), gg[0]
    return v, gg


def evaluate_expval(circuit: Circuit, ham: PauliHamiltonian, theta=None, engine: str = "tt", eps: float = 0.0,
                    chi_max=None, *, dtype: str | None = None, device=None, segments=None):
    """Forward-only <H> (reference autodiff.py:490-503): one right-to-left sweep, nothing stored.
    With truncation requested (eps > 0, or chi_max below the exact bond) the truncated TT
    engine runs instead (row f3, ``truncated.py``)."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    arr, single = _check_theta(circuit, circuit.params() if theta is None else theta)
    if _truncating(circuit, eps, chi_max):
        # long truncated evolutions accumulate rounding with depth: complex128 unless asked
        v = _truncated_expval(circuit, ham, arr, eps, chi_max, dtype or "complex128", device)
        return float(v[0]) if single else v
    dtype = dtype or "complex64"
    dev = _device(device)
    terms = _terms(ham, circuit.n_qubits)
    dp = E.device_plan(circuit, terms, "energy", arr.shape[0], dev, segments, dtype=dtype)
    _check_chi(dp.plan, chi_max)
    th = torch.tensor(arr, dtype=E.DTYPES[dtype][1], device=dev)
    v = energy(circuit, ham, th, dtype=dtype, segments=segments).cpu().numpy()
    return float(v[0]) if single else v


def expval_state(circuit: Circuit, ham: PauliHamiltonian, theta, state, *, want_grad: bool = True,
                 dtype: str = "complex128", device=None):
    """<state|U(theta)^H H U(theta)|state> and its exact gradient for an ARBITRARY input train
    (a reference TTState's cores, tt.py:38-76, or a truncated.GPUTrain): the reference's expval on
    any TTState (hamiltonians.py:167-187) with the circuit applied first.  Runs the taped
    truncated engine from that train with eps = 0 and no bond cap, where every split keeps a
    square unitary factor, so the frozen-constant shift rule is the exact gradient
    (autodiff.py:8-13; truncated.straight_through).  Bonds above 32 raise BondTooLarge.

    1-D theta -> (float, float64[P] | None); 2-D [B, P] -> (float64[B], float64[B, P] | None)."""
    from . import truncated as TR

    arr, single = _check_theta(circuit, theta)
    terms = _terms(ham, circuit.n_qubits)
    train = state if isinstance(state, TR.GPUTrain) else TR.GPUTrain.from_cores(
        list(getattr(state, "cores", state)), dtype=dtype, device=_device(device))
    vals, grad = TR.straight_through(circuit, terms, arr, 0.0, None, dtype=dtype, device=device,
                                     want_grad=want_grad, init=train.row(0) if train.batch > 1 else train)
    e = vals @ np.array([c for c, _ in terms], dtype=complex) if terms else np.zeros(arr.shape[0], complex)
    if not (np.all(np.isfinite(e)) and (grad is None or np.all(np.isfinite(grad)))):
        from .errors import NotFinite
        raise NotFinite("engine produced NaN or Inf")
    tol = E.residue_tol(dtype, sum(abs(c) for c, _ in terms))
    if e.size and float(np.max(np.abs(e.imag))) > tol:
        from .errors import NonHermitianResidue
        raise NonHermitianResidue(f"imaginary residue {float(np.max(np.abs(e.imag))):.3e} exceeds {tol:.0e}")
    if single:
        return float(e.real[0]), (None if grad is None else grad[0])
    return e.real, grad


def expectation_values(circuit: Circuit, theta, op_groups, engine: str = "tt", eps: float = 0.0, chi_max=None, *,
                       dtype: str = "complex64", device=None, segments=None):
    """Complex <P> per op-group sharing one state per theta-set (the values of
    reference taped_expectations, autodiff.py:405-425).  op_groups: dicts {qubit: letter}.
    With a truncation that cuts the reference's tape (eps > 0, or chi_max below its taped bonds)
    the values come from the taped truncated state, as the reference's do (complex128)."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    arr, single = _check_theta(circuit, theta)
    n = circuit.n_qubits
    from .hamiltonians import PauliTerm

    terms = []
    for ops in op_groups:
        for q, letter in dict(ops).items():
            if letter not in PAULI_MATRICES:
                raise InputError(f"unknown Pauli letter {letter!r}")
            if not 0 <= int(q) < n:
                raise WireOutOfRange(f"qubit {q} outside 0..{n - 1}")
        terms.append(PauliTerm(1.0, tuple(dict(ops).items())))
    ham_terms = C.normalize_terms(PauliHamiltonian(n, tuple(terms)))
    if _truncating(circuit, eps, chi_max) or _taped_truncates(circuit, eps, chi_max):
        from . import truncated as TR

        vals, _ = TR.straight_through(circuit, ham_terms, arr, eps, chi_max, dtype="complex128", device=device,
                                      want_grad=False)
        return vals[0] if single else vals
    dev = _device(device)
    dp = E.device_plan(circuit, ham_terms, "values", arr.shape[0], dev, segments, dtype=dtype)
    th = torch.tensor(arr, dtype=E.DTYPES[dtype][1], device=dev)
    vals = E.values_raw(dp, th, dtype).cpu().numpy()
    return vals[0] if single else vals


def parameter_shift_grad(circuit: Circuit, ham: PauliHamiltonian, theta, engine: str = "tt", eps: float = 0.0,
                         chi_max=None, *, coords=None, dtype: str = "complex64", device=None):
    """Exact shift-rule gradient (reference autodiff.py:514-550), all shifted angle
    sets evaluated in ONE batched forward launch."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    arr, _ = _check_theta(circuit, theta)
    th = arr[0]
    names = [circuit.gates[g].name for g in circuit.trainable]
    for name in names:
        if name not in SHIFTABLE_GATES:
            raise UnsupportedGateForShift(f"no shift rule for gate {name!r}")
    ks = list(range(len(th))) if coords is None else [int(k) for k in coords]
    rows, plan_rows = [], []
    for k in ks:
        shifts = (np.pi / 2, -np.pi / 2, 3 * np.pi / 2, -3 * np.pi / 2) if names[k] == "crz" else (np.pi / 2, -np.pi / 2)
        idx = []
        for d in shifts:
            t = th.copy()
            t[k] += d
            idx.append(len(rows))
            rows.append(t)
        plan_rows.append((k, idx))
    grad = np.zeros(len(th))
    if not rows:
        return grad
    e = np.atleast_1d(evaluate_expval(circuit, ham, np.array(rows), eps=eps, chi_max=chi_max, dtype=dtype,
                                      device=device))
    for k, idx in plan_rows:
        if names[k] == "crz":
            grad[k] = _CRZ_Y1 * (e[idx[0]] - e[idx[1]]) - _CRZ_Y2 * (e[idx[2]] - e[idx[3]])
        else:
            grad[k] = 0.5 * (e[idx[0]] - e[idx[1]])
    return grad


def finite_diff_grad(circuit: Circuit, ham: PauliHamiltonian, theta, step: float = 1e-5, engine: str = "tt",
                     eps: float = 0.0, chi_max=None, *, dtype: str = "complex128", device=None):
    """Central differences (reference autodiff.py:553-576), batched into one launch."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    if step <= 0:
        raise InputError(f"step must be positive, got {step}")
    arr, _ = _check_theta(circuit, theta)
    th = arr[0]
    rows = []
    for k in range(len(th)):
        up, dn = th.copy(), th.copy()
        up[k] += step
        dn[k] -= step
        rows += [up, dn]
    if not rows:
        return np.zeros(0)
    e = np.atleast_1d(evaluate_expval(circuit, ham, np.array(rows), eps=eps, chi_max=chi_max, dtype=dtype,
                                      device=device))
    return (e[0::2] - e[1::2]) / (2 * step)


# --------------------------------------------------------------------------- optimisation
@dataclass(frozen=True)
class MinimizeStep:
    iteration: int
    theta: np.ndarray
    value: float
    grad_norm: float


@dataclass(frozen=True)
class MinimizeResult:
    steps: tuple
    converged: bool

    @property
    def theta(self):
        return self.steps[-1].theta

    @property
    def value(self):
        return self.steps[-1].value

    @property
    def n_iters(self):
        return self.steps[-1].iteration


def init_params(n_params: int, rng) -> np.ndarray:
    """Uniform angles in [-pi, pi) (reference autodiff.py:609-611)."""
    return rng.uniform(-np.pi, np.pi, size=int(n_params))


def minimize(fun, theta0, optimizer: str = "gd", rate: float = 0.05, max_iters: int = 200, tol: float = 1e-8,
             betas=(0.9, 0.999), adam_eps: float = 1e-8) -> MinimizeResult:
    """Fixed-rate descent on fun(theta) -> (value, grad) (reference autodiff.py:614-659)."""
    if optimizer not in ("gd", "adam"):
        raise InputError(f"unknown optimizer {optimizer!r}")
    theta = np.asarray(theta0, dtype=float).reshape(-1).copy()
    if theta.size and not np.all(np.isfinite(theta)):
        raise InputError("initial parameters must be finite")
    steps = []
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    for it in range(max_iters + 1):
        value, grad = fun(theta)
        value = float(value)
        grad = np.asarray(grad, dtype=float).reshape(-1)
        if not np.isfinite(value) or not np.all(np.isfinite(grad)):
            raise DivergenceDetected(f"non-finite objective at iteration {it}")
        gnorm = float(np.linalg.norm(grad))
        steps.append(MinimizeStep(it, theta.copy(), value, gnorm))
        if gnorm < tol:
            return MinimizeResult(tuple(steps), True)
        if it == max_iters:
            break
        if optimizer == "gd":
            theta = theta - rate * grad
        else:
            b1, b2 = betas
            m = b1 * m + (1 - b1) * grad
            v = b2 * v + (1 - b2) * grad * grad
            mhat = m / (1 - b1 ** (it + 1))
            vhat = v / (1 - b2 ** (it + 1))
            theta = theta - rate * mhat / (np.sqrt(vhat) + adam_eps)
    return MinimizeResult(tuple(steps), False)


def state_inner_product(ket_circuit: Circuit, ket_theta, bra_circuit: Circuit | None = None, bra_theta=None, *,
                        ket_init=None, bra_init=None, dtype: str = "complex64", device=None):
    """<bra|ket> with |ket> = U_ket(theta)|ket_init>, |bra> = U_bra(theta')|bra_init>
    (the first argument of the reference's tt_inner is conjugated, tt.py:247-255).

    ``bra_circuit=None`` means no gates on the bra side (a product state, e.g. tlquantum's
    ``state_inner_product(state, compare_state)`` = <compare|U|state>).  Init vectors are
    per-qubit complex 2-vectors (default |0>).  theta may be batched [B, P]."""
    n = ket_circuit.n_qubits
    bra_circuit = bra_circuit if bra_circuit is not None else Circuit(n, (), ())
    if bra_circuit.n_qubits != n:
        from .errors import SizeMismatch
        raise SizeMismatch(f"{bra_circuit.n_qubits} vs {n} qubits")
    tk, single = _check_theta(ket_circuit, ket_theta)
    tb, _ = _check_theta(bra_circuit, np.zeros((tk.shape[0], 0)) if bra_theta is None else bra_theta)
    if tb.shape[0] == 1 and tk.shape[0] > 1:
        tb = np.repeat(tb, tk.shape[0], axis=0)
    dev = _device(device)
    limit = C.MAX_CHI if dtype == "complex64" else C.MAX_CHI_F64

    def plan(circ, init):
        key_terms = []
        return E.device_plan(circ, key_terms, "state", 1, dev, 1, init=init, dtype=dtype)

    dk, db = plan(ket_circuit, ket_init), plan(bra_circuit, bra_init)
    tdt = E.DTYPES[dtype][1]
    out = E.inner_raw(db, torch.tensor(tb, dtype=tdt, device=dev), dk, torch.tensor(tk, dtype=tdt, device=dev),
                      dtype).cpu().numpy()
    return complex(out[0]) if single else out


# --------------------------------------------------------------------------- differentiable inner product
class InnerFunction(torch.autograd.Function):
    """z_b = <bra(theta_bra_b)|ket(theta_ket_b)> (complex128 [B]) with exact gradients.

    Every trainable gate is C + A cos(t/2) + B sin(t/2) (rx, ry, rz, crz), and z is linear in
    each gate of either side.  Hence dz/dt = (z(t + pi) - z(t - pi)) / 4, exactly.  The
    backward evaluates all 2P shifted angle sets of the batch in ONE tq_inner launch.  The
    forward value is the kernel's; there is no tape (reference tt_inner, tt.py:247-255)."""

    @staticmethod
    def forward(ctx, theta_ket, theta_bra, dk, db, dtype):
        ctx.save_for_backward(theta_ket, theta_bra)
        ctx.dk, ctx.db, ctx.dtype = dk, db, dtype
        return E.inner_raw(db, theta_bra.detach(), dk, theta_ket.detach(), dtype)

    @staticmethod
    def backward(ctx, gz):
        theta_ket, theta_bra = ctx.saved_tensors
        gk = gb = None

        def shifted_grad(th, other, ket_side):
            B, P = th.shape
            if P == 0:
                return torch.zeros_like(th)
            eye = torch.eye(P, dtype=th.dtype, device=th.device) * np.pi
            rows = torch.cat([th[:, None, :] + eye[None], th[:, None, :] - eye[None]], dim=1).reshape(B * 2 * P, P)
            oth = other.repeat_interleave(2 * P, dim=0)
            if ket_side:
                z = E.inner_raw(ctx.db, oth, ctx.dk, rows, ctx.dtype)
            else:
                z = E.inner_raw(ctx.db, rows, ctx.dk, oth, ctx.dtype)
            z = z.reshape(B, 2, P)
            dz = (z[:, 0] - z[:, 1]) / 4.0
            return (torch.conj(gz)[:, None] * dz).real.to(th.dtype)

        if ctx.needs_input_grad[0]:
            gk = shifted_grad(theta_ket.detach(), theta_bra.detach(), True)
        if ctx.needs_input_grad[1]:
            gb = shifted_grad(theta_bra.detach(), theta_ket.detach(), False)
        return gk, gb, None, None, None


def inner(ket_circuit: Circuit, theta_ket: torch.Tensor, bra_circuit: Circuit | None = None,
          theta_bra: torch.Tensor | None = None, *, ket_init=None, bra_init=None,
          dtype: str = "complex128") -> torch.Tensor:
    """Torch-native, differentiable <bra|ket> (complex128 [B]) for device angle tensors
    theta_ket [B, Pk] (and theta_bra [B, Pb]); gradients flow to both sides."""
    n = ket_circuit.n_qubits
    bra_circuit = bra_circuit if bra_circuit is not None else Circuit(n, (), ())
    for circ in (ket_circuit, bra_circuit):
        for g in circ.trainable:
            if circ.gates[g].name not in SHIFTABLE_GATES:
                raise UnsupportedGateForShift(f"no shift rule for gate {circ.gates[g].name!r}")
    if theta_ket.dim() == 1:
        theta_ket = theta_ket[None]
    B = theta_ket.shape[0]
    dev = theta_ket.device
    if theta_bra is None:
        theta_bra = torch.zeros(B, bra_circuit.n_params, dtype=theta_ket.dtype, device=dev)
    if theta_bra.dim() == 1:
        theta_bra = theta_bra[None]
    if theta_bra.shape[0] == 1 and B > 1:
        theta_bra = theta_bra.expand(B, -1)
    tdt = E.DTYPES[dtype][1]
    dk = E.device_plan(ket_circuit, [], "state", 1, dev, 1, init=ket_init, dtype=dtype)
    db = E.device_plan(bra_circuit, [], "state", 1, dev, 1, init=bra_init, dtype=dtype)
    return InnerFunction.apply(theta_ket.to(tdt), theta_bra.to(tdt), dk, db, dtype)
