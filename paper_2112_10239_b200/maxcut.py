"""MaxCut through the multi-basis encoding (MBE), on the B200 engine.

Mirrors ``tnsim.maxcut`` (reference ``maxcut.py:39-319``).  Vertex 2k is read out
as <Z_k>, vertex 2k+1 as <X_k> (single-site readouts, ``maxcut.py:127-135``); the
relaxed loss is ``L = sum_(u,v,w) w tanh(a<s_u>) tanh(a<s_v>)`` (``maxcut.py:219-252``).

Device path per optimiser step, for B restarts at once (the reference's thread
pool over restarts, ``maxcut.py:309-313``, becomes the batch dimension):
  values sweep   -> readouts r[B, V]                     (tq_term_values)
  torch          -> t = tanh(a r), loss, cotangents g_v = a (1 - t_v^2) sum_nbr w t_u
  energy sweep   -> grad[B, P] with per-restart coefficients g (tq_energy_grad)
  torch          -> Adam update (reference autodiff.py:650-658)
Neighbour sums use padded adjacency lists (gather + fixed-order sum, no atomics),
so results are bit-identical run to run.  Final readouts for the sign rounding use
the complex128 kernels so cuts are bit-exact whenever the readout margin exceeds 1e-9.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import chain as C
from . import engine as E
from .autodiff import _check_engine, _device, _engine_args, _taped_truncates, _truncating, init_params
from .circuits import Circuit, standard_gate
from .errors import (
    DivergenceDetected,
    DuplicateEdge,
    InputError,
    InvalidLabel,
    ParamCountMismatch,
    ParseError,
    SelfLoop,
    SizeMismatch,
    TooManyVertices,
)
from .hamiltonians import PauliHamiltonian, PauliTerm
from .seeding import spawn

MAX_BRUTE_FORCE_VERTICES = 22


@dataclass(frozen=True)
class Graph:
    """Undirected weighted graph on vertices 0..num_vertices-1 (reference maxcut.py:39-79)."""

    num_vertices: int
    edges: tuple = ()

    def __post_init__(self):
        if isinstance(self.num_vertices, bool) or not isinstance(self.num_vertices, (int, np.integer)):
            raise InputError("num_vertices must be an integer")
        if self.num_vertices < 0:
            raise InputError("num_vertices must be non-negative")
        out, seen = [], set()
        for e in self.edges:
            if len(e) != 3:
                raise InputError(f"edge {e!r} is not a (u, v, weight) triple")
            u, v, w = e
            if isinstance(u, bool) or isinstance(v, bool) or not isinstance(u, (int, np.integer)) \
                    or not isinstance(v, (int, np.integer)):
                raise InvalidLabel("vertex labels must be integers")
            u, v, w = int(u), int(v), float(w)
            if not (0 <= u < self.num_vertices and 0 <= v < self.num_vertices):
                raise InvalidLabel(f"edge ({u}, {v}) references a vertex outside 0..{self.num_vertices - 1}")
            if u == v:
                raise SelfLoop(f"vertex {u} connected to itself")
            if not math.isfinite(w):
                raise InputError(f"edge ({u}, {v}) has non-finite weight")
            key = (min(u, v), max(u, v))
            if key in seen:
                raise DuplicateEdge(f"edge ({u}, {v}) listed twice")
            seen.add(key)
            out.append((u, v, w))
        object.__setattr__(self, "num_vertices", int(self.num_vertices))
        object.__setattr__(self, "edges", tuple(out))

    @property
    def total_abs_weight(self) -> float:
        return float(sum(abs(w) for _, _, w in self.edges))


def load_graph(text: str) -> Graph:
    """Edge-list parser (reference maxcut.py:82-124)."""
    header, raw, first = None, [], True
    for lineno, line in enumerate(text.splitlines(), start=1):
        body = line.split("#", 1)[0].strip()
        if not body:
            continue
        fields = body.split()
        if first and len(fields) == 1:
            try:
                header = int(fields[0])
            except ValueError:
                raise ParseError(f"line {lineno}: expected an integer header, got {body!r}")
            if header < 0:
                raise ParseError(f"line {lineno}: vertex count must be non-negative")
            first = False
            continue
        first = False
        if len(fields) not in (2, 3):
            raise ParseError(f"line {lineno}: expected 'u v [w]', got {body!r}")
        try:
            u, v = int(fields[0]), int(fields[1])
        except ValueError:
            raise ParseError(f"line {lineno}: vertex labels must be integers, got {body!r}")
        if u < 0 or v < 0:
            raise ParseError(f"line {lineno}: vertex labels must be non-negative")
        w = 1.0
        if len(fields) == 3:
            try:
                w = float(fields[2])
            except ValueError:
                raise ParseError(f"line {lineno}: weight must be a number, got {fields[2]!r}")
        raw.append((u, v, w))
    n = header if header is not None else (1 + max(max(u, v) for u, v, _ in raw) if raw else 0)
    return Graph(n, tuple(raw))


def pairing_graph(num_vertices: int, degree: int, rng) -> Graph:
    """Random simple d-regular graph by the pairing model (SURVEY.md section 8d cfg3 spec)."""
    while True:
        stubs = np.repeat(np.arange(num_vertices), degree)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        keys = {(min(u, v), max(u, v)) for u, v in pairs}
        if all(u != v for u, v in pairs) and len(keys) == len(pairs):
            return Graph(num_vertices, tuple((int(u), int(v), 1.0) for u, v in pairs))


def mbe_encode(graph: Graph):
    """(n_qubits, [(qubit, 'Z'|'X') per vertex]) (reference maxcut.py:127-135)."""
    n = (graph.num_vertices + 1) // 2
    return n, tuple((v // 2, "Z" if v % 2 == 0 else "X") for v in range(graph.num_vertices))


def mbe_loss(t_vals, graph: Graph) -> float:
    """Reference maxcut.py:138-145."""
    t = np.asarray(t_vals, dtype=float).reshape(-1)
    if t.size != graph.num_vertices:
        raise SizeMismatch(f"{t.size} values supplied for a graph with {graph.num_vertices} vertices")
    return float(sum(w * t[u] * t[v] for u, v, w in graph.edges))


def round_cut(expectations) -> tuple:
    """Sign rounding, 0 -> +1 (reference maxcut.py:148-153)."""
    x = np.asarray(expectations, dtype=float).reshape(-1)
    if x.size and not np.all(np.isfinite(x)):
        raise InputError("expectations must be finite")
    return tuple(1 if v >= 0 else -1 for v in x)


def cut_value(graph: Graph, assignment) -> float:
    """Reference maxcut.py:156-164."""
    a = np.asarray(assignment).reshape(-1)
    if a.size != graph.num_vertices:
        raise SizeMismatch(f"assignment length {a.size} does not match {graph.num_vertices} vertices")
    if not all(v in (-1, 1) for v in a.tolist()):
        raise InvalidLabel("assignment entries must be +1 or -1")
    return float(sum(w * (1 - int(a[u]) * int(a[v])) / 2 for u, v, w in graph.edges))


def brute_force_maxcut(graph: Graph):
    """Exhaustive optimum with vertex 0 fixed (reference maxcut.py:167-183); V <= 22."""
    nv = graph.num_vertices
    if nv > MAX_BRUTE_FORCE_VERTICES:
        raise TooManyVertices(f"{nv} vertices exceeds the brute-force limit of {MAX_BRUTE_FORCE_VERTICES}")
    if nv == 0:
        return 0.0, ()
    pats = np.arange(1 << (nv - 1), dtype=np.uint32)
    cuts = np.zeros(pats.shape)
    for u, v, w in graph.edges:
        bu = (pats >> (u - 1)) & 1 if u > 0 else np.zeros_like(pats)
        bv = (pats >> (v - 1)) & 1 if v > 0 else np.zeros_like(pats)
        cuts += w * (bu ^ bv)
    best = int(np.argmax(cuts))
    return float(cuts[best]), (1,) + tuple(-1 if (best >> (v - 1)) & 1 else 1 for v in range(1, nv))


def brickwork_ansatz(n_qubits: int, depth: int = 4) -> Circuit:
    """ry+rz rows separated by cz lines with alternating offset (reference maxcut.py:186-203)."""
    if n_qubits < 1:
        raise InputError("ansatz needs at least one qubit")
    if depth < 1:
        raise InputError("depth must be at least 1")
    gates, train = [], []
    for layer in range(depth):
        for name in ("ry", "rz"):
            for q in range(n_qubits):
                train.append(len(gates))
                gates.append(standard_gate(name, (q,), 0.0))
        if layer < depth - 1:
            for q in range(layer % 2, n_qubits - 1, 2):
                gates.append(standard_gate("cz", (q, q + 1)))
    return Circuit(n_qubits, tuple(gates), tuple(train))


def _readout_terms(graph: Graph):
    n, mapping = mbe_encode(graph)
    return n, PauliHamiltonian(max(n, 1), tuple(PauliTerm(1.0, ((q, letter),)) for q, letter in mapping))


class MBEObjective:
    """Batched device objective: theta [B, P] -> (loss [B], grad [B, P]) on the GPU."""

    def __init__(self, circuit: Circuit, graph: Graph, alpha: float = 1.0, *, dtype: str = "complex64",
                 device=None, batch: int = 1, segments=None):
        n, ham = _readout_terms(graph)
        if circuit.n_qubits != n:
            raise SizeMismatch(f"circuit has {circuit.n_qubits} qubits, encoding needs {n}")
        if not math.isfinite(alpha) or alpha <= 0:
            raise InputError("alpha must be positive and finite")
        self.circuit, self.graph, self.alpha, self.dtype = circuit, graph, float(alpha), dtype
        self.device = _device(device)
        terms = C.normalize_terms(ham)
        self.dp_values = E.device_plan(circuit, terms, "values", batch, self.device, segments, dtype=dtype)
        self.dp_energy = E.device_plan(circuit, terms, "energy", batch, self.device, segments, dtype=dtype)
        V = graph.num_vertices
        deg = np.zeros(V, dtype=np.int64)
        for u, v, _ in graph.edges:
            deg[u] += 1
            deg[v] += 1
        md = int(deg.max()) if V and len(graph.edges) else 1
        nbr = np.full((V, md), V, dtype=np.int64)   # index V = padding slot holding t = 0
        wts = np.zeros((V, md))
        fill = np.zeros(V, dtype=np.int64)
        for u, v, w in graph.edges:
            nbr[u, fill[u]], wts[u, fill[u]] = v, w
            nbr[v, fill[v]], wts[v, fill[v]] = u, w
            fill[u] += 1
            fill[v] += 1
        tdt = E.DTYPES[dtype][1]
        self.nbr = torch.tensor(nbr, device=self.device)
        self.wts = torch.tensor(wts, dtype=torch.float64, device=self.device)
        eu = np.array([e[0] for e in graph.edges], dtype=np.int64)
        ev = np.array([e[1] for e in graph.edges], dtype=np.int64)
        self.eu = torch.tensor(eu, device=self.device)
        self.ev = torch.tensor(ev, device=self.device)
        self.ew = torch.tensor([e[2] for e in graph.edges], dtype=torch.float64, device=self.device)
        self.tdt = tdt
        self._ws = {}

    def _scratch(self, key, dp, batch, values):
        """This objective's own workspaces (captured graphs bake the pointer in: an AdamGraph and
        an mbe_objective graph over the same plans must not share scratch)."""
        need = E.workspace_bytes(dp, batch, True, self.dtype, values=values)
        buf = self._ws.get(key)
        if buf is None or buf.numel() < need:
            buf = self._ws[key] = torch.empty(need, dtype=torch.uint8, device=self.device)
        return buf

    def readouts(self, theta: torch.Tensor, dtype: str | None = None) -> torch.Tensor:
        """Re<sigma_v> [B, V] (float64)."""
        dt = dtype or self.dtype
        dp = self.dp_values if dt == self.dtype else E.device_plan(
            self.circuit, C.normalize_terms(_readout_terms(self.graph)[1]), "values", theta.shape[0],
            self.device, None, dtype=dt)
        ws = self._scratch(("v", theta.shape[0]), dp, theta.shape[0], True) if dp is self.dp_values else None
        return E.values_raw(dp, theta, dt, ws=ws).real

    def host_evaluator(self, batch: int) -> "_HostEvaluator":
        """fun(theta [batch, P] numpy) -> (loss [batch], grad [batch, P]) numpy, one captured
        device round trip per call (the batched form of ``mbe_objective``'s fun)."""
        return _HostEvaluator(self, batch)

    def __call__(self, theta: torch.Tensor):
        r = self.readouts(theta)                                  # [B, V] float64
        t = torch.tanh(self.alpha * r)
        loss = (self.ew * t[:, self.eu] * t[:, self.ev]).sum(dim=1)
        tp = torch.cat([t, torch.zeros(t.shape[0], 1, dtype=t.dtype, device=t.device)], dim=1)
        nsum = (tp[:, self.nbr] * self.wts).sum(dim=2)             # sum_nbr w t_u   [B, V]
        g = self.alpha * (1.0 - t * t) * nsum
        ws = self._scratch(("e", theta.shape[0]), self.dp_energy, theta.shape[0], False)
        _, grad = E.energy_grad_raw(self.dp_energy, theta, g, True, self.dtype, ws=ws)
        return loss, grad


class _HostEvaluator:
    """Host-buffer serving path of an ``MBEObjective`` for a fixed batch B: pinned theta [B, P]
    -> device, readout sweeps, tanh loss, gradient sweeps, loss and gradient -> pinned host.
    The first call runs eagerly; the second captures the whole evaluation as one CUDA graph
    that every later call replays.  The reference hands one ``fun`` to a thread pool
    (maxcut.py:309-313): the staging buffers and the captured graph are shared, so one call
    runs at a time."""

    def __init__(self, obj: "MBEObjective", batch: int):
        P = obj.circuit.n_params
        self.obj, self.batch, self.P = obj, int(batch), P
        self.th_host = torch.empty(batch, P, dtype=torch.float64, pin_memory=True)
        self.out_host = torch.empty(batch, P + 1, dtype=torch.float64, pin_memory=True)
        self.th_dev = torch.empty(batch, P, dtype=torch.float64, device=obj.device)
        self.calls, self.graph = 0, None
        self.lock = threading.Lock()

    @property
    def h2d_bytes(self) -> int:
        return self.th_host.numel() * 8

    @property
    def d2h_bytes(self) -> int:
        return self.out_host.numel() * 8

    def _body(self):
        self.th_dev.copy_(self.th_host, non_blocking=True)
        loss, grad = self.obj(self.th_dev.to(self.obj.tdt))
        self.out_host.copy_(torch.cat([loss.reshape(-1, 1).double(), grad.double()], dim=1), non_blocking=True)

    def __call__(self, theta):
        th = np.asarray(theta, dtype=float)
        if th.ndim != 2 or th.shape[0] != self.batch:
            raise SizeMismatch(f"expected theta of shape ({self.batch}, {self.P}), got {th.shape}")
        if th.shape[1] != self.P:
            raise ParamCountMismatch(f"expected {self.P} parameters, got {th.shape[1]}")
        if not np.all(np.isfinite(th)):
            raise InputError("theta contains non-finite values")
        with self.lock:
            self.th_host.numpy()[:] = th
            dev = self.obj.device
            if self.graph is None and self.calls >= 1:
                side = torch.cuda.Stream(device=dev)
                side.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(side):
                    self._body()
                torch.cuda.current_stream(dev).wait_stream(side)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="relaxed"):
                    self._body()
                self.graph = g
            self.calls += 1
            if self.graph is not None:
                self.graph.replay()
            else:
                self._body()
            torch.cuda.current_stream(dev).synchronize()
            out = self.out_host.numpy().copy()
        return out[:, 0], out[:, 1:]


def _truncation(engine, circuit, eps, chi_max):
    """(eps, chi_max, truncating) of an MBE entry point after the engine seam.  A truncating run
    follows the reference's taped truncated path (taped_expectations with eps / chi_max,
    autodiff.py:405-425): readouts of the taped state, straight-through gradients
    (truncated.straight_through)."""
    eps, chi_max = _engine_args(engine, circuit, eps, chi_max)
    return eps, chi_max, _truncating(circuit, eps, chi_max) or _taped_truncates(circuit, eps, chi_max)


def _edge_loss_and_cotangents(graph: Graph, alpha: float, r: np.ndarray):
    """L = sum w tanh(a r_u) tanh(a r_v) and dL/dr_u = a (1 - t_u^2) sum_(u,v,w) w t_v (host, float64)."""
    t = np.tanh(alpha * r)
    loss = sum(w * t[u] * t[v] for u, v, w in graph.edges)
    g = np.zeros_like(r)
    for u, v, w in graph.edges:
        g[u] += w * t[v]
        g[v] += w * t[u]
    return float(loss), alpha * (1.0 - t * t) * g


def vertex_expectations(circuit: Circuit, theta, graph: Graph, engine: str = "tt", eps: float = 0.0,
                        chi_max=None, *, dtype: str = "complex128", device=None):
    """Per-vertex readouts (reference maxcut.py:206-216); complex128 by default for exact rounding."""
    eps, chi_max, trunc = _truncation(engine, circuit, eps, chi_max)
    n, ham = _readout_terms(graph)
    if circuit.n_qubits != n:
        raise SizeMismatch(f"circuit has {circuit.n_qubits} qubits, encoding needs {n}")
    th = np.asarray(theta, dtype=float)
    single = th.ndim == 1
    th2 = th.reshape(1, -1) if single else th
    if trunc:   # readouts of the taped truncated state
        from . import truncated as TR

        vals, _ = TR.straight_through(circuit, C.normalize_terms(ham), th2, eps, chi_max, dtype="complex128",
                                      device=device, want_grad=False)
        return vals.real[0] if single else vals.real
    dev = _device(device)
    dp = E.device_plan(circuit, C.normalize_terms(ham), "values", th2.shape[0], dev, None, dtype=dtype)
    vals = E.values_raw(dp, torch.tensor(th2, dtype=E.DTYPES[dtype][1], device=dev), dtype).real.cpu().numpy()
    return vals[0] if single else vals


def mbe_objective(circuit: Circuit, graph: Graph, alpha: float = 1.0, engine: str = "tt", eps: float = 0.0,
                  chi_max=None, *, dtype: str = "complex128", device=None):
    """fun(theta) -> (loss, grad) (reference maxcut.py:219-252), one device round trip per call.
    complex128 by default, like the reference; ``dtype="complex64"`` is the fast path."""
    eps, chi_max, trunc = _truncation(engine, circuit, eps, chi_max)
    if trunc:
        return _mbe_objective_truncated(circuit, graph, alpha, eps, chi_max, device)
    obj = MBEObjective(circuit, graph, alpha, dtype=dtype, device=device)
    call = obj.host_evaluator(1)

    def fun(theta):
        th = np.asarray(theta, dtype=float).reshape(-1)
        loss, grad = call(th.reshape(1, -1))
        return float(loss[0]), grad[0]

    return fun


def _mbe_objective_truncated(circuit: Circuit, graph: Graph, alpha: float, eps: float, chi_max, device):
    """The reference's truncated MBE objective: readouts of the taped truncated state and the
    straight-through gradient of the edge loss through them (the reference's one tape,
    maxcut.py:219-252): the cotangents dL/dr_u weight the frozen-constant replays."""
    from . import truncated as TR

    n, ham = _readout_terms(graph)
    if circuit.n_qubits != n:
        raise SizeMismatch(f"circuit has {circuit.n_qubits} qubits, encoding needs {n}")
    if not math.isfinite(alpha) or alpha <= 0:
        raise InputError("alpha must be positive and finite")
    terms = C.normalize_terms(ham)
    P = circuit.n_params

    def fun(theta):
        th = np.asarray(theta, dtype=float).reshape(-1)
        if th.shape[0] != P:
            raise ParamCountMismatch(f"expected {P} parameters, got {th.shape[0]}")
        if not np.all(np.isfinite(th)):
            raise InputError("theta contains non-finite values")
        out = {}

        def weights(vals):
            loss, g = _edge_loss_and_cotangents(graph, alpha, vals.real[0])
            out["loss"] = loss
            return g[None, :]

        _, grad = TR.straight_through(circuit, terms, th[None], eps, chi_max, dtype="complex128", device=device,
                                      weights=weights)
        return out["loss"], grad[0]

    return fun


@dataclass(frozen=True)
class MbeResult:
    assignment: tuple
    cut_value: float
    relaxed_loss: float
    iterations: int
    restart_index: int
    seed: int


class AdamGraph:
    """One optimiser iteration of every restart as a replayable CUDA graph: the readout sweeps,
    tanh loss and cotangents, the gradient sweeps, the convergence mask and the Adam/GD update,
    all in place on device tensors.  The host only replays, and inspects the flags every
    ``check_every`` iterations.

    The semantics are those of the reference's ``minimize``, run once per restart
    (autodiff.py:614-659):
    - each restart freezes when its gradient norm drops below ``tol``;
    - the final iteration evaluates without updating;
    - the first non-finite loss or gradient raises ``DivergenceDetected`` with its iteration."""

    def __init__(self, obj: MBEObjective, theta0: np.ndarray, rate: float, max_iters: int, tol: float = 1e-8,
                 betas=(0.9, 0.999), adam_eps: float = 1e-8, optimizer: str = "adam"):
        dev = obj.device
        self.obj, self.rate, self.max_iters, self.tol = obj, float(rate), int(max_iters), float(tol)
        self.b1, self.b2, self.adam_eps, self.optimizer = float(betas[0]), float(betas[1]), float(adam_eps), optimizer
        self.theta = torch.tensor(theta0, dtype=torch.float64, device=dev)
        B = self.theta.shape[0]
        self.m = torch.zeros_like(self.theta)
        self.v = torch.zeros_like(self.theta)
        self.active = torch.ones(B, dtype=torch.bool, device=dev)
        self.value = torch.zeros(B, dtype=torch.float64, device=dev)
        self.iters = torch.zeros(B, dtype=torch.int64, device=dev)
        self.it = torch.zeros((), dtype=torch.int64, device=dev)
        self.bad = torch.full((), -1, dtype=torch.int64, device=dev)
        self.graph = None

    def _iteration(self):
        o = self.obj
        loss, grad = o(self.theta.to(o.tdt))
        grad = grad.double()
        finite = torch.isfinite(loss).all() & torch.isfinite(grad).all()
        self.bad.copy_(torch.where(~finite & (self.bad < 0), self.it, self.bad))
        self.value.copy_(torch.where(self.active, loss, self.value))
        self.iters.copy_(torch.where(self.active, self.it.expand_as(self.iters), self.iters))
        gnorm = torch.linalg.vector_norm(grad, dim=1)
        self.active.copy_(self.active & (gnorm >= self.tol))
        upd_mask = (self.active & (self.it < self.max_iters))[:, None]
        if self.optimizer == "gd":
            upd = self.rate * grad
        else:
            self.m.copy_(torch.where(upd_mask, self.b1 * self.m + (1 - self.b1) * grad, self.m))
            self.v.copy_(torch.where(upd_mask, self.b2 * self.v + (1 - self.b2) * grad * grad, self.v))
            step = (self.it + 1).to(torch.float64)
            mhat = self.m / (1 - torch.pow(self.b1, step))
            vhat = self.v / (1 - torch.pow(self.b2, step))
            upd = self.rate * mhat / (torch.sqrt(vhat) + self.adam_eps)
        self.theta.copy_(torch.where(upd_mask, self.theta - upd, self.theta))
        self.it.add_(1)

    def capture(self):
        """Warm up outside the graph (plans, workspaces, kernel attributes), restore the state,
        then capture one iteration."""
        saved = [t.clone() for t in (self.theta, self.m, self.v, self.active, self.value, self.iters, self.it, self.bad)]
        side = torch.cuda.Stream(device=self.obj.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._iteration()
        torch.cuda.current_stream().wait_stream(side)
        for t, s0 in zip((self.theta, self.m, self.v, self.active, self.value, self.iters, self.it, self.bad), saved):
            t.copy_(s0)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self._iteration()
        torch.cuda.synchronize()
        return self

    def run(self, check_every: int = 16):
        if self.graph is None:
            self.capture()
        done = 0
        while done < self.max_iters + 1:
            n = min(check_every, self.max_iters + 1 - done)
            for _ in range(n):
                self.graph.replay()
            done += n
            bad = int(self.bad.item())
            if bad >= 0:
                raise DivergenceDetected(f"non-finite objective at iteration {bad}")
            if not bool(self.active.any()):
                break
        return self.theta.cpu().numpy(), self.value.cpu().numpy(), self.iters.cpu().numpy()


def adam_batched(obj: MBEObjective, theta0: np.ndarray, rate: float, max_iters: int, tol: float = 1e-8,
                 betas=(0.9, 0.999), adam_eps: float = 1e-8, optimizer: str = "adam"):
    """Per-restart minimise (reference autodiff.py:614-659) with restarts as the batch.

    Each restart stops on its own when its gradient norm drops below ``tol`` (frozen
    thereafter), exactly like independent reference runs.  The iterations replay one captured
    CUDA graph (``AdamGraph``)."""
    return AdamGraph(obj, theta0, rate, max_iters, tol, betas, adam_eps, optimizer).run()


def solve_maxcut(graph: Graph, depth: int = 4, engine: str = "tt", eps: float = 0.0, chi_max=None,
                 optimizer: str = "adam", rate: float = 0.1, restarts: int = 5, max_iters: int = 300,
                 seed: int = 0, alpha: float = 1.0, threads: int = 1, *, dtype: str = "complex128", device=None):
    """Train the brickwork ansatz, round to a cut (reference maxcut.py:273-319).

    All restarts advance together as one batch; ``threads`` is accepted for API
    compatibility (the batch replaces the reference's thread pool).  complex128 by default:
    the reference trains in complex128, and the trained angles (hence the rounded cut) follow
    its trajectory only at that precision (tests/test_gpu_f1.py)."""
    trunc = False
    if graph.num_vertices and graph.edges:
        eps, chi_max, trunc = _truncation(engine, brickwork_ansatz(mbe_encode(graph)[0], depth), eps, chi_max)
    else:
        _check_engine(engine)
    if optimizer not in ("gd", "adam"):
        raise InputError(f"unknown optimizer {optimizer!r}")
    if restarts < 1:
        raise InputError("need at least one restart")
    if graph.num_vertices == 0 or not graph.edges:
        return MbeResult((1,) * graph.num_vertices, 0.0, 0.0, 0, 0, seed)
    n, _ = mbe_encode(graph)
    circuit = brickwork_ansatz(n, depth)
    theta0 = np.stack([init_params(circuit.n_params, rng) for rng in spawn(seed, restarts)])
    if trunc:
        # the reference's truncated runs: minimize on the taped objective per restart (host loop
        # over device calls; autodiff.minimize = the reference's minimize, autodiff.py:614-659)
        from .autodiff import minimize

        fun = _mbe_objective_truncated(circuit, graph, alpha, eps, chi_max, device)
        runs = [minimize(fun, theta0[r], optimizer=optimizer, rate=rate, max_iters=max_iters) for r in range(restarts)]
        theta = np.stack([res.theta for res in runs])
        loss = np.array([res.value for res in runs])
        iters = np.array([res.n_iters for res in runs])
        exps = vertex_expectations(circuit, theta, graph, eps=eps, chi_max=chi_max, device=device)
    else:
        obj = MBEObjective(circuit, graph, alpha, dtype=dtype, device=device, batch=restarts)
        theta, loss, iters = adam_batched(obj, theta0, rate, max_iters, optimizer=optimizer)
        exps = vertex_expectations(circuit, theta, graph, device=obj.device)
    outcomes = []
    for r in range(restarts):
        asg = round_cut(exps[r])
        outcomes.append((asg, cut_value(graph, asg), float(loss[r]), int(iters[r])))
    best = 0
    for r in range(1, restarts):
        if outcomes[r][1] > outcomes[best][1]:
            best = r
    asg, cut, lval, it = outcomes[best]
    return MbeResult(asg, cut, lval, it, best, seed)


def result_to_dict(result: MbeResult, optimal=None) -> dict:
    return {"cut": result.cut_value, "optimal": None if optimal is None else float(optimal),
            "assignment": list(result.assignment), "loss": result.relaxed_loss, "iters": result.iterations,
            "seed": result.seed}
