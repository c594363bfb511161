"""Prepared batched evaluation (serving path): compile once, evaluate many angle batches.

``ExpvalProgram(circuit, ham, batch)(theta_host)`` is the host-buffer entry a
service calls: pinned host angles -> device, one engine launch pair, energies
and gradients back to pinned host memory.  It is what ``bench.py`` times for the
end-to-end (``e2e``) number.
"""

from __future__ import annotations

import numpy as np
import torch

from . import chain as C
from . import engine as E
from .errors import InputError


class ExpvalProgram:
    def __init__(self, circuit, ham, batch: int, *, dtype: str = "complex64", device=None, segments=None,
                 grad: bool = True):
        self.circuit, self.ham, self.batch, self.dtype, self.grad = circuit, ham, int(batch), dtype, grad
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.terms = C.normalize_terms(ham)
        self.dp = E.device_plan(circuit, self.terms, "energy", self.batch, self.device, segments, dtype=dtype)
        tdt = E.DTYPES[dtype][1]
        P = circuit.n_params
        self.coef = torch.tensor([[c.real for c, _ in self.terms]], dtype=tdt, device=self.device)
        self.theta_dev = torch.empty(self.batch, P, dtype=tdt, device=self.device)
        self.theta_host = torch.empty(self.batch, P, dtype=tdt, pin_memory=True)
        self.e_host = torch.empty(self.batch, 2, dtype=torch.float64, pin_memory=True)
        self.g_host = torch.empty(self.batch, P, dtype=tdt, pin_memory=True) if grad else None
        # scratch owned by this program: one buffer per captured graph (a graph bakes its
        # workspace pointer in; graphs that may replay concurrently must not share one)
        nws = E.workspace_bytes(self.dp, self.batch, grad, dtype)
        self.ws_dev = torch.empty(nws, dtype=torch.uint8, device=self.device)
        self.ws_io = torch.empty(nws, dtype=torch.uint8, device=self.device)

    @property
    def plan(self):
        return self.dp.plan

    @property
    def h2d_bytes(self) -> int:
        return self.theta_host.numel() * self.theta_host.element_size()

    @property
    def d2h_bytes(self) -> int:
        n = self.e_host.numel() * self.e_host.element_size()
        if self.g_host is not None:
            n += self.g_host.numel() * self.g_host.element_size()
        return n

    def run_device(self, theta_dev: torch.Tensor):
        """Device-resident inputs -> device outputs (no host traffic)."""
        return E.energy_grad_raw(self.dp, theta_dev, self.coef, self.grad, self.dtype, ws=self.ws_dev)

    def capture(self, io: bool = True):
        """Capture one evaluation of ``theta_dev`` into a CUDA graph (the serving loop replays
        it: one launch per batch instead of one per kernel).  Outputs land in the static
        tensors ``energy`` / ``grad_dev``.  With ``io`` a second graph also holds the pinned
        staging copies (``theta_host`` -> device, energies and gradients -> ``e_host`` /
        ``g_host``), so a host-buffer call is a single graph launch."""
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):           # warm-up: plan upload, workspace, kernel attributes
            self.run_device(self.theta_dev)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self.energy, self.grad_dev = self.run_device(self.theta_dev)
        self.io_graph = None
        if io:
            self.io_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.io_graph, capture_error_mode="relaxed"):
                self.theta_dev.copy_(self.theta_host, non_blocking=True)
                # the reduction kernels store the energies and gradients straight into the
                # pinned host buffers (mapped, same pointer under UVA): no separate D2H copies
                self.io_energy, self.io_grad = E.energy_grad_raw(self.dp, self.theta_dev, self.coef, self.grad,
                                                                 self.dtype, out=(self.e_host, self.g_host),
                                                                 ws=self.ws_io)
        torch.cuda.synchronize()
        return self

    def replay(self):
        """Evaluate the current ``theta_dev`` through the captured graph."""
        self.graph.replay()
        return self.energy, self.grad_dev

    def __call__(self, theta, copy_out: bool = True):
        """theta: [batch, P] host array (numpy or pinned torch). Returns (E[B], grad[B,P] | None)."""
        if isinstance(theta, np.ndarray):
            if theta.shape != tuple(self.theta_host.shape):
                raise InputError(f"theta must be {tuple(self.theta_host.shape)}")
            self.theta_host.numpy()[...] = theta
            src = self.theta_host
        else:
            src = theta
        io_graph = getattr(self, "io_graph", None)
        if io_graph is not None:
            if src is not self.theta_host:
                if tuple(src.shape) != tuple(self.theta_host.shape):
                    raise InputError(f"theta must be {tuple(self.theta_host.shape)}")
                self.theta_host.copy_(src)
            io_graph.replay()   # H2D copy, the evaluation kernels, D2H copies
            grad = self.io_grad
        else:
            self.theta_dev.copy_(src, non_blocking=True)
            energy, grad = self.replay() if getattr(self, "graph", None) is not None else self.run_device(self.theta_dev)
            self.e_host.copy_(energy, non_blocking=True)
            if grad is not None:
                self.g_host.copy_(grad, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if not copy_out:
            return self.e_host, self.g_host
        e = self.e_host[:, 0].numpy().copy()
        return e, (self.g_host.numpy().copy() if grad is not None else None)
