"""Multi-GPU execution: one process per GPU, ``torch.distributed`` (NCCL on B200s).

Two decompositions (DESIGN.md section "Multi-GPU"):

``chain`` (cfg4 / cfg5): the qubit chain is cut into contiguous owned ranges, one per
rank.  A rank owns every Pauli term whose first site lies in its range and evaluates
exactly those terms on the light-cone sub-chain around its range (halo = backward
light cone, reference-free: gates outside a term's cone cancel, SURVEY.md finding 3).
No environment crosses ranks.  The only exchange is one all-reduce(SUM) of the
partial energies [B] and of the gradients [B, P]; every angle's gradient is the sum
of the contributions of the ranks whose sub-chain contains it (halo overlap).

``batch`` (cfg1 / cfg2): angle sets are split across ranks; results are gathered.

The local evaluator is injectable (default: the B200 engine) so the host logic can
be tested on CPU with the gloo backend.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .hamiltonians import PauliHamiltonian


def owned_range(n_qubits: int, rank: int, world: int):
    """[lo, hi) of sites owned by ``rank`` (contiguous, balanced)."""
    return rank * n_qubits // world, (rank + 1) * n_qubits // world


def shard_hamiltonian(ham: PauliHamiltonian, rank: int, world: int) -> PauliHamiltonian:
    """Terms whose first (lowest) site lies in the rank's owned range.  Identity terms
    (no support) go to rank 0 so the constant is counted once."""
    lo, hi = owned_range(ham.n_qubits, rank, world)
    keep = []
    for t in ham.terms:
        if not t.ops:
            if rank == 0:
                keep.append(t)
        elif lo <= t.support[0] < hi:
            keep.append(t)
    return PauliHamiltonian(ham.n_qubits, tuple(keep))


def _engine_evaluator(circuit, ham, theta: torch.Tensor, dtype: str):
    from . import chain as C
    from . import engine as E

    terms = C.normalize_terms(ham)
    if not terms:
        B = theta.shape[0]
        return (torch.zeros(B, dtype=torch.float64, device=theta.device),
                torch.zeros_like(theta))
    dp = E.device_plan(circuit, terms, "energy", theta.shape[0], theta.device, None, dtype=dtype)
    coef = torch.tensor([[c.real for c, _ in terms]], dtype=torch.float64, device=theta.device)
    energy, grad = E.energy_grad_raw(dp, theta, coef, True, dtype)
    return energy[:, 0].contiguous(), grad


def chain_sharded_energy_grad(circuit, ham: PauliHamiltonian, theta: torch.Tensor, *, group=None,
                              dtype: str = "complex64", evaluator=None):
    """E[b] and dE/dtheta[b] with the chain split over the ranks of ``group``.

    Every rank passes the same theta [B, P] and gets the full results back."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = shard_hamiltonian(ham, rank, world)
    ev = evaluator or _engine_evaluator
    energy, grad = ev(circuit, local, theta, dtype)
    energy = energy.to(torch.float64)
    grad = grad.to(torch.float64)
    if world > 1:
        dist.all_reduce(energy, group=group)
        dist.all_reduce(grad, group=group)
    return energy, grad


def batch_sharded_energy_grad(circuit, ham: PauliHamiltonian, theta: torch.Tensor, *, group=None,
                              dtype: str = "complex64", evaluator=None):
    """Angle sets split evenly over ranks (theta [B, P] identical on all ranks, B divisible
    by the world size); results all-gathered so every rank returns all B rows."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    B = theta.shape[0]
    if B % world:
        raise ValueError(f"batch {B} not divisible by world size {world}")
    per = B // world
    mine = theta[rank * per:(rank + 1) * per]
    ev = evaluator or _engine_evaluator
    e, g = ev(circuit, ham, mine, dtype)
    e, g = e.to(torch.float64).contiguous(), g.to(torch.float64).contiguous()
    if world == 1:
        return e, g
    es = [torch.empty_like(e) for _ in range(world)]
    gs = [torch.empty_like(g) for _ in range(world)]
    dist.all_gather(es, e, group=group)
    dist.all_gather(gs, g, group=group)
    return torch.cat(es), torch.cat(gs)


def halo_overlap(circuit, ham: PauliHamiltonian, world: int) -> np.ndarray:
    """Per-rank sub-chain length (sites) for the chain decomposition, for reporting redundancy."""
    from . import chain as C

    tg = C.time_gates(circuit)
    out = []
    for r in range(world):
        loc = shard_hamiltonian(ham, r, world)
        if not loc.terms:
            out.append(0)
            continue
        lo = min(t.support[0] for t in loc.terms if t.ops)
        hi = max(t.support[-1] for t in loc.terms if t.ops)
        clo, chi = C.light_cone(tg, lo, hi)
        out.append(chi - clo + 1)
    return np.array(out)
