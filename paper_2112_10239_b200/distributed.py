"""Multi-GPU execution: one process per GPU, ``torch.distributed`` (NCCL on B200s).

Two decompositions (DESIGN.md section "Multi-GPU"):

``chain`` (cfg4 / cfg5): the qubit chain is cut into contiguous owned ranges, one per
rank.  A rank owns every Pauli term whose first site lies in its range and evaluates
exactly those terms on the light-cone sub-chain around its range (halo = backward
light cone, reference-free: gates outside a term's cone cancel, SURVEY.md finding 3).
No environment crosses ranks.  The exchange is one all-reduce(SUM) of the partial
energies [B] plus the gradient exchange of :class:`ChainExchange`: halo columns are sent
to the angles' owners (send/recv with the neighbours), then the owned columns are
all-gathered; every angle's gradient is the sum of the contributions of the ranks whose
sub-chain contains it.

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


class ChainExchange:
    """The gradient exchange of the chain decomposition (collective 2).

    Rank r's sweep yields dE/dtheta contributions only for angles whose gate lies inside its
    light-cone sub-chain [clo_r, chi_r]: its owned sites plus a halo of about one site per
    entangler line on each side.  Angle p is OWNED by the rank owning its gate's first wire.
    The exchange is

      1. halo: rank r sends the fp32 columns of its halo angles to their owners
         (``batch_isend_irecv`` of [B, |halo|] blocks -- NCCL send/recv over NVLink on B200);
         owners add them to their own columns in ascending-rank order (deterministic);
      2. owned gather: every rank all-gathers the owned columns (padded to the largest owned
         count), so each rank returns the full [B, P] gradient.

    Bytes per rank: B x 4 x (|halo| + P) instead of an all-reduce's 2 x B x 4 x P."""

    def __init__(self, circuit, ham: PauliHamiltonian, world: int):
        from . import chain as C

        self.world = world
        n = circuit.n_qubits
        P = circuit.n_params
        tg = C.time_gates(circuit)
        gate_wires = [tuple(int(w) for w in circuit.gates[gi].wires) for gi in circuit.trainable]
        owner = np.array([min(np.searchsorted([owned_range(n, r, world)[1] for r in range(world)], min(w), "right"),
                              world - 1) for w in gate_wires], dtype=np.int64)
        self.owner = owner
        self.owned = [np.nonzero(owner == r)[0] for r in range(world)]
        self.sub = []
        for r in range(world):
            loc = shard_hamiltonian(ham, r, world)
            sup = [t.support for t in loc.terms if t.ops]
            if not sup:
                self.sub.append(None)
                continue
            self.sub.append(C.light_cone(tg, min(s[0] for s in sup), max(s[-1] for s in sup)))
        # halo[r][s]: angles in rank r's sub-chain (gate fully inside) owned by s != r
        self.halo = [[np.zeros(0, dtype=np.int64) for _ in range(world)] for _ in range(world)]
        for r in range(world):
            if self.sub[r] is None:
                continue
            lo, hi = self.sub[r]
            inside = np.array([min(w) >= lo and max(w) <= hi for w in gate_wires], dtype=bool) if P else np.zeros(0, bool)
            for s in range(world):
                if s != r:
                    self.halo[r][s] = np.nonzero(inside & (owner == s))[0]
        pos = np.full(P, -1, dtype=np.int64)
        for r in range(world):
            pos[self.owned[r]] = np.arange(len(self.owned[r]))
        self.pos = pos
        self.max_owned = max((len(o) for o in self.owned), default=0)
        self._dev = {}

    def halo_elems(self, rank: int) -> int:
        return int(sum(len(h) for h in self.halo[rank]))

    def _t(self, key, a, device):
        """Device copy of index array ``a`` (a fixed attribute of this layout), cached by ``key``."""
        k = (key, str(device))
        t = self._dev.get(k)
        if t is None:
            t = self._dev[k] = torch.as_tensor(a, dtype=torch.long, device=device)
        return t

    def exchange(self, grad: torch.Tensor, rank: int, group=None) -> torch.Tensor:
        """grad [B, P] (this rank's contributions) -> full gradient [B, P] on every rank."""
        world = self.world
        if world == 1:
            return grad
        B, dev = grad.shape[0], grad.device
        ops, recvs = [], []
        gr = (lambda s: dist.get_global_rank(group, s)) if group is not None else (lambda s: s)
        # gloo's point-to-point ops take host tensors only (the CPU test path); NCCL sends device memory
        host = dev.type == "cuda" and dist.get_backend(group) == "gloo"
        bdev = torch.device("cpu") if host else dev
        for s in range(world):
            if s == rank:
                continue
            hs = self.halo[rank][s]
            if len(hs):
                blk = grad.index_select(1, self._t(('h', rank, s), hs, dev)).contiguous()
                ops.append(dist.P2POp(dist.isend, blk.to(bdev), gr(s), group))
            hr = self.halo[s][rank]
            if len(hr):
                buf = torch.empty(B, len(hr), dtype=grad.dtype, device=bdev)
                ops.append(dist.P2POp(dist.irecv, buf, gr(s), group))
                recvs.append((s, hr, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        own = torch.zeros(B, self.max_owned, dtype=grad.dtype, device=dev)
        mine = self.owned[rank]
        own[:, :len(mine)] = grad.index_select(1, self._t(('o', rank), mine, dev))
        for s, hr, buf in sorted(recvs, key=lambda x: x[0]):     # fixed order: ascending source rank
            own.index_add_(1, self._t(('p', s, rank), self.pos[hr], dev), buf.to(dev))
        outs = [torch.empty_like(own) for _ in range(world)]
        dist.all_gather(outs, own, group=group)
        full = torch.empty_like(grad)
        for s in range(world):
            o = self.owned[s]
            if len(o):
                full.index_copy_(1, self._t(('o', s), o, dev), outs[s][:, :len(o)])
        return full


def chain_sharded_energy_grad(circuit, ham: PauliHamiltonian, theta: torch.Tensor, *, group=None,
                              dtype: str = "complex64", evaluator=None, exchange: ChainExchange | None = None):
    """E[b] and dE/dtheta[b] with the chain split over the ranks of ``group``.

    Every rank passes the same theta [B, P] and gets the full results back: one all-reduce of
    the partial energies [B] (float64) and the halo + owned-gather gradient exchange
    (:class:`ChainExchange`, in the engine's real dtype)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    local = shard_hamiltonian(ham, rank, world)
    ev = evaluator or _engine_evaluator
    energy, grad = ev(circuit, local, theta, dtype)
    energy = energy.to(torch.float64)
    if world > 1:
        dist.all_reduce(energy, group=group)
        ex = exchange or ChainExchange(circuit, ham, world)
        grad = ex.exchange(grad.contiguous(), rank, group)
    return energy, grad.to(torch.float64)


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
