"""Multi-rank host logic on CPU: world_size 2 over gloo.  The local evaluator is the
numpy kernel mirror (test infrastructure), so the sharding + all-reduce path is
checked end to end against the reference golden vectors without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def mirror_evaluator(circuit, ham, theta, dtype):
    import mirror
    from paper_2112_10239_b200 import chain as C

    terms = C.normalize_terms(ham)
    B = theta.shape[0]
    if not terms:
        return torch.zeros(B, dtype=torch.float64), torch.zeros(B, circuit.n_params, dtype=torch.float64)
    plan = C.compile_chain(circuit, terms, "energy", segments=1)
    coef = np.array([c.real for c, _ in terms])
    es, gs = [], []
    for b in range(B):
        e, g = mirror.energy_grad(plan, theta[b].numpy(), coef)
        es.append(e.real)
        gs.append(g)
    return torch.tensor(es, dtype=torch.float64), torch.tensor(np.array(gs), dtype=torch.float64)


def _worker(rank, world, port, mode, q, n=12, layers=6):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_10239_b200 import distributed as D
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

    c = layered_circuit(n, layers, "ry", "cz")
    th = torch.tensor(theta_sets(c.n_params, 2, seed=4))
    fn = D.chain_sharded_energy_grad if mode == "chain" else D.batch_sharded_energy_grad
    e, g = fn(c, tfim(n), th, evaluator=mirror_evaluator)
    q.put((rank, e.numpy(), g.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["chain", "batch"])
def test_two_rank_sharding_matches_oracle(mode):
    import oracle as O
    from paper_2112_10239_b200.workloads import theta_sets

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    th = theta_sets(O.ry_cz_layers(12, 6).n_params, 2, seed=4)
    oc, ot = O.ry_cz_layers(12, 6), O.tfim_terms(12)
    for _, e, g in res:
        for b in range(2):
            ov, og = O.grad_expval_tt(oc, ot, th[b])
            assert abs(e[b] - ov) < 1e-11
            np.testing.assert_allclose(g[b], og, atol=1e-11)


def test_shard_partition_is_exact():
    from paper_2112_10239_b200 import distributed as D
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.workloads import layered_circuit

    ham = tfim(1000)
    for world in (1, 2, 4, 8):
        parts = [D.shard_hamiltonian(ham, r, world) for r in range(world)]
        assert sum(len(p.terms) for p in parts) == len(ham.terms)
        got = sorted(t.ops for p in parts for t in p.terms)
        assert got == sorted(t.ops for t in ham.terms)
    sub = D.halo_overlap(layered_circuit(1000, 20), ham, 8)
    assert np.all(sub <= 125 + 2 * 11 + 2)   # owned 125 sites + light-cone halo of the 10 lines


def test_four_rank_chain_exchange_matches_oracle():
    """World 4 over gloo with a light-cone halo wider than an owned range (n=12, 5 entangler
    lines): rank 1's sub-chain reaches angles owned by rank 3, so the halo exchange is not
    neighbour-only.  The full gradient on every rank must equal the oracle's."""
    import oracle as O
    from paper_2112_10239_b200 import distributed as D
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

    ex = D.ChainExchange(layered_circuit(12, 10), tfim(12), 4)
    assert len(ex.halo[1][3]) > 0                       # a non-neighbour halo exists
    assert sum(len(o) for o in ex.owned) == layered_circuit(12, 10).n_params
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, "chain", q, 12, 10)) for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oc, ot = O.ry_cz_layers(12, 10), O.tfim_terms(12)
    th = theta_sets(oc.n_params, 2, seed=4)
    for _, e, g in res:
        for b in range(2):
            ov, og = O.grad_expval_tt(oc, ot, th[b])
            assert abs(e[b] - ov) < 1e-11
            np.testing.assert_allclose(g[b], og, atol=1e-11)
