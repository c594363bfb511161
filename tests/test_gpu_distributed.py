"""The multi-rank host path with the real engine: world size 2 over gloo, both ranks on
cuda:0.  The ranks' kernels never wait on each other; only the host-side gloo all-reduce
or all-gather joins them.  This exercises distributed.py end to end on one GPU.  The NCCL
transport itself needs more GPUs than this pool gives one call."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_10239_b200 import distributed as D
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

    c = layered_circuit(60, 8, "ry", "cz")
    th = torch.tensor(theta_sets(c.n_params, 4, seed=2), device="cuda")
    ec, gc = D.chain_sharded_energy_grad(c, tfim(60), th, dtype="complex128")
    eb, gb = D.batch_sharded_energy_grad(c, tfim(60), th, dtype="complex128")
    q.put((rank, ec.cpu().numpy(), gc.cpu().numpy(), eb.cpu().numpy(), gb.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_process():
    from paper_2112_10239_b200 import autodiff as AD
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = layered_circuit(60, 8, "ry", "cz")
    th = theta_sets(c.n_params, 4, seed=2)
    v, g = AD.grad_expval(c, tfim(60), th, dtype="complex128")
    for _, ec, gc, eb, gb in res:
        np.testing.assert_allclose(ec, v, atol=1e-11)
        np.testing.assert_allclose(gc, g, atol=1e-11)
        np.testing.assert_allclose(eb, v, atol=1e-11)
        np.testing.assert_allclose(gb, g, atol=1e-11)


@pytest.mark.parametrize("config", ["cfg4", "cfg5"])
def test_bench_gpus2_relaunch_matches_single_process(config):
    """``bench.py --gpus 2`` re-launches itself as two ranks (torchrun); with
    TQ_DIST_BACKEND=gloo both ranks share cuda:0.  Rank 0's line must report n_gpus 2 and the
    chain-sharded energies/gradients (energy all-reduce + halo exchange + owned gather) must
    match one process evaluating the whole operator (--check)."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, TQ_DIST_BACKEND="gloo")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--batch", "4",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--check"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    par = line["parity"]
    assert par["max_abs_dE"] < 1e-4, par
    if par["max_abs_dgrad"] is not None:
        assert par["max_abs_dgrad"] <= 1e-5 * max(par["max_abs_grad"], 1.0), par
