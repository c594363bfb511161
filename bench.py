#!/usr/bin/env python
"""Benchmark: TT-circuit TFIM energy+gradient evaluations per second on B200.

Default workload: BASELINE.json configs[3] = cfg4, the configuration the metric is quoted on
("n qubits, L layers (1/2/4/8 B200)"): TTCircuit n=1000, 20 layers (10 RotY rows + 10 CZ
lines, reading A), TFIM energy + full gradient, 64 parameter sets per step, the qubit chain
sharded over the ranks (strong scaling).  ``--config cfg2`` (n=100, B=256, theta-set data
parallel), ``cfg5`` (n=1024 per GPU, forward only, weak scaling), ``cfg1``, ``cfg3`` (MBE
MaxCut Adam step) and ``f3`` (truncated engine) are also available.  ``--gpus N`` outside
torchrun re-launches itself as N ranks (one per GPU, NCCL).

One JSON line on rank 0 (contract in the task brief): value = whole-job evals/s from
device-resident inputs; e2e = same metric through ExpvalProgram with pinned host
buffers (H2D + D2H inside the timed region); roofline for the dominant sweep kernel
with SURVEY.md section 8(d)'s work formulas against the measured FP32 FFMA peak;
cpu_baseline = the CPU oracle port of the reference timed on this host.
``--impl reference`` times that CPU path alone.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "expectation+gradient evals/sec at n qubits, L layers (1/2/4/8 B200); HBM GB/s frac"
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc, self.thread = index, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.samples:
            return None
        loaded = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        reasons = set()
        for _, _, r in loaded:
            for bit, name in REASON_BITS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": max(s[1] for s in loaded),
                "reasons": sorted(reasons), "samples": len(loaded)}


# ----------------------------------------------------------------------------- CPU oracle
def _oracle_eval(args):
    n, layers, rot, ent, theta = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    import oracle as O

    c = O.ry_cz_layers(n, layers, rot, ent)
    t0 = time.perf_counter()
    O.grad_expval_tt(c, O.tfim_terms(n), theta)
    return time.perf_counter() - t0


def _oracle_forward(args):
    n, layers, rot, ent, theta = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    import oracle as O

    c = O.ry_cz_layers(n, layers, rot, ent)
    t0 = time.perf_counter()
    O.evaluate_expval(c, O.tfim_terms(n), theta, eps=1e-12)
    return time.perf_counter() - t0


def cpu_baseline_block(cfg, circuit, n, workers):
    """CPU oracle port on this host, sized to ~10-30 s of CPU work, in the metric's unit.

    cfg1/cfg2: exact taped E+grad (reference grad_expval engine='tt' eps=0).
    cfg4: the exact taped gradient is infeasible (eps=0 bond 2^lines = 1024); the reference's
          exact alternative is the shift rule, 2P+1 forward evaluations, so E+grad/s =
          forwards/s / (2P + 1) from timed forward evaluate_expval(eps=1e-12) runs.
    cfg5: forward only -> forwards/s."""
    from paper_2112_10239_b200.workloads import theta_sets

    if cfg.name in ("cfg4", "cfg5"):
        k = max(1, min(workers, 4))
        jobs = [(n, cfg.layers, cfg.rot, cfg.ent, th) for th in theta_sets(circuit.n_params, k, seed=99)]
        import multiprocessing as mp

        with mp.get_context("fork").Pool(k) as pool:
            t0 = time.perf_counter()
            per = pool.map(_oracle_forward, jobs)
            wall = time.perf_counter() - t0
        fwd_rate = k / wall
        if cfg.name == "cfg5":
            return {"value": fwd_rate, "unit": "evals/s", "cores": k, "kind": "port",
                    "sample": f"{k} forward evaluations n={n} (oracle port of tnsim evaluate_expval eps=1e-12), "
                              f"{sum(per):.1f} CPU-s"}
        P = circuit.n_params
        return {"value": fwd_rate / (2 * P + 1), "unit": "evals/s", "cores": k, "kind": "port",
                "sample": f"{k} forward evaluations n={n} (evaluate_expval eps=1e-12, {sum(per):.1f} CPU-s); "
                          f"E+grad via the exact shift rule = {2 * P + 1} forwards per evaluation"}
    sample_n = min(256, max(2 * workers, 16))
    rate, wall, cpu_s = cpu_oracle_rate(cfg, theta_sets(circuit.n_params, sample_n, seed=99), workers)
    return {"value": rate, "unit": "evals/s", "cores": workers, "kind": "port",
            "sample": f"{sample_n} theta-sets of {cfg.name} (oracle port of tnsim grad_expval engine='tt' eps=0), "
                      f"{cpu_s:.1f} CPU-s over {wall:.1f} s wall"}


def cpu_oracle_rate(cfg, thetas, workers):
    """Evaluate theta-sets with the CPU oracle port on `workers` processes; returns evals/s."""
    import multiprocessing as mp

    jobs = [(cfg.n, cfg.layers, cfg.rot, cfg.ent, th) for th in thetas]
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        pool.map(_oracle_eval, jobs[:workers])  # warm the workers (imports)
        t0 = time.perf_counter()
        per = pool.map(_oracle_eval, jobs)
        wall = time.perf_counter() - t0
    return len(jobs) / wall, wall, float(sum(per))


def _init_dist(dist, dev):
    """NCCL, one process per GPU.  TQ_DIST_BACKEND=gloo runs the same host path with every rank
    on the visible GPUs (a functional check of the multi-rank code on a 1-GPU box; its numbers
    are not measurements)."""
    backend = os.environ.get("TQ_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    """The reference's CPU path (the oracle port of tnsim) on this host's cores, same metric and
    config as our arm.  cfg1/cfg2: exact taped E+grad (grad_expval engine='tt', eps=0), one
    theta-set per process.  cfg4: the exact taped gradient is infeasible on the reference
    (eps=0 bond 2^lines = 1024), its exact alternative is the shift rule = 2P+1 forward
    evaluations, so each step times one forward evaluate_expval(eps=1e-12) per process and
    evals/s = forwards/s / (2P+1).  cfg5: forward-only, evals/s = forwards/s.  Under torchrun
    only rank 0 runs (the others exit without work)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2112_10239_b200.workloads import theta_sets

    cores = host_cores()
    n = cfg.n * ws if cfg.name == "cfg5" else cfg.n
    forward = cfg.name in ("cfg4", "cfg5")
    per_step = max(cores, 4) if not forward else cores
    circuit = cfg.circuit() if cfg.name != "cfg5" else __import__(
        "paper_2112_10239_b200.workloads", fromlist=["x"]).layered_circuit(n, cfg.layers, cfg.rot, cfg.ent)
    P = circuit.n_params
    thetas = theta_sets(P, per_step * (args.steps + args.warmup), seed=0)
    import multiprocessing as mp

    fn = _oracle_forward if forward else _oracle_eval
    jobs = [(n, cfg.layers, cfg.rot, cfg.ent, th) for th in thetas]
    with mp.get_context("fork").Pool(cores) as pool:
        for w in range(args.warmup):
            pool.map(fn, jobs[w * per_step:(w + 1) * per_step])
        t0 = time.perf_counter()
        off = args.warmup * per_step
        for s in range(args.steps):
            pool.map(fn, jobs[off + s * per_step: off + (s + 1) * per_step])
        wall = time.perf_counter() - t0
    rate = args.steps * per_step / wall
    if cfg.name == "cfg4":
        value = rate / (2 * P + 1)
        sample = (f"{per_step} forward evaluations of cfg4 per step (oracle port of tnsim evaluate_expval "
                  f"engine='tt' eps=1e-12), {rate:.3f} forwards/s; exact E+grad = shift rule, {2 * P + 1} forwards")
    elif cfg.name == "cfg5":
        value = rate
        sample = f"{per_step} forward evaluations of cfg5 n={n} per step (oracle port of tnsim evaluate_expval eps=1e-12)"
    else:
        value = rate
        sample = f"{per_step} theta-sets of {cfg.name} per step (CPU oracle port of tnsim grad_expval(engine='tt', eps=0))"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "strong" if cfg.name == "cfg4" else "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (seeded U[-pi,pi) angles, float32-rounded)",
        "config": config_block(cfg, None, cfg.batch if forward else per_step, n, ws),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(cfg, plan, batch, n_override=None, world=1):
    n = n_override or cfg.n
    blk = {"workload": f"{cfg.name}: {cfg.description}", "n_qubits": n, "layers": cfg.layers,
           "rotation_rows": (cfg.layers + 1) // 2, "entangler_lines": cfg.layers // 2,
           "rotation": cfg.rot, "entangler": cfg.ent, "operator": "TFIM open chain j=h=1",
           "batch_per_gpu": batch, "gradient": cfg.grad,
           "layer_semantics": "reading A (layer = one TTCircuit unitary)"}
    if plan is not None:
        blk.update({"segments": plan.n_segments, "chi_max": plan.chi_max, "mpo_channels": plan.d_max,
                    "sub_chain_sites": int(plan.info.get("sub_chain_sites", 0))})
    blk["parallelism"] = ("theta-set data parallel" if cfg.name in ("cfg1", "cfg2") else "qubit-chain segments") + (
        f" over {world} GPUs" if world > 1 else "")
    return blk


# ----------------------------------------------------------------------------- our arm
def work_model(cfg, circuit, ham, batch):
    """SURVEY.md section 8(d) per-evaluation work (the official formulas) plus the kernels'
    executed-cMAC model, both from the unsegmented plan of the full chain."""
    from paper_2112_10239_b200 import chain as C
    from paper_2112_10239_b200 import roofline

    terms = C.normalize_terms(ham)
    t1 = sum(1 for _, ops in terms if len(ops) == 1)
    t2 = sum(1 for _, ops in terms if len(ops) == 2)
    plan1 = C.compile_chain(circuit, terms, "energy", batch=batch, segments=1)
    # the bench arm computes in complex64: real-path plans run the real-part instantiation
    real = bool(C.real_path(plan1)) and plan1.mode != "values"
    return (roofline.survey_model(plan1, t1, t2, cfg.layers, cfg.grad),
            roofline.eval_model(plan1, grad=cfg.grad, real=real))


def run_ours(args, cfg):
    import torch

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        _init_dist(dist, dev)
    from paper_2112_10239_b200 import _lib, engine as E
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.program import ExpvalProgram
    from paper_2112_10239_b200.workloads import layered_circuit, theta_sets

    batch = args.batch or cfg.batch
    sharded = cfg.name in ("cfg4", "cfg5")
    n = cfg.n * ws if cfg.name == "cfg5" else cfg.n
    circuit = layered_circuit(n, cfg.layers, cfg.rot, cfg.ent)
    ham_full = tfim(n)
    exch = None
    if sharded and ws > 1:
        from paper_2112_10239_b200.distributed import ChainExchange, shard_hamiltonian

        ham = shard_hamiltonian(ham_full, rank, ws)   # terms owned by this rank's chain range
        exch = ChainExchange(circuit, ham_full, ws) if cfg.grad else None
    else:
        ham = ham_full
    seed = 0 if sharded else rank
    thetas = theta_sets(circuit.n_params, batch, seed=seed)
    prog = ExpvalProgram(circuit, ham, batch, device=dev, segments=args.segments, grad=cfg.grad)
    plan = prog.plan
    theta_dev = torch.tensor(thetas, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    lib = _lib.load()
    import ctypes

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    code = _lib.TQ_C64
    ws_buf, ws_bytes = prog.dp.workspace(batch, _lib.TQ_FLAG_GRAD if cfg.grad else 0, code, stream.cuda_stream)
    energy = torch.empty(batch, 2, dtype=torch.float64, device=dev)
    grad = torch.empty(batch, circuit.n_params, dtype=torch.float32, device=dev) if cfg.grad else None
    ms_k = (ctypes.c_float * 3)()

    def collect(e_dev, g_dev):
        """Chain sharding: E partials all-reduced, gradient halo exchange + owned gather."""
        if ws > 1 and sharded:
            dist.all_reduce(e_dev)
            if g_dev is not None:
                g_dev = exch.exchange(g_dev, rank)
        return e_dev, g_dev

    def step(timed=False):
        fn = lib.tq_energy_grad_timed if timed else lib.tq_energy_grad
        extra = (ms_k,) if timed else ()
        st = fn(ctypes.byref(prog.dp.chain), code, batch, theta_dev.data_ptr(), theta_dev.stride(0),
                prog.coef.data_ptr(), 0, energy.data_ptr(), grad.data_ptr() if grad is not None else None,
                ws_buf.data_ptr(), ws_bytes, stream.cuda_stream, *extra)
        _lib.check(st)
        return collect(energy, grad)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    warm = max(3, args.warmup)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    E.check_finite(energy, grad)

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.25)
    # per-kernel times for the roofline: eager steps through the timed entry point (CUDA events
    # recorded by the library around each sweep launch on this stream)
    rl_ms, lr_ms, adj_ms = [], [], []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        step(timed=True)
        rl_ms.append(ms_k[0])
        lr_ms.append(ms_k[1])
        adj_ms.append(ms_k[2])
    # the step: the serving program's captured evaluation (ExpvalProgram.capture), replayed on
    # the device-resident angles; the chain-sharding exchange follows each replay
    prog.theta_dev.copy_(theta_dev)
    prog.capture()
    for _ in range(warm):
        collect(*prog.replay())
    torch.cuda.synchronize()
    step_ms = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2); not timed
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e_out, g_out = collect(*prog.replay())
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    barrier()
    E.check_finite(e_out, g_out)
    res_e, res_g = e_out[:, 0].double().cpu().numpy(), (g_out.double().cpu().numpy() if g_out is not None else None)
    clocks = sampler.stop() if sampler else None

    def max_over_ranks(x):
        if ws > 1:
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t)
        return x

    ms_per_step = max_over_ranks(sum(step_ms)) / args.steps
    evals_per_step = batch * (ws if not sharded else 1)
    value = evals_per_step / (ms_per_step * 1e-3)

    # ---- e2e through the host-buffer entry (pinned host -> device -> host)
    # The batch sits in the program's pinned staging buffer (where a service places each request
    # batch).  Every timed call copies it to the device, evaluates, and reads the energies and
    # gradients back into pinned host memory.  N = 1: one captured graph launch
    # (ExpvalProgram.capture, io graph).  Chain-sharded N > 1: H2D, the device graph, the exchange
    # on the device, then D2H of the full results.
    prog.theta_host.copy_(torch.as_tensor(np.asarray(thetas), dtype=prog.theta_host.dtype))
    host = prog.theta_host

    def e2e_call():
        if ws > 1 and sharded:
            prog.theta_dev.copy_(host, non_blocking=True)
            e_d, g_d = collect(*prog.replay())
            prog.e_host.copy_(e_d, non_blocking=True)
            if g_d is not None:
                prog.g_host.copy_(g_d, non_blocking=True)
            stream.synchronize()
        else:
            prog(host, copy_out=False)

    for _ in range(3):
        e2e_call()
    e2e_ms = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_call()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    barrier()
    e2e_ms_step = max_over_ranks(sum(e2e_ms)) / args.steps
    e2e_value = evals_per_step / (e2e_ms_step * 1e-3)

    parity = None
    if args.check:
        # the sharded results against one process evaluating the full operator on this GPU
        from paper_2112_10239_b200 import autodiff as AD

        v1, g1 = AD.grad_expval(circuit, ham_full, thetas) if cfg.grad else (
            AD.evaluate_expval(circuit, ham_full, thetas), None)
        v1 = np.atleast_1d(v1)
        parity = {"max_abs_dE": float(np.max(np.abs(res_e - v1))),
                  "max_abs_dgrad": float(np.max(np.abs(res_g - g1))) if g1 is not None else None,
                  "max_abs_grad": float(np.max(np.abs(g1))) if g1 is not None else None}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    # ---- roofline: SURVEY.md section 8(d) work against the measured FFMA peak
    survey, executed = work_model(cfg, circuit, ham_full, batch)
    ffma = ctypes.c_double(0)
    _lib.check(lib.tq_ffma_peak(20000, stream.cuda_stream, ctypes.byref(ffma)))
    peak_fp32 = ffma.value
    mean_rl = statistics.mean(rl_ms)
    mean_lr = statistics.mean(lr_ms) if cfg.grad else 0.0
    mean_adj = statistics.mean(adj_ms) if cfg.grad else 0.0
    # evaluations this rank's kernels processed per step (chain sharding: the rank's share of
    # the chain, counted as owned sites / n of each evaluation)
    share = (1.0 / ws) if sharded else 1.0
    f_fwd = survey["F_fwd"] * batch * share
    # forward work = rl_sweep; reverse work (2 F_fwd) = lr_sweep + adj_sweep
    if not cfg.grad or mean_rl >= mean_lr + mean_adj:
        kname, kms, kflops = "rl_sweep (forward: MPO environments, energy)", mean_rl, f_fwd
    else:
        kname, kms, kflops = ("lr_sweep + adj_sweep (reverse: environments, core cotangents, column adjoint)",
                              mean_lr + mean_adj, 2 * f_fwd)
    achieved = kflops / (kms * 1e-3) / 1e12
    exec_flops = batch * share * (executed["flops_rl"] if kname.startswith("rl")
                                  else executed["flops_lr"] + executed["flops_adj"])
    exec_tf = exec_flops / (kms * 1e-3) / 1e12
    step_flops = survey["F_eval"] * batch * share
    step_tf = step_flops / (ms_per_step * 1e-3) / 1e12
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    step_bytes = survey["B_eval"] * batch * share
    hbm_gbs = step_bytes / (ms_per_step * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(cfg.name, {})
            keys = ("lr_sweep", "adj_sweep") if kname.startswith("lr") else ("rl_sweep",)
            traffic = sum(tj[k] for k in keys) if all(k in tj for k in keys) else None
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = cpu_baseline_block(cfg, circuit, n, host_cores())

    # rl_sweep + reduce_energy (+ lr_sweep + adj_sweep + reduce_grad)
    # (+ build_wct: channel-pair bracket matrices, shared coefficient row, <= 4 MPO channels)
    launches_per_step = 2 + (3 if cfg.grad else 0) + (1 if plan.d_max <= 4 else 0)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
        "warmup": warm, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if cfg.name == "cfg4" else "weak",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic (seeded U[-pi,pi) angles, float32-rounded; random-init circuit of the named architecture)",
        "config": {**config_block(cfg, plan, batch, n, ws),
                   "l2": "flushed between timed steps (256 MiB memset, untimed)",
                   "step": "one replay of the captured evaluation (program.ExpvalProgram.capture)"
                           + (" + NCCL energy all-reduce and gradient halo exchange" if ws > 1 and sharded else "")},
        "roofline": {"bound": "fp32_simt", "kernel": kname, "achieved": achieved, "peak": peak_fp32,
                     "unit": "TFLOP/s", "frac": achieved / peak_fp32 if peak_fp32 else None, "traffic": traffic,
                     "peak_source": "measured FFMA probe (tq_ffma_peak) on this GPU in this run "
                                    "(MEASURED_PEAKS.json has no FP32 SIMT figure)",
                     "work_model": "SURVEY.md 8(d): F_fwd per eval to rl_sweep, 2 F_fwd to lr_sweep + adj_sweep",
                     "F_eval": survey["F_eval"], "F_fwd": survey["F_fwd"], "flops_per_launch": kflops, "kernel_ms": kms,
                     "step": {"achieved": step_tf, "frac": step_tf / peak_fp32 if peak_fp32 else None,
                              "flops_per_step": step_flops},
                     "rl_ms": mean_rl, "lr_ms": mean_lr, "adj_ms": mean_adj,
                     "step_frac": {"rl": mean_rl / ms_per_step, "lr": mean_lr / ms_per_step,
                                   "adj": mean_adj / ms_per_step},
                     "executed_model": {"flops_rl": executed["flops_rl"], "flops_lr": executed["flops_lr"],
                                        "flops_adj": executed["flops_adj"],
                                        "flops_per_launch": exec_flops, "achieved": exec_tf,
                                        "real_path": executed["real_path"],
                                        "flops_per_cmac": executed["flops_per_cmac"],
                                        "frac": exec_tf / peak_fp32 if peak_fp32 else None,
                                        "note": "roofline.eval_model: cMACs the kernels issue (unsegmented chain, "
                                                "Hermitian transfers on upper tiles). 8(d)'s F counts every "
                                                "transfer in full, so its frac can exceed 1 where the kernels "
                                                "skip work the formula counts; this frac is the FFMA share the "
                                                "useful executed work reaches (real_path: 2 flops per cMAC, the "
                                                "one real FMA the real-part instantiation issues)"}},
        "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": hbm_peak, "frac": hbm_gbs / hbm_peak,
                "bytes_per_step": step_bytes, "B_eval": survey["B_eval"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs", "work_model": "SURVEY.md 8(d) B_eval"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": prog.h2d_bytes,
                "d2h_bytes_per_step": prog.d2h_bytes, "ms_per_step": e2e_ms_step},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    if parity is not None:
        line["parity"] = parity
    if exch is not None:
        line["config"]["halo_angles_exchanged"] = exch.halo_elems(rank)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- cfg3 (MBE MaxCut)
def cfg3_problem():
    from paper_2112_10239_b200 import maxcut as MC
    from paper_2112_10239_b200.seeding import generator

    rng = generator(3)
    graph = MC.pairing_graph(2048, 3, rng)
    circuit = MC.brickwork_ansatz(1024, 4)
    return MC, graph, circuit, rng


def _mbe_oracle_step(args):
    edges, theta = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    import oracle as O

    t0 = time.perf_counter()
    O.mbe_objective(O.brickwork(1024, 4), 2048, edges)(theta)
    return time.perf_counter() - t0


def run_cfg3(args, cfg):
    """One Adam step (readouts -> tanh loss -> cotangents -> gradient sweep -> update) for
    B restarts at once; metric = restart-steps (loss+gradient evaluations) per second."""
    import ctypes

    import torch

    from paper_2112_10239_b200 import _lib, engine as E, roofline

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    MC, graph, circuit, rng = cfg3_problem()
    B = args.batch or cfg.batch
    from paper_2112_10239_b200.seeding import spawn
    from paper_2112_10239_b200.workloads import f32

    theta0 = np.stack([f32(r.uniform(-np.pi, np.pi, circuit.n_params)) for r in spawn(3 + rank, B)])
    obj = MC.MBEObjective(circuit, graph, 1.0, device=dev, batch=B)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    theta = torch.tensor(theta0, dtype=torch.float64, device=dev)
    m = torch.zeros_like(theta)
    v = torch.zeros_like(theta)
    ms_k = (ctypes.c_float * 3)()
    dpe = obj.dp_energy
    ws_buf, ws_bytes = dpe.workspace(B, _lib.TQ_FLAG_GRAD, _lib.TQ_C64, stream.cuda_stream)
    energy = torch.empty(B, 2, dtype=torch.float64, device=dev)
    grad = torch.empty(B, circuit.n_params, dtype=torch.float32, device=dev)
    kt = {"values": [], "rl": [], "lr": [], "adj": []}

    def step(it, timed=False):
        nonlocal theta, m, v
        th32 = theta.to(torch.float32)
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        r = E.values_raw(obj.dp_values, th32, "complex64").real
        if timed:
            b.record(stream)
        t = torch.tanh(obj.alpha * r)
        tp = torch.cat([t, torch.zeros(B, 1, dtype=t.dtype, device=dev)], dim=1)
        g = (obj.alpha * (1.0 - t * t) * (tp[:, obj.nbr] * obj.wts).sum(dim=2)).to(torch.float32).contiguous()
        fn = lib.tq_energy_grad_timed if timed else lib.tq_energy_grad
        extra = (ms_k,) if timed else ()
        _lib.check(fn(ctypes.byref(dpe.chain), _lib.TQ_C64, B, th32.data_ptr(), th32.stride(0), g.data_ptr(),
                      g.stride(0), energy.data_ptr(), grad.data_ptr(), ws_buf.data_ptr(), ws_bytes,
                      stream.cuda_stream, *extra))
        gd = grad.double()
        m = 0.9 * m + 0.1 * gd
        v = 0.999 * v + 0.001 * gd * gd
        theta = theta - 0.1 * (m / (1 - 0.9 ** (it + 1))) / (torch.sqrt(v / (1 - 0.999 ** (it + 1))) + 1e-8)
        if timed:
            b.synchronize()
            kt["values"].append(a.elapsed_time(b))
            kt["rl"].append(ms_k[0])
            kt["lr"].append(ms_k[1])
            kt["adj"].append(ms_k[2])

    for it in range(max(3, args.warmup)):
        step(it)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.25)
    # per-kernel times for the roofline (eager steps through the timed entry point)
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        step(k, timed=True)
    torch.cuda.synchronize()
    # the step itself: the product's captured Adam iteration (MC.AdamGraph), replayed
    ag = MC.AdamGraph(obj, theta0, 0.1, max_iters=1 << 30).capture()
    for _ in range(max(3, args.warmup)):
        ag.graph.replay()
    torch.cuda.synchronize()
    times = []
    for k in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ag.graph.replay()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    assert int(ag.bad.item()) < 0, "non-finite objective in the timed Adam steps"
    clocks = sampler.stop() if sampler else None
    ms = sum(times) / len(times)
    value = B * ws / (ms * 1e-3)
    # e2e: host theta [B, P] in, host loss [B] + gradient [B, P] out, through the public batched
    # objective (MBEObjective.host_evaluator: one captured round trip per call)
    hev = obj.host_evaluator(B)

    def e2e_rate(call, host, batch):
        for _ in range(2):
            call(host)
        et = []
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call(host)
            e1.record(stream)
            e1.synchronize()
            et.append(e0.elapsed_time(e1))
        return batch / (statistics.mean(et) * 1e-3)

    e2e = e2e_rate(hev, theta0, B)
    # and the reference-shaped single-restart fun(theta) -> (loss, grad) (latency bound at B=1)
    fun = MC.mbe_objective(circuit, graph, device=dev, dtype="complex64")
    e2e_single = e2e_rate(fun, theta0[0], 1)
    if rank != 0:
        return
    ffma = ctypes.c_double(0)
    _lib.check(lib.tq_ffma_peak(20000, stream.cuda_stream, ctypes.byref(ffma)))
    from paper_2112_10239_b200 import chain as C

    terms = C.normalize_terms(MC._readout_terms(graph)[1])
    pe = roofline.eval_model(C.compile_chain(circuit, terms, "energy", segments=1), grad=True)
    pv = roofline.eval_model(C.compile_chain(circuit, terms, "values", segments=1), grad=True)
    cand = {"values_sweeps (rl+lr values)": (statistics.mean(kt["values"]), (pv["flops_rl"] + pv["flops_lr"]) * B),
            "rl_sweep (cotangent-weighted)": (statistics.mean(kt["rl"]), pe["flops_rl"] * B),
            "lr_sweep (gradient)": (statistics.mean(kt["lr"]), pe["flops_lr"] * B),
            "adj_sweep (column adjoint)": (statistics.mean(kt["adj"]), pe["flops_adj"] * B)}
    kname = max(cand, key=lambda k: cand[k][0])
    kms, kfl = cand[kname]
    achieved = kfl / (kms * 1e-3) / 1e12
    cpu = None
    if not args.no_cpu_baseline:
        import multiprocessing as mp

        cores = host_cores()
        nsamp = max(2, min(cores, 16))
        jobs = [(list(graph.edges), theta0[i % B]) for i in range(nsamp)]
        with mp.get_context("fork").Pool(min(cores, nsamp)) as pool:
            t0 = time.perf_counter()
            per = pool.map(_mbe_oracle_step, jobs)
            wall = time.perf_counter() - t0
        cpu = {"value": nsamp / wall, "unit": "evals/s", "cores": min(cores, nsamp), "kind": "port",
               "sample": f"{nsamp} MBE objective evaluations (oracle port of tnsim mbe_objective, eps=0), "
                         f"{sum(per):.1f} CPU-s"}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    byts = (pe["bytes"] + pv["bytes"]) * B
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64", "data": "synthetic pairing-model 3-regular graph (seed 3), seeded angles",
        "config": {"workload": f"cfg3: {cfg.description}", "n_qubits": 1024, "vertices": 2048, "edges": 3072,
                   "restarts_per_gpu": B, "segments": obj.dp_energy.plan.n_segments,
                   "chi_max": obj.dp_energy.plan.chi_max, "l2": "flushed between timed steps (256 MiB memset, untimed)",
                   "parallelism": "restarts as the batch dimension",
                   "step": "one replay of the captured Adam iteration (maxcut.AdamGraph)"},
        "roofline": {"bound": "fp32_simt", "kernel": kname, "achieved": achieved, "peak": ffma.value,
                     "unit": "TFLOP/s", "frac": achieved / ffma.value, "traffic": None,
                     "peak_source": "measured FFMA probe (tq_ffma_peak) on this GPU in this run",
                     "kernel_ms": {k: statistics.mean(vv) for k, vv in kt.items()}},
        "hbm": {"achieved_gbs": byts / (ms * 1e-3) / 1e9, "peak_gbs": float(peaks.get("hbm_gbs", 6650.0)),
                "frac": byts / (ms * 1e-3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)), "bytes_per_step": byts},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": hev.h2d_bytes,
                "d2h_bytes_per_step": hev.d2h_bytes,
                "note": f"{B} restarts per call through MBEObjective.host_evaluator (float64 theta [B, P] in, "
                        "loss + float64 gradient out; captured host-buffer graph from the second call); "
                        "no optimizer update",
                "single_restart": {"value": e2e_single, "unit": "evals/s",
                                   "note": "mbe_objective fun(theta) at B=1 (the reference's call shape)"}},
        # per step: fill_identity_values + rl/lr values sweeps, build_wct is skipped (per-restart
        # cotangent rows), rl/lr/adj + reduce_energy/reduce_grad
        "gpu_launches": 8 * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- f3 (truncated TT engine)
F3 = {"n": 500, "gates": 5000, "chi_max": 16, "eps": 0.0}   # the reference's `bench tfim` defaults
F3_METRIC = "truncated TT simulations/sec (simulate_tt + all TFIM term values)"


def f3_problem():
    from paper_2112_10239_b200 import chain as C
    from paper_2112_10239_b200.hamiltonians import tfim
    from paper_2112_10239_b200.report import tfim_workload

    circuit = tfim_workload(F3["n"], F3["gates"])
    return circuit, C.normalize_terms(tfim(F3["n"]))


def _f3_oracle_sim(theta):
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    import oracle as O

    t0 = time.perf_counter()
    oc = O.tfim_workload_gates(F3["n"], F3["gates"])
    tt = O.simulate_tt(oc, theta, eps=F3["eps"], chi_max=F3["chi_max"])
    O.tt_term_values(tt, O.tfim_terms(F3["n"]))
    return time.perf_counter() - t0


def f3_config(batch):
    return {"workload": "f3: reference `bench tfim` defaults, truncated TT engine (SURVEY.md row f3)",
            "n_qubits": F3["n"], "gates": F3["gates"], "chi_max": F3["chi_max"], "eps": F3["eps"],
            "circuit": "tfim_workload: ry+rz rows and alternating cz lines, cut to the gate count",
            "operator": "TFIM open chain j=h=1 (all 999 term values)", "batch_per_gpu": batch,
            "parallelism": "theta-set data parallel (one 128-thread CTA per theta-set, 4 resident per SM)",
            "l2": "flushed between timed steps (256 MiB memset, untimed)"}


def run_f3_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_2112_10239_b200.workloads import theta_sets

    circuit, _ = f3_problem()
    cores = host_cores()
    per = cores
    th = theta_sets(circuit.n_params, per * (args.steps + args.warmup), seed=0)
    with mp.get_context("fork").Pool(cores) as pool:
        for w in range(args.warmup):
            pool.map(_f3_oracle_sim, list(th[w * per:(w + 1) * per]))
        t0 = time.perf_counter()
        for s_ in range(args.steps):
            off = (args.warmup + s_) * per
            pool.map(_f3_oracle_sim, list(th[off:off + per]))
        wall = time.perf_counter() - t0
    value = args.steps * per / wall
    sample = f"{per} truncated simulations per step (oracle port of tnsim simulate_tt + expval windows)"
    print(json.dumps({
        "impl": "reference", "metric": F3_METRIC, "value": value, "unit": "sims/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded angles, float32-rounded)", "config": f3_config(per),
        "cpu_baseline": {"value": value, "unit": "sims/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def run_f3(args):
    """Row f3: B theta-sets of the reference's `bench tfim` workload through the truncated
    engine per step (one tq_tt_simulate launch), complex128 like the reference."""
    import ctypes

    import torch

    from paper_2112_10239_b200 import _lib, truncated as TR
    from paper_2112_10239_b200.workloads import theta_sets

    ws, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    circuit, terms = f3_problem()
    n, T = circuit.n_qubits, len(terms)
    # six 128-thread CTAs (theta-sets) resident per SM (csrc/tq_trunc.cu NT, TQT_MINB): one wave
    B = args.batch or 6 * torch.cuda.get_device_properties(dev).multi_processor_count
    thetas = theta_sets(circuit.n_params, B, seed=rank)
    table, _ = TR.compile_gates(circuit)
    lo, hi, offs, codes = TR.term_table(terms, n)

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    d_gates, d_lo, d_hi, d_offs, d_codes = up(table.view(np.uint8)), up(lo), up(hi), up(offs), up(codes)
    th = torch.tensor(thetas, dtype=torch.float64, device=dev)
    values = torch.zeros(B, T, 2, dtype=torch.float64, device=dev)
    disc = torch.zeros(B, dtype=torch.float64, device=dev)
    norm2 = torch.zeros(B, dtype=torch.float64, device=dev)
    bonds = torch.zeros(B, n + 1, dtype=torch.int32, device=dev)
    flags = torch.zeros(B, dtype=torch.int32, device=dev)
    lib = _lib.load()
    cap = F3["chi_max"]
    wsb = lib.tq_tt_workspace_bytes(n, B, cap, _lib.TQ_C128)
    wsp = torch.empty(int(wsb), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        _lib.check(lib.tq_tt_simulate(n, d_gates.data_ptr(), len(table), _lib.TQ_C128, B, th.data_ptr(), th.stride(0),
                                      ctypes.c_double(F3["eps"]), cap, F3["chi_max"], d_lo.data_ptr(), d_hi.data_ptr(),
                                      d_offs.data_ptr(), d_codes.data_ptr(), T, values.data_ptr(), disc.data_ptr(),
                                      norm2.data_ptr(), bonds.data_ptr(), flags.data_ptr(), wsp.data_ptr(),
                                      ctypes.c_size_t(int(wsb)), stream.cuda_stream))

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    assert not bool(flags.any()) and bool(torch.isfinite(values).all())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.25)
    times = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks = sampler.stop() if sampler else None
    ms = statistics.mean(times)
    if ws > 1:
        import torch.distributed as dist

        if not dist.is_initialized():
            _init_dist(dist, dev)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    value = B * ws / (ms * 1e-3)
    # e2e: host angles in, host values out, through the public entry
    e2e_t = []
    for i in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        TR.simulate_terms(circuit, terms, thetas, F3["eps"], F3["chi_max"], dtype="complex128")
        e2e_t.append(time.perf_counter() - t0)
    e2e = B * ws / statistics.mean(e2e_t[1:] if len(e2e_t) > 1 else e2e_t)
    if rank != 0:
        return
    model = TR.work_model(circuit, terms, F3["chi_max"])
    peak = ctypes.c_double(0)
    _lib.check(lib.tq_tt_dfma_peak(2000, stream.cuda_stream, ctypes.byref(peak)))
    achieved = model["flops"] * B / (ms * 1e-3) / 1e12
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        import multiprocessing as mp

        cores = host_cores()
        nsamp = min(cores, 16)
        with mp.get_context("fork").Pool(nsamp) as pool:
            t0 = time.perf_counter()
            per = pool.map(_f3_oracle_sim, list(thetas[:nsamp]) if nsamp <= B else list(thetas))
            wall = time.perf_counter() - t0
        cpu = {"value": len(per) / wall, "unit": "sims/s", "cores": nsamp, "kind": "port",
               "sample": f"{len(per)} truncated simulations, one per process (oracle port of tnsim simulate_tt "
                         f"+ expval windows), {sum(per):.1f} CPU-s"}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("f3", {}).get("tt_kernel")
        except Exception:
            traffic = None
    print(json.dumps({
        "metric": F3_METRIC, "value": value, "unit": "sims/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded angles, float32-rounded)",
        "config": f3_config(B),
        "roofline": {"bound": "fp64_simt", "kernel": "tt_kernel", "achieved": achieved, "peak": peak.value,
                     "unit": "TFLOP/s", "frac": achieved / peak.value if peak.value else None, "traffic": traffic,
                     "peak_source": "measured DFMA probe (tq_tt_dfma_peak) on this GPU in this run",
                     "flops_per_sim": model["flops"], "svd_flops_per_sim": model["svd_flops"],
                     "work_model": "truncated.work_model (LAPACK-style counts; DESIGN.md section 11)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": "sims/s", "h2d_bytes_per_step": int(thetas.nbytes),
                "d2h_bytes_per_step": int(B * T * 16 + B * 8 * 2 + B * (n + 1) * 4 + B * 4)},
        "gpu_launches": args.steps,
        "clocks": clocks,
        "results": {"max_bond": int(bonds.max()), "discarded_weight_max": float(disc.max())},
    }), flush=True)


def relaunch_under_torchrun(n: int) -> int:
    """``--gpus N`` outside torchrun: re-exec this command as N ranks (one per GPU) on this node,
    exactly as the driver launches it.  Returns the launcher's exit code."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "f3"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--segments", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check", action="store_true",
                    help="also compare the (sharded) results with a single-process evaluation")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using the launcher's {ws} ranks", file=sys.stderr)
    from paper_2112_10239_b200.workloads import CONFIGS

    if args.config == "f3":
        run_f3_reference(args) if args.impl == "reference" else run_f3(args)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.config == "cfg3":
        run_cfg3(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
