"""Goldens for the exact plans ``bench.py`` times, made by running the REAL reference
(``tnsim``) in the build container (it does not travel to the GPU box).

* cfg4 bench batch (n=1000, 20 layers, B=64, theta_b = init_params(10000, spawn(0, 64)[b])):
  E for b in {0, 31, 63} and 32 parameter-shift coordinates of b=0 and 16 of b=63
  (``parameter_shift_grad`` semantics: 0.5 (E(t + pi/2) - E(t - pi/2)), autodiff.py:514-550).
* cfg4 golden set (init_params(10000, generator(0))): 28 more shift coordinates, so with the
  4 in golden_large.npz the set has 32.
* cfg5 bench batch at n=1024 (10 layers, B=64, spawn(0, 64)): E for b in {0, 63}.
* cfg5 at n=8192 (init_params(40960, generator(0))): E (64.1075367256).

Forward values use ``evaluate_expval(engine="tt", eps=1e-12)``, which keeps the true Schmidt
rank.  Runs the forwards on a process pool (one BLAS thread each).

Usage: python tests/golden/make_golden_bench.py [--procs 8] [--skip8192]
"""

from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _setup():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def layers_circuit(n, layers, rot="ry", ent="cz"):
    from tnsim.circuits import Circuit, standard_gate

    gates, train = [], []
    for l in range(layers):
        if l % 2 == 0:
            for q in range(n):
                train.append(len(gates))
                gates.append(standard_gate(rot, (q,), 0.0))
        else:
            p = (l // 2) % 2
            for q in range(p, n - 1, 2):
                gates.append(standard_gate(ent, (q, q + 1)))
    return Circuit(n, tuple(gates), tuple(train))


def _forward(job):
    _setup()
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    from tnsim.autodiff import evaluate_expval
    from tnsim.hamiltonians import tfim

    key, n, layers, theta = job
    t0 = time.time()
    e = evaluate_expval(layers_circuit(n, layers), tfim(n), theta, engine="tt", eps=1e-12)
    return key, float(e), time.time() - t0


def thetas_spawn(P, B, seed=0):
    _setup()
    from tnsim.autodiff import init_params
    from tnsim.seeding import spawn

    return np.stack([f32(init_params(P, r)) for r in spawn(seed, B)])


def theta_gen(P, seed=0):
    _setup()
    from tnsim.autodiff import init_params
    from tnsim.seeding import generator

    return f32(init_params(P, generator(seed)))


def shift_jobs(tag, n, layers, theta, coords):
    jobs = []
    for k in coords:
        for sgn in (+1, -1):
            t = theta.copy()
            t[k] += sgn * np.pi / 2
            jobs.append(((tag, int(k), sgn), n, layers, t))
    return jobs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--skip8192", action="store_true")
    a = ap.parse_args()
    _setup()
    from tnsim.seeding import generator

    res = {}
    th4 = thetas_spawn(10000, 64)
    th5 = thetas_spawn(5 * 1024, 64)
    g0 = theta_gen(10000)
    old = dict(np.load(os.path.join(HERE, "golden_large.npz")))
    assert np.array_equal(old["cfg4_theta"], g0)
    c_b0 = np.sort(generator(45).choice(10000, size=32, replace=False))
    c_b63 = np.sort(generator(46).choice(10000, size=16, replace=False))
    rest = [int(k) for k in np.sort(generator(47).choice(10000, size=64, replace=False)) if k not in set(old["cfg4_coords"])][:28]
    c_g0 = np.array(sorted(rest))
    jobs = []
    if not a.skip8192:
        jobs.append((("cfg5_8192",), 8192, 10, theta_gen(5 * 8192)))
    for b in (0, 31, 63):
        jobs.append((("cfg4E", b), 1000, 20, th4[b]))
    for b in (0, 63):
        jobs.append((("cfg5E", b), 1024, 10, th5[b]))
    jobs += shift_jobs("b0", 1000, 20, th4[0], c_b0)
    jobs += shift_jobs("b63", 1000, 20, th4[63], c_b63)
    jobs += shift_jobs("g0", 1000, 20, g0, c_g0)
    print(f"{len(jobs)} forward evaluations on {a.procs} processes", flush=True)
    out = {}
    t0 = time.time()
    with mp.get_context("spawn").Pool(a.procs) as pool:
        for key, e, dt in pool.imap_unordered(_forward, jobs):
            out[key] = e
            print(f"{time.time() - t0:7.1f}s {key} E={e!r} ({dt:.1f}s)", flush=True)

    def shifts(tag, coords):
        return np.array([0.5 * (out[(tag, int(k), 1)] - out[(tag, int(k), -1)]) for k in coords])

    res.update(cfg4b_theta_idx=np.array([0, 31, 63]), cfg4b_E=np.array([out[("cfg4E", b)] for b in (0, 31, 63)]),
               cfg4b_coords_b0=c_b0, cfg4b_shift_b0=shifts("b0", c_b0),
               cfg4b_coords_b63=c_b63, cfg4b_shift_b63=shifts("b63", c_b63),
               cfg4_coords_more=c_g0, cfg4_shift_more=shifts("g0", c_g0),
               cfg5b_theta_idx=np.array([0, 63]), cfg5b_E=np.array([out[("cfg5E", b)] for b in (0, 63)]))
    if not a.skip8192:
        res["cfg5_8192_E"] = np.array(out[("cfg5_8192",)])
    np.savez_compressed(os.path.join(HERE, "golden_bench.npz"), **res)
    print("wrote golden_bench.npz", {k: (v if v.size < 4 else v.shape) for k, v in res.items()})


if __name__ == "__main__":
    main()
