"""Goldens for row f1 (the MBE MaxCut optimisation loop), made by running the REAL reference
(``tnsim``) in the build container: ``minimize`` (autodiff.py:614-659) on ``mbe_objective``
(maxcut.py:219-252) per restart, and ``solve_maxcut`` (maxcut.py:273-319) end to end.

For each case: the graph, the restarts' initial angles (``init_params`` on
``spawn(seed, restarts)``, float64 as the reference draws them), every restart's
per-iteration loss and gradient norm, its final theta, and solve_maxcut's result.

Usage (build container only): python tests/golden/make_golden_f1.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from tnsim.autodiff import init_params, minimize  # noqa: E402
from tnsim.maxcut import Graph, brickwork_ansatz, mbe_encode, mbe_objective, solve_maxcut  # noqa: E402
from tnsim.seeding import generator, spawn  # noqa: E402


def rand_graph(V, p, seed):
    rng = generator(seed)
    edges = []
    for u in range(V):
        for w in range(u + 1, V):
            if rng.random() < p:
                edges.append((u, w, float(rng.uniform(0.2, 1.5))))
    return Graph(V, tuple(edges))


def case(name, graph, depth, restarts, iters, seed, optimizer="adam", rate=0.1, alpha=1.0):
    n, _ = mbe_encode(graph)
    circ = brickwork_ansatz(n, depth)
    fun = mbe_objective(circ, graph, alpha=alpha, engine="tt")
    runs = []
    for rng in spawn(seed, restarts):
        th0 = init_params(circ.n_params, rng)
        res = minimize(fun, th0, optimizer=optimizer, rate=rate, max_iters=iters)
        runs.append({"theta0": th0.tolist(), "loss": [s.value for s in res.steps],
                     "gnorm": [s.grad_norm for s in res.steps], "theta_final": res.theta.tolist(),
                     "converged": res.converged})
    sol = solve_maxcut(graph, depth=depth, engine="tt", optimizer=optimizer, rate=rate, restarts=restarts,
                       max_iters=iters, seed=seed, alpha=alpha)
    return {"name": name, "V": graph.num_vertices, "edges": [list(e) for e in graph.edges], "depth": depth,
            "restarts": restarts, "max_iters": iters, "seed": seed, "optimizer": optimizer, "rate": rate,
            "alpha": alpha, "runs": runs,
            "solve": {"assignment": list(sol.assignment), "cut": sol.cut_value, "loss": sol.relaxed_loss,
                      "iters": sol.iterations, "restart_index": sol.restart_index}}


def main():
    cases = [case("g10_adam", rand_graph(10, 0.5, 101), 3, 3, 25, 5),
             case("g12_adam", rand_graph(12, 0.4, 202), 4, 2, 25, 9),
             case("g11_gd", rand_graph(11, 0.45, 303), 3, 2, 20, 13, optimizer="gd", rate=0.05, alpha=1.3)]
    with open(os.path.join(HERE, "golden_f1.json"), "w") as fh:
        json.dump({"cases": cases}, fh)
    for c in cases:
        print(c["name"], c["solve"]["cut"], [r["loss"][-1] for r in c["runs"]])


if __name__ == "__main__":
    main()
