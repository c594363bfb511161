"""Generate golden vectors by running the REAL reference (``tnsim``) in the build
container.  The reference does not travel to the GPU box, so its outputs are
committed here as fixtures (``golden_small.json``, ``golden_large.npz``).

Usage (build container only):  python tests/golden/make_golden.py [--large]

Every angle vector is rounded to float32 first and that exact value (as
float64) is what the reference sees, so the GPU engine consumes bit-identical
inputs.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import tnsim  # noqa: E402
from tnsim.autodiff import evaluate_expval, grad_expval, init_params, parameter_shift_grad  # noqa: E402
from tnsim.circuits import Circuit, standard_gate  # noqa: E402
from tnsim.hamiltonians import PauliHamiltonian, term, tfim  # noqa: E402
from tnsim.maxcut import Graph, brickwork_ansatz, mbe_objective, round_cut, cut_value, vertex_expectations  # noqa: E402
from tnsim.seeding import generator, spawn  # noqa: E402
from tnsim.tt import simulate_tt, tt_inner  # noqa: E402


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def layers_circuit(n, layers, rot="ry", ent="cz"):
    """Reading-A generator."""
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


def circ_doc(c):
    return {"n": c.n_qubits, "gates": [[g.name, list(g.wires), g.param] for g in c.gates],
            "trainable": list(c.trainable)}


def ham_doc(h):
    return [[t.coeff.real, t.coeff.imag, [[q, l] for q, l in t.ops]] for t in h.terms]


ONE = ("h", "x", "y", "z", "s", "t", "rx", "ry", "rz")
TWO = ("cnot", "cz", "crz", "swap")
PARAM = ("rx", "ry", "rz", "crz")


def rand_circuit(rng, n, n_gates, p_two, adjacent_only):
    gates, train = [], []
    for _ in range(n_gates):
        if n >= 2 and rng.random() < p_two:
            name = TWO[int(rng.integers(len(TWO)))]
            if adjacent_only:
                q = int(rng.integers(n - 1))
                wires = (q, q + 1) if rng.random() < 0.5 else (q + 1, q)
            else:
                wires = tuple(int(w) for w in rng.choice(n, size=2, replace=False))
        else:
            name = ONE[int(rng.integers(len(ONE)))]
            wires = (int(rng.integers(n)),)
        param = float(f32(rng.uniform(-np.pi, np.pi))) if name in PARAM else None
        if param is not None:
            train.append(len(gates))
        gates.append(standard_gate(name, wires, param))
    return Circuit(n, tuple(gates), tuple(train))


def rand_ham(rng, n, n_terms):
    terms = []
    for _ in range(n_terms):
        k = int(rng.integers(1, min(n, 3) + 1))
        qs = sorted(int(q) for q in rng.choice(n, size=k, replace=False))
        terms.append(term(float(rng.uniform(-1, 1)), {q: "XYZ"[int(rng.integers(3))] for q in qs}))
    return PauliHamiltonian(n, tuple(terms))


def small():
    out = {"reference": f"tnsim {tnsim.__version__} at {REF}", "cases": []}
    # cfg1 (SURVEY.md section 8c golden recipe)
    c1 = layers_circuit(10, 4, "ry", "cnot")
    th = f32(init_params(20, generator(0)))
    v, g = grad_expval(c1, tfim(10), th, engine="tt", eps=0.0)
    out["cases"].append({"name": "cfg1", "circuit": circ_doc(c1), "ham": ham_doc(tfim(10)),
                         "theta": th.tolist(), "value": v, "grad": g.tolist()})
    # cfg2 first four theta-sets
    c2 = layers_circuit(100, 10, "ry", "cz")
    for b, rng in enumerate(spawn(0, 256)[:4]):
        th = f32(init_params(500, rng))
        t0 = time.time()
        v, g = grad_expval(c2, tfim(100), th, engine="tt", eps=0.0)
        print(f"cfg2[{b}] {time.time() - t0:.2f}s E={v}")
        out["cases"].append({"name": f"cfg2_b{b}", "circuit": circ_doc(c2), "ham": ham_doc(tfim(100)),
                             "theta": th.tolist(), "value": v, "grad": g.tolist()})
    # random adjacent-gate circuits over the full gate set, random Pauli sums
    rng = generator(4242)
    for r in range(12):
        n = int(rng.integers(2, 8))
        c = rand_circuit(rng, n, int(rng.integers(6, 16)), 0.4, adjacent_only=(r % 3 != 2))
        h = rand_ham(rng, n, int(rng.integers(1, 6))) if r % 2 else tfim(n, j=float(f32(rng.uniform(0.5, 1.5))),
                                                                         h=float(f32(rng.uniform(0.5, 1.5))))
        th = np.array([c.gates[i].param for i in c.trainable])
        v, g = grad_expval(c, h, th, engine="tt", eps=0.0)
        vd, gd = grad_expval(c, h, th, engine="dense")
        out["cases"].append({"name": f"random{r}", "circuit": circ_doc(c), "ham": ham_doc(h),
                             "theta": th.tolist(), "value": v, "grad": g.tolist(),
                             "value_dense": vd, "grad_dense": gd.tolist()})
    # periodic TFIM on a reading-A circuit
    c = layers_circuit(7, 6, "ry", "cz")
    th = f32(init_params(c.n_params, generator(9)))
    h = tfim(7, periodic=True)
    v, g = grad_expval(c, h, th, engine="tt", eps=0.0)
    out["cases"].append({"name": "periodic7", "circuit": circ_doc(c), "ham": ham_doc(h),
                         "theta": th.tolist(), "value": v, "grad": g.tolist()})
    # rx/rz reading-A variants
    for rot, ent in (("rx", "cz"), ("rz", "cnot"), ("rx", "cnot")):
        c = layers_circuit(9, 6, rot, ent)
        th = f32(init_params(c.n_params, generator(11)))
        v, g = grad_expval(c, tfim(9), th, engine="tt", eps=0.0)
        out["cases"].append({"name": f"{rot}_{ent}_9", "circuit": circ_doc(c), "ham": ham_doc(tfim(9)),
                             "theta": th.tolist(), "value": v, "grad": g.tolist()})
    # MBE MaxCut on a 10-vertex random graph (reference test_maxcut.py:229-245 shape)
    grng = generator(91)
    edges = []
    for u in range(10):
        for w in range(u + 1, 10):
            if grng.random() < 0.5:
                edges.append((u, w, float(f32(grng.uniform(0.1, 1.0)))))
    graph = Graph(10, tuple(edges))
    bw = brickwork_ansatz(5, 3)
    th = f32(grng.uniform(-np.pi, np.pi, bw.n_params))
    fun = mbe_objective(bw, graph, alpha=1.3, engine="tt")
    loss, grad = fun(th)
    ev = vertex_expectations(bw, th, graph, engine="tt")
    asg = round_cut(ev)
    out["mbe10"] = {"edges": [list(e) for e in edges], "depth": 3, "alpha": 1.3, "theta": th.tolist(),
                    "loss": loss, "grad": grad.tolist(), "vertex": ev.tolist(),
                    "assignment": list(asg), "cut": cut_value(graph, asg)}
    # tt_inner of two reading-A states
    ca = layers_circuit(8, 4, "ry", "cz")
    ta = f32(init_params(ca.n_params, generator(21)))
    tb = f32(init_params(ca.n_params, generator(22)))
    from tnsim.circuits import with_params
    ip = tt_inner(simulate_tt(with_params(ca, ta), eps=0.0), simulate_tt(with_params(ca, tb), eps=0.0))
    out["inner8"] = {"circuit": circ_doc(ca), "theta_a": ta.tolist(), "theta_b": tb.tolist(),
                     "re": ip.real, "im": ip.imag}
    with open(os.path.join(HERE, "golden_small.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote golden_small.json")


def large():
    """cfg3 full objective; cfg4 energy + sampled shift gradient; cfg5 energy."""
    res = {}
    # cfg3: pairing graph from generator(3), theta from the same rng
    rng = generator(3)
    V = 2048
    while True:
        stubs = np.repeat(np.arange(V), 3)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        keys = {(min(u, v), max(u, v)) for u, v in pairs}
        if all(u != v for u, v in pairs) and len(keys) == len(pairs):
            break
    edges = tuple((int(u), int(v), 1.0) for u, v in pairs)
    graph = Graph(V, edges)
    bw = brickwork_ansatz(1024, 4)
    th = f32(init_params(bw.n_params, rng))
    t0 = time.time()
    loss, grad = mbe_objective(bw, graph, engine="tt")(th)
    ev = vertex_expectations(bw, th, graph, engine="tt")
    print(f"cfg3 {time.time() - t0:.1f}s loss={loss}")
    asg = np.array(round_cut(ev), dtype=np.int8)
    res.update(cfg3_edges=np.array(pairs, dtype=np.int32), cfg3_theta=th, cfg3_loss=loss, cfg3_grad=grad,
               cfg3_vertex=ev, cfg3_assignment=asg, cfg3_cut=cut_value(graph, tuple(int(a) for a in asg)))
    # cfg4
    c4 = layers_circuit(1000, 20, "ry", "cz")
    th4 = f32(init_params(10000, generator(0)))
    t0 = time.time()
    e4 = evaluate_expval(c4, tfim(1000), th4, engine="tt", eps=1e-12)
    print(f"cfg4 E {time.time() - t0:.1f}s E={e4}")
    coords = np.sort(generator(44).choice(10000, size=4, replace=False))
    sub = Circuit(c4.n_qubits, c4.gates, c4.trainable)
    g4 = np.zeros(len(coords))
    for i, k in enumerate(coords):
        t = th4.copy(); t[k] += np.pi / 2
        ep = evaluate_expval(sub, tfim(1000), t, engine="tt", eps=1e-12)
        t = th4.copy(); t[k] -= np.pi / 2
        em = evaluate_expval(sub, tfim(1000), t, engine="tt", eps=1e-12)
        g4[i] = 0.5 * (ep - em)
        print(f"cfg4 shift coord {k}: {g4[i]}")
    res.update(cfg4_theta=th4, cfg4_E=e4, cfg4_coords=coords, cfg4_shift=g4)
    np.savez_compressed(os.path.join(HERE, "golden_large.npz"), **res)
    print("wrote golden_large.npz")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    a = ap.parse_args()
    if a.large:
        large()
    else:
        small()
