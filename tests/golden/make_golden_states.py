"""Goldens for ARBITRARY tensor-train input states, made by running the REAL reference (tnsim) in
the build container: a random TTState (tt.py:38-76, ortho_center None), every gate of a circuit
applied with apply_gate_tt(eps=0) (tt.py:186-234), then expval (hamiltonians.py:167-187) and
tt_inner (tt.py:247-255) with a second random train, plus the exact gradient of the energy by the
reference's own parameter-shift rule on those evaluations (the function is c + a cos t + b sin t
in every angle).

Usage (build container only): python tests/golden/make_golden_states.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)
sys.dont_write_bytecode = True

from tnsim.circuits import with_params  # noqa: E402
from tnsim.hamiltonians import expval, tfim  # noqa: E402
from tnsim.seeding import generator  # noqa: E402
from tnsim.tt import TTState, apply_gate_tt, tt_inner  # noqa: E402

from make_golden import circ_doc, f32, ham_doc, layers_circuit, rand_circuit, rand_ham  # noqa: E402


def rand_train(rng, n, chi):
    dims = [1] + [int(rng.integers(1, chi + 1)) for _ in range(n - 1)] + [1]
    cores = [(rng.normal(size=(dims[k], 2, dims[k + 1])) + 1j * rng.normal(size=(dims[k], 2, dims[k + 1])))
             / np.sqrt(2 * dims[k + 1]) for k in range(n)]
    return TTState(n, tuple(cores))


def run(c, th, state):
    tt = state
    for g in with_params(c, th).gates:
        tt = apply_gate_tt(tt, g, eps=0.0)
    return tt


def main():
    rng = generator(2024)
    cases = []
    specs = [(6, 4, layers_circuit(6, 4, "ry", "cz"), None), (7, 3, None, "rand"), (5, 2, layers_circuit(5, 6, "rx", "cnot"), None),
             (8, 4, layers_circuit(8, 4, "ry", "cz"), None)]
    for i, (n, chi, c, kind) in enumerate(specs):
        if c is None:
            c = rand_circuit(rng, n, 18, 0.5, adjacent_only=True)
        th = f32(rng.uniform(-np.pi, np.pi, c.n_params))
        h = tfim(n) if i % 2 == 0 else rand_ham(rng, n, 4)
        a, b = rand_train(rng, n, chi), rand_train(rng, n, chi)
        out = run(c, th, a)
        e = expval(out, h)
        from tnsim.autodiff import _CRZ_Y1, _CRZ_Y2

        def shifted(k, d):
            t = th.copy()
            t[k] += d
            return expval(run(c, t, a), h)

        grad = []
        for k in range(c.n_params):   # the reference's shift rules (autodiff.py:509-550)
            if c.gates[c.trainable[k]].name == "crz":
                grad.append(_CRZ_Y1 * (shifted(k, np.pi / 2) - shifted(k, -np.pi / 2))
                            - _CRZ_Y2 * (shifted(k, 3 * np.pi / 2) - shifted(k, -3 * np.pi / 2)))
            else:
                grad.append(0.5 * (shifted(k, np.pi / 2) - shifted(k, -np.pi / 2)))
        ip = tt_inner(b, out)
        ip_in = tt_inner(a, b)
        cases.append({"name": f"state{i}", "circuit": circ_doc(c), "ham": ham_doc(h), "theta": th.tolist(),
                      "state": [[x.real.tolist(), x.imag.tolist()] for x in a.cores],
                      "other": [[x.real.tolist(), x.imag.tolist()] for x in b.cores],
                      "energy": float(e), "grad": grad, "inner_other_out": [ip.real, ip.imag],
                      "inner_state_other": [ip_in.real, ip_in.imag], "out_bonds": list(out.bond_dims)})
        print(cases[-1]["name"], e, np.linalg.norm(grad), ip)
    with open(os.path.join(HERE, "golden_states.json"), "w") as fh:
        json.dump({"cases": cases}, fh)


if __name__ == "__main__":
    main()
