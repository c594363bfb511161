"""Golden vectors for the truncated TT engine (row f3), made by the REAL reference
(tnsim.tt.simulate_tt with eps / chi_max, then tnsim.hamiltonians.expval).

Usage (build container only): python tests/golden/make_golden_trunc.py -> golden_trunc.json
The theta vectors are float32-rounded, as in make_golden.py.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
from make_golden import circ_doc, f32, ham_doc, layers_circuit, rand_circuit  # noqa: E402
from tnsim.circuits import with_params  # noqa: E402
from tnsim.hamiltonians import PauliHamiltonian, expval, term, tfim  # noqa: E402
from tnsim.seeding import generator  # noqa: E402
from tnsim.tt import compress, simulate_tt, tt_to_dense  # noqa: E402


def case(name, circ, ham, theta, eps, chi_max):
    tt = simulate_tt(with_params(circ, theta), eps=eps, chi_max=chi_max)
    return {"name": name, "circuit": circ_doc(circ), "ham": ham_doc(ham), "theta": [float(x) for x in theta],
            "eps": eps, "chi_max": chi_max, "value": float(expval(tt, ham)),
            "discarded": float(tt.discarded_weight), "bonds": [int(b) for b in tt.bond_dims]}


def main():
    rng = generator(5)
    cases = []
    for i, (n, layers, ent, eps, chi) in enumerate([(10, 10, "cnot", 0.0, 4), (12, 12, "cz", 0.0, 8),
                                                    (11, 9, "cnot", 1e-3, None), (12, 14, "cz", 1e-2, 6),
                                                    (9, 12, "cnot", 0.0, 3), (14, 10, "cz", 1e-4, 16)]):
        c = layers_circuit(n, layers, "ry", ent)
        th = f32(rng.uniform(-np.pi, np.pi, c.n_params))
        cases.append(case(f"layers{i}", c, tfim(n), th, eps, chi))
    for i in range(4):
        n = 8 + i
        c = rand_circuit(rng, n, 60, 0.4, adjacent_only=False)
        th = f32(rng.uniform(-np.pi, np.pi, c.n_params))
        ham = tfim(n, 0.7, 1.1) + PauliHamiltonian(n, (term(0.3, {0: "Y", 3: "X"}), term(-0.2, {1: "Z", n - 1: "Y"})))
        cases.append(case(f"random{i}", c, ham, th, (0.0, 1e-3, 1e-2, 0.0)[i], (4, None, 5, 6)[i]))
    # compress (tt.py:299-320) of an exact / truncated train, with the dense amplitudes of
    # the result (gauge-free) for n <= 10
    comp = []
    for i, (n, layers, ent, eps0, chi0, eps, chi) in enumerate([(10, 10, "cz", 0.0, None, 0.0, 4),
                                                                (10, 12, "cnot", 0.0, 8, 1e-2, None),
                                                                (9, 10, "cz", 0.0, None, 1e-3, 6)]):
        c = layers_circuit(n, layers, "ry", ent)
        th = f32(rng.uniform(-np.pi, np.pi, c.n_params))
        tt0 = simulate_tt(with_params(c, th), eps=eps0, chi_max=chi0)
        tt = compress(tt0, eps, chi)
        psi = tt_to_dense(tt).amplitudes.array.reshape(-1)
        comp.append({"name": f"compress{i}", "circuit": circ_doc(c), "ham": ham_doc(tfim(n)),
                     "theta": [float(x) for x in th], "eps0": eps0, "chi0": chi0, "eps": eps, "chi_max": chi,
                     "value": float(expval(tt, tfim(n))), "discarded": float(tt.discarded_weight),
                     "bonds": [int(b) for b in tt.bond_dims], "bonds0": [int(b) for b in tt0.bond_dims],
                     "psi_re": [float(x) for x in psi.real], "psi_im": [float(x) for x in psi.imag]})
    with open(os.path.join(HERE, "golden_trunc.json"), "w") as f:
        json.dump({"cases": cases, "compress": comp}, f)
    for c in comp:
        print(c["name"], c["value"], c["discarded"], c["bonds"])
    for c in cases:
        print(c["name"], c["value"], c["discarded"], max(c["bonds"]))


if __name__ == "__main__":
    main()
