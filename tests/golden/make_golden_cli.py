"""Golden RunReports from the REAL reference CLI (``tnsim.cli``), for the f4 parity tests.

Usage (build container only): python tests/golden/make_golden_cli.py
Writes golden_cli.json: the circuit / Hamiltonian / graph documents the reference writes,
and the reference's RunReport (minus ``measured``) for each command run on them.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
import tnsim.cli as cli  # noqa: E402
from tnsim.circuits import Circuit, circuit_to_dict, standard_gate  # noqa: E402
from tnsim.hamiltonians import PauliHamiltonian, hamiltonian_to_dict, term, tfim  # noqa: E402


def f32(x):
    return float(np.float32(x))


def docs():
    rng = np.random.default_rng(11)
    bell = Circuit(2, (standard_gate("h", (0,)), standard_gate("cnot", (0, 1))))
    ry = Circuit(2, (standard_gate("ry", (0,), 0.7), standard_gate("cnot", (0, 1))), trainable=(0,))
    g = []
    for layer in range(3):
        for q in range(5):
            g.append(standard_gate(("ry", "rx", "rz")[layer], (q,), f32(rng.uniform(-np.pi, np.pi))))
        for q in range(layer % 2, 4, 2):
            g.append(standard_gate(("cz", "cnot", "cz")[layer], (q, q + 1)))
    g.append(standard_gate("crz", (1, 2), f32(0.37)))
    g.append(standard_gate("h", (3,)))
    g.append(standard_gate("s", (4,)))
    mixed = Circuit(5, tuple(g), tuple(i for i, x in enumerate(g) if x.name in ("ry", "rx", "rz", "crz")))
    z0 = PauliHamiltonian(2, (term(1.0, {0: "Z"}),))
    h5 = tfim(5, 0.8, 1.3) + PauliHamiltonian(5, (term(0.25, {0: "Y", 2: "X", 4: "Z"}), term(-0.5, {})))
    return {"bell": circuit_to_dict(bell), "ry": circuit_to_dict(ry), "mixed": circuit_to_dict(mixed)}, \
           {"z0": hamiltonian_to_dict(z0), "h5": hamiltonian_to_dict(h5)}


def run(argv):
    out = io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(io.StringIO()):
        code = cli.run_cli(argv)
    assert code == 0, argv
    rep = json.loads(out.getvalue())
    rep.pop("measured")
    return rep


def main():
    circuits, hams = docs()
    runs = []
    with tempfile.TemporaryDirectory() as tmp:
        for k, v in {**circuits, **hams}.items():
            with open(os.path.join(tmp, k + ".json"), "w") as f:
                json.dump(v, f)
        with open(os.path.join(tmp, "tri.txt"), "w") as f:
            f.write("# triangle\n0 1\n1 2\n0 2\n")
        p = lambda k: os.path.join(tmp, k + ".json")  # noqa: E731
        cases = [
            ("expval", ["expval", "--circuit", p("bell"), "--ham", p("z0"), "--engine", "tt"], ("bell", "z0")),
            ("expval", ["expval", "--circuit", p("mixed"), "--ham", p("h5"), "--engine", "tt"], ("mixed", "h5")),
        ]
        for m in ("ad", "shift", "fd"):
            cases.append(("grad", ["grad", "--circuit", p("ry"), "--ham", p("z0"), "--method", m], ("ry", "z0", m)))
        for m in ("ad", "shift"):
            cases.append(("grad", ["grad", "--circuit", p("mixed"), "--ham", p("h5"), "--method", m,
                                   "--engine", "tt"], ("mixed", "h5", m)))
        cases.append(("simulate", ["simulate", "--circuit", p("mixed"), "--engine", "dense"], ("mixed",)))
        cases.append(("simulate", ["simulate", "--circuit", p("bell"), "--engine", "dense"], ("bell",)))
        cases.append(("bench", ["bench", "tfim", "--n", "4", "--gates", "25", "--chi", "8", "--seed", "2"], ()))
        cases.append(("bench", ["bench", "tfim", "--n", "6", "--gates", "60", "--chi", "16", "--seed", "4"], ()))
        cases.append(("bench", ["bench", "tfim", "--n", "2", "--gates", "0", "--seed", "0", "--no-grad"], ()))
        # truncating runs (row f3): chi below the exact bond, eps > 0
        cases.append(("bench", ["bench", "tfim", "--n", "12", "--gates", "260", "--chi", "4", "--seed", "3",
                                "--no-grad"], ()))
        cases.append(("bench", ["bench", "tfim", "--n", "10", "--gates", "300", "--chi", "16", "--eps", "1e-3",
                                "--seed", "5", "--no-grad"], ()))
        cases.append(("expval", ["expval", "--circuit", p("mixed"), "--ham", p("h5"), "--engine", "tt",
                                 "--chi", "2"], ("mixed", "h5", "chi2")))
        cases.append(("grad", ["grad", "--circuit", p("mixed"), "--ham", p("h5"), "--method", "shift",
                               "--engine", "tt", "--chi", "2"], ("mixed", "h5", "shift", "chi2")))
        cases.append(("simulate", ["simulate", "--circuit", p("mixed"), "--engine", "tt", "--chi", "2"],
                      ("mixed", "chi2")))
        cases.append(("simulate", ["simulate", "--circuit", p("mixed"), "--engine", "tt"], ("mixed", "tt")))
        for kind, argv, key in cases:
            rep = run(argv)
            runs.append({"kind": kind, "key": list(key), "argv_tail": [a for a in argv if not a.startswith(tmp)],
                         "report": rep})
    with open(os.path.join(HERE, "golden_cli.json"), "w") as f:
        json.dump({"circuits": circuits, "hams": hams, "runs": runs}, f, indent=1)
    print("wrote", len(runs), "reports")


if __name__ == "__main__":
    main()
