"""Goldens for the straight-through gradient through truncated splits, made by running the REAL
reference (``tnsim``) in the build container: ``grad_expval(engine="tt", eps, chi_max)`` with a
binding truncation (autodiff.py:315-363,471-487), the CLI's ``grad --chi`` (method ad) and
``bench tfim --grad --chi`` reports (bench.py:99-156).

Usage (build container only): python tests/golden/make_golden_st.py
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)
sys.dont_write_bytecode = True

import tnsim.cli as cli  # noqa: E402
from tnsim.autodiff import grad_expval, init_params  # noqa: E402
from tnsim.circuits import Circuit, circuit_from_dict, standard_gate  # noqa: E402
from tnsim.hamiltonians import PauliHamiltonian, hamiltonian_from_dict, term, tfim  # noqa: E402
from tnsim.seeding import generator  # noqa: E402

from make_golden import circ_doc, f32, ham_doc, layers_circuit, rand_circuit, rand_ham  # noqa: E402


class SplitWatch:
    """Collects every taped split's spectrum while a reference call runs, and says whether the
    straight-through gradient is well posed: it freezes U_k (or Vh_k), which is unique up to
    phases only if no KEPT singular value is zero while the factor is not square, and no
    singular value at the cut is degenerate with the first dropped one (otherwise LAPACK's basis
    choice inside a degenerate subspace decides the gradient, and any other SVD gives an equally
    valid but different straight-through value)."""

    def __init__(self, eps, chi):
        self.eps, self.chi, self.ok, self.n = eps, chi, True, 0

    def __enter__(self):
        import tnsim.autodiff as A
        from tnsim.tt import _truncate_spectrum

        self._orig = A.np.linalg.svd
        watch = self

        def svd(mat, full_matrices=False):
            u, sv, vh = watch._orig(mat, full_matrices=False)
            m, n = mat.shape
            k, _, _ = _truncate_spectrum(sv, watch.eps, watch.chi)
            side = m if m <= n else n
            if sv.size and sv[0] > 0:
                tiny = 1e-9 * sv[0]
                if k < side and sv[k - 1] <= tiny:
                    watch.ok = False
                if k < sv.size and sv[k - 1] - sv[k] <= tiny:
                    watch.ok = False
            watch.n += 1
            return u, sv, vh

        A.np.linalg.svd = svd
        return self

    def __exit__(self, *a):
        import tnsim.autodiff as A

        A.np.linalg.svd = self._orig


def case(name, c, h, eps, chi):
    th = np.array([c.gates[i].param for i in c.trainable], dtype=float)
    with SplitWatch(eps, chi) as w:
        v, g = grad_expval(c, h, th, engine="tt", eps=eps, chi_max=chi)
    return {"name": name, "circuit": circ_doc(c), "ham": ham_doc(h), "theta": th.tolist(), "eps": eps,
            "chi_max": chi, "value": v, "grad": g.tolist(), "well_posed": w.ok, "splits": w.n}


def with_theta(c, th):
    gates = list(c.gates)
    for slot, gi in enumerate(c.trainable):
        g = gates[gi]
        gates[gi] = standard_gate(g.name, g.wires, float(th[slot]))
    return Circuit(c.n_qubits, tuple(gates), c.trainable)


def run_cli(argv):
    out = io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(io.StringIO()):
        code = cli.run_cli(argv)
    assert code == 0, argv
    rep = json.loads(out.getvalue())
    rep.pop("measured")
    return rep


def main():
    cases = []
    rng = generator(777)
    for r in range(6):
        n = int(rng.integers(3, 8))
        c = rand_circuit(rng, n, int(rng.integers(14, 30)), 0.5, adjacent_only=(r % 2 == 0))
        h = rand_ham(rng, n, int(rng.integers(2, 6))) if r % 2 else tfim(n)
        cases.append(case(f"random{r}_chi{1 + r % 2}", c, h, 0.0, 1 + r % 2))
    for r in range(6):
        n = int(rng.integers(4, 9))
        c = rand_circuit(rng, n, int(rng.integers(20, 40)), 0.5, adjacent_only=(r % 3 != 0))
        h = rand_ham(rng, n, int(rng.integers(2, 6))) if r % 2 else tfim(n)
        cases.append(case(f"random_eps{r}", c, h, 0.03 * (1 + r), None))
    c = layers_circuit(8, 8, "ry", "cz")
    cases.append(case("ry_cz_8x8_chi2", with_theta(c, f32(init_params(c.n_params, generator(5)))), tfim(8), 0.0, 2))
    c = layers_circuit(10, 6, "rx", "cnot")
    cases.append(case("rx_cnot_10x6_eps", with_theta(c, f32(init_params(c.n_params, generator(6)))), tfim(10), 0.05, None))
    c = layers_circuit(9, 10, "ry", "cz")
    cases.append(case("ry_cz_9x10_chi3", with_theta(c, f32(init_params(c.n_params, generator(7)))),
                      tfim(9, periodic=True), 0.0, 3))
    # the CLI: grad --method ad through truncation, and bench tfim --grad with a binding chi
    from make_golden_cli import docs
    circs, hams = docs()
    cli_runs = []
    with tempfile.TemporaryDirectory() as tmp:
        cp, hp = os.path.join(tmp, "mixed.json"), os.path.join(tmp, "h5.json")
        json.dump(circs["mixed"], open(cp, "w"))
        json.dump(hams["h5"], open(hp, "w"))
        for extra, eps, chi in ((["--chi", "2"], 0.0, 2), (["--chi", "3"], 0.0, 3), (["--eps", "0.2"], 0.2, None)):
            argv = ["grad", "--engine", "tt"] + extra
            with SplitWatch(eps, chi) as w:
                rep = run_cli(argv[:1] + ["--circuit", cp, "--ham", hp] + argv[1:])
            cli_runs.append({"argv": ["grad", "--circuit", "mixed", "--ham", "h5", "--engine", "tt"] + extra,
                             "report": rep, "well_posed": w.ok})
    for n, gates, chi, eps in ((20, 300, 2, 0.0), (40, 2000, 4, 0.0), (30, 900, 3, 0.0), (24, 600, 8, 1e-3),
                               (500, 5000, 16, 0.0)):   # the last: the reference's `bench tfim` defaults
        argv = ["bench", "tfim", "--n", str(n), "--gates", str(gates), "--chi", str(chi), "--eps", str(eps)]
        with SplitWatch(eps, chi) as w:
            rep = run_cli(argv)
        cli_runs.append({"argv": argv, "report": rep, "well_posed": w.ok})
    # MBE MaxCut through truncated splits (maxcut.py:206-319 with eps / chi_max)
    from tnsim.maxcut import Graph, brickwork_ansatz, mbe_objective, solve_maxcut, vertex_expectations
    small = json.load(open(os.path.join(HERE, "golden_small.json")))["mbe10"]
    graph = Graph(10, tuple((int(u), int(v), float(w)) for u, v, w in small["edges"]))
    bw = brickwork_ansatz(5, small["depth"])
    mbe = []
    for eps, chi in ((0.0, 2), (0.15, None)):
        with SplitWatch(eps, chi) as w:
            loss, grad = mbe_objective(bw, graph, alpha=small["alpha"], engine="tt", eps=eps, chi_max=chi)(
                np.array(small["theta"]))
            ev = vertex_expectations(bw, np.array(small["theta"]), graph, engine="tt", eps=eps, chi_max=chi)
            sol = solve_maxcut(graph, depth=small["depth"], engine="tt", eps=eps, chi_max=chi, restarts=2,
                               max_iters=6, seed=3, alpha=small["alpha"])
        mbe.append({"eps": eps, "chi_max": chi, "loss": loss, "grad": grad.tolist(), "vertex": ev.tolist(),
                    "solve": {"assignment": list(sol.assignment), "cut": sol.cut_value, "loss": sol.relaxed_loss,
                              "iters": sol.iterations, "restart_index": sol.restart_index},
                    "well_posed": w.ok})
        print("mbe", eps, chi, loss, w.ok, sol.cut_value)
    with open(os.path.join(HERE, "golden_st.json"), "w") as fh:
        json.dump({"cases": cases, "cli": cli_runs, "mbe": mbe}, fh)
    for c in cases:
        print(c["name"], c["value"], np.linalg.norm(c["grad"]), "well_posed", c["well_posed"], c["splits"])
    for r in cli_runs:
        print(r["argv"], r["well_posed"], {k: r["report"]["outputs"].get(k) for k in ("value", "grad_value", "grad_norm")})


if __name__ == "__main__":
    main()
