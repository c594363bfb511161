"""``tq`` command line: the reference CLI's hot-path subcommands on the B200 engine (row f4).

Mirrors ``tnsim.cli`` (``cli.py:70-160,238-248,274-332``):
- ``expval``, ``grad --method ad|shift|fd``, ``simulate``, ``maxcut`` and ``bench tfim``;
- every subcommand prints one RunReport (JSON, or ``--format csv`` rows);
- the same file formats (circuit / Hamiltonian JSON, edge-list graphs);
- the same exit codes: 0 ok, 2 input errors (missing or malformed files, bad flags), 1
  numerical errors.

Differences:
- ``--engine`` takes the reference's choices with the reference's default: ``dense`` (exact
  values, ``--eps``/``--chi`` ignored, at most 26 qubits) and ``tt`` (``b200`` is an alias).
  Both run on the B200 engines; ``dense`` is their exact path.
- ``--eps`` / ``--chi`` select the truncated TT engine (row f3) whenever they can truncate.
  ``grad --method ad`` then returns the reference's straight-through gradient of its taped
  truncated state (autodiff.py:10-13,315-363; truncated.straight_through); ``shift`` and ``fd``
  work as in the reference, on truncated forwards.
- ``ptrace`` and ``paths`` (density matrices, contraction-order search) are outside the hot
  path and are not offered.
- ``--dtype`` picks complex128 (default, the reference's precision) or complex64.
- ``simulate`` reports the norm, bond dimensions and discarded weight of the truncated
  engine's run.  That run repeats the reference's simulate_tt.  For n <= 8, when nothing
  was discarded, it also reports the amplitudes <x|psi>, each computed on the GPU as a
  batched inner product against the basis product states.

Run as ``python -m paper_2112_10239_b200.cli ...``.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

import numpy as np

from . import __version__
from .errors import InputError, NumericalError, ParseError
from .report import RunReport, bench_tfim, bond_profile, device_info, measure

AMPLITUDE_DUMP_LIMIT = 8   # reference cli.py:42


def _read_text(path: str) -> str:
    try:
        return Path(path).read_text()
    except OSError as exc:
        raise InputError(f"cannot read {path}: {exc}")


def _read_json(path: str) -> dict:
    try:
        return json.loads(_read_text(path))
    except json.JSONDecodeError as exc:
        raise ParseError(f"{path}: {exc}")


def _engine_kwargs(args) -> dict:
    # 'dense' keeps the reference's meaning (exact values, eps/chi ignored, 26-qubit guard),
    # computed by the B200 engine (autodiff._engine_args)
    return {"engine": "dense" if args.engine == "dense" else "tt", "eps": args.eps, "chi_max": args.chi,
            "dtype": args.dtype}


def _load(args, ham: bool = True):
    from .circuits import circuit_from_dict
    from .hamiltonians import hamiltonian_from_dict

    circuit = circuit_from_dict(_read_json(args.circuit))
    return circuit, (hamiltonian_from_dict(_read_json(args.ham)) if ham else None)


def evaluate_expval(*a, **k):   # module-level seams (monkeypatched by the CLI tests, as in the reference)
    from .autodiff import evaluate_expval as f
    return f(*a, **k)


def _measured(name: str, ms: float, peak: int) -> dict:
    return {"wall_ms": {name: ms}, "peak_bytes": peak, "device": device_info()}


def _cmd_expval(args) -> RunReport:
    circuit, ham = _load(args)
    kw = _engine_kwargs(args)
    value, ms, peak = measure(lambda: evaluate_expval(circuit, ham, **kw))
    return RunReport("expval", args.seed,
                     {"circuit": args.circuit, "ham": args.ham, "engine": args.engine, "chi": args.chi,
                      "eps": args.eps, "dtype": args.dtype},
                     {"value": float(value), "n_qubits": circuit.n_qubits, "n_terms": len(ham.terms)},
                     _measured("expval", ms, peak))


def _cmd_grad(args) -> RunReport:
    from . import autodiff as AD

    circuit, ham = _load(args)
    kw = _engine_kwargs(args)
    theta = circuit.params()

    def run():
        if args.method == "ad":
            return AD.grad_expval(circuit, ham, theta, **kw)
        if args.method == "shift":
            g = AD.parameter_shift_grad(circuit, ham, theta, **kw)
        else:
            g = AD.finite_diff_grad(circuit, ham, theta, engine=kw["engine"], eps=args.eps, chi_max=args.chi,
                                    dtype=args.dtype)
        return evaluate_expval(circuit, ham, theta, **kw), g

    (value, grad), ms, peak = measure(run)
    grad = np.asarray(grad, dtype=float)
    return RunReport("grad", args.seed,
                     {"circuit": args.circuit, "ham": args.ham, "engine": args.engine, "chi": args.chi,
                      "eps": args.eps, "method": args.method, "dtype": args.dtype},
                     {"value": float(value), "gradient": [float(g) for g in grad],
                      "grad_norm": float(np.linalg.norm(grad)), "n_params": circuit.n_params},
                     _measured("grad", ms, peak))


def amplitudes(circuit, dtype: str = "complex128") -> np.ndarray:
    """<x|psi> for every basis state x (qubit 0 most significant, the reference's dense
    ravel order): one batched inner-product launch.  The bra of row x is ry(pi*x_q) on
    every qubit: ry(pi)|0> = |1> up to cos(pi/2) ~ 6e-17."""
    from . import autodiff as AD
    from .circuits import Circuit, standard_gate

    n = circuit.n_qubits
    bra = Circuit(n, tuple(standard_gate("ry", (q,), 0.0) for q in range(n)), tuple(range(n)))
    xs = np.arange(1 << n)
    bits = (xs[:, None] >> (n - 1 - np.arange(n))[None, :]) & 1
    ket_theta = np.repeat(circuit.params()[None, :], len(xs), axis=0)
    return np.asarray(AD.state_inner_product(circuit, ket_theta, bra, np.pi * bits, dtype=dtype))


def _cmd_simulate(args) -> RunReport:
    from . import autodiff as AD
    from . import truncated as TR
    from .errors import BondTooLarge

    circuit, _ = _load(args, ham=False)
    if args.engine == "dense":   # the reference's exact state-vector path: no truncation
        AD._engine_args("dense", circuit, 0.0, None)
        args.eps, args.chi = 0.0, None
    truncating = AD._truncating(circuit, args.eps, args.chi)

    def run():
        try:   # the truncated engine repeats the reference's simulate_tt: same bonds, weight, norm
            res = TR.simulate_terms(circuit, [], circuit.params()[None, :], args.eps, args.chi, dtype=args.dtype)
            bonds, disc, nrm2 = [int(x) for x in res.bonds[0]], float(res.discarded[0]), float(res.norm2[0])
        except BondTooLarge:
            if truncating:
                raise
            nrm2 = float(np.real(AD.state_inner_product(circuit, circuit.params(), circuit, circuit.params(),
                                                        dtype=args.dtype)))
            bonds, disc = bond_profile(circuit), 0.0
        # amplitudes of the exact state: identical to the truncated one when nothing was discarded
        small = circuit.n_qubits <= AMPLITUDE_DUMP_LIMIT and (not truncating or disc < 1e-24)
        amps = amplitudes(circuit, args.dtype) if small else None
        return float(np.sqrt(max(nrm2, 0.0))), bonds, disc, amps

    (norm, bonds, disc, amps), ms, peak = measure(run)
    outputs = {"n_qubits": circuit.n_qubits, "engine": args.engine, "norm": norm, "bond_dims": bonds,
               "discarded_weight": disc}
    if amps is not None:
        outputs["amplitudes"] = [[float(a.real), float(a.imag)] for a in amps]
    return RunReport("simulate", args.seed,
                     {"circuit": args.circuit, "engine": args.engine, "chi": args.chi, "eps": args.eps,
                      "dtype": args.dtype},
                     outputs, _measured("simulate", ms, peak))


def _cmd_maxcut(args) -> RunReport:
    from .maxcut import MAX_BRUTE_FORCE_VERTICES, brute_force_maxcut, load_graph, result_to_dict, solve_maxcut

    graph = load_graph(_read_text(args.graph))
    result, ms, peak = measure(lambda: solve_maxcut(graph, depth=args.depth, restarts=args.restarts,
                                                    max_iters=args.max_iters, seed=args.seed, alpha=args.alpha,
                                                    threads=args.threads))
    optimal = brute_force_maxcut(graph)[0] if graph.num_vertices <= MAX_BRUTE_FORCE_VERTICES else None
    return RunReport("maxcut", args.seed,
                     {"graph": args.graph, "depth": args.depth, "restarts": args.restarts, "alpha": args.alpha,
                      "max_iters": args.max_iters, "num_vertices": graph.num_vertices,
                      "num_edges": len(graph.edges)},
                     result_to_dict(result, optimal), _measured("solve", ms, peak))


def _cmd_bench(args) -> RunReport:
    return bench_tfim(n_qubits=args.n, n_gates=args.gates, chi_max=args.chi, grad=args.grad, eps=args.eps,
                      seed=args.seed, dtype=args.dtype)


def _common(sp) -> None:
    sp.add_argument("--seed", type=int, default=0, help="master RNG seed")
    sp.add_argument("--format", choices=("json", "csv"), default="json")
    sp.add_argument("--threads", type=int, default=1, help="accepted for compatibility (restarts are batched)")
    sp.add_argument("--dtype", choices=("complex128", "complex64"), default="complex128")


def _engine(sp) -> None:
    sp.add_argument("--engine", choices=("dense", "tt", "b200"), default="dense")
    sp.add_argument("--chi", type=int, default=None, help="TT bond cap (truncated engine when it binds)")
    sp.add_argument("--eps", type=float, default=0.0, help="TT relative truncation threshold")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="tq", description="B200 TT-circuit expectation values, gradients, benchmarks")
    ap.add_argument("--version", action="version", version=__version__)
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("expval", help="expectation value of a Pauli sum")
    p.add_argument("--circuit", required=True)
    p.add_argument("--ham", required=True)
    _engine(p)
    _common(p)
    p = sub.add_parser("grad", help="gradient of an expectation value")
    p.add_argument("--circuit", required=True)
    p.add_argument("--ham", required=True)
    p.add_argument("--method", choices=("ad", "shift", "fd"), default="ad")
    _engine(p)
    _common(p)
    p = sub.add_parser("simulate", help="norm, bonds and (n <= 8) amplitudes of a circuit state")
    p.add_argument("--circuit", required=True)
    _engine(p)
    _common(p)
    p = sub.add_parser("maxcut", help="MBE MaxCut on an edge-list graph")
    p.add_argument("--graph", required=True)
    p.add_argument("--depth", type=int, default=4)
    p.add_argument("--restarts", type=int, default=5)
    p.add_argument("--alpha", type=float, default=1.0)
    p.add_argument("--max-iters", type=int, default=300)
    _common(p)
    p = sub.add_parser("bench", help="benchmark workloads")
    bsub = p.add_subparsers(dest="bench_kind", required=True)
    bt = bsub.add_parser("tfim", help="TFIM energy (+gradient) of the brickwork stream")
    bt.add_argument("--n", type=int, default=500)
    bt.add_argument("--gates", type=int, default=5000)
    bt.add_argument("--chi", type=int, default=16)
    bt.add_argument("--grad", action=argparse.BooleanOptionalAction, default=True)
    bt.add_argument("--eps", type=float, default=0.0)
    _common(bt)
    return ap


_DISPATCH = {"expval": _cmd_expval, "grad": _cmd_grad, "simulate": _cmd_simulate, "maxcut": _cmd_maxcut,
             "bench": _cmd_bench}


def _flat(obj, prefix="", into=None):
    into = {} if into is None else into
    for k, v in obj.items():
        key = prefix + str(k)
        if isinstance(v, dict):
            _flat(v, key + ".", into)
        else:
            into[key] = json.dumps(v) if isinstance(v, list) else v
    return into


def emit(report: RunReport, fmt: str, stream=None) -> None:
    stream = sys.stdout if stream is None else stream
    if fmt == "json":
        json.dump(report.to_dict(), stream, indent=2)
        stream.write("\n")
        return
    row = _flat(report.outputs, into={"command": report.command, "version": report.version, "seed": report.seed})
    row["wall_ms"] = sum(report.measured.get("wall_ms", {}).values())
    w = csv.DictWriter(stream, fieldnames=list(row))
    w.writeheader()
    w.writerow(row)


def run_cli(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return 0 if not exc.code else int(exc.code)
    try:
        report = _DISPATCH[args.command](args)
    except InputError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except NumericalError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    emit(report, args.format)
    return 0


def main() -> None:
    sys.exit(run_cli())


if __name__ == "__main__":
    main()
