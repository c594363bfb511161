"""Race / uninitialised-read stress (compute-sanitizer is closed on this pool).

usage: python tools/race_stress.py OUT.npz [reps]
Runs every sweep path (tools/sanitize_case.py's coverage plus the cfg2 and cfg4 bench plans at
small batch) `reps` times with the library named by TQ_ENGINE_LIB, checks the repeats are
bitwise identical and finite, and saves the first repeat.  tools/race_check.sh runs it with
the production library and with libtq_engine_debug.so (poisoned shared memory, randomly
delayed barriers: csrc/tq_debug.cuh) and compares the two bit for bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_10239_b200 import _lib  # noqa: E402
from paper_2112_10239_b200 import autodiff as AD  # noqa: E402
from paper_2112_10239_b200 import chain as C  # noqa: E402
from paper_2112_10239_b200 import truncated as TR  # noqa: E402
from paper_2112_10239_b200.hamiltonians import tfim  # noqa: E402
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets  # noqa: E402


def cases():
    out = {}
    for n, layers, ent, segs, B in ((10, 4, "cnot", None, 8), (24, 10, "cz", 2, 4), (20, 12, "cz", 3, 4),
                                    (14, 20, "cz", 2, 3), (100, 10, "cz", None, 16), (200, 20, "cz", 2, 4)):
        c = layered_circuit(n, layers, "ry", ent)
        th = theta_sets(c.n_params, B, seed=n)
        for dt in ("complex64", "complex128"):
            if dt == "complex128" and C.factored_chi(n, C.time_gates(c)) > 16:
                continue
            v, g = AD.grad_expval(c, tfim(n), th, segments=segs, dtype=dt)
            out[f"E_{n}_{layers}_{dt}"], out[f"g_{n}_{layers}_{dt}"] = v, g
        out[f"vals_{n}_{layers}"] = AD.expectation_values(c, th, [{0: "Z"}, {3: "X", 4: "Z"}, {n - 1: "Y"}],
                                                          segments=segs)
    c = layered_circuit(8, 4)
    out["inner"] = np.array(AD.state_inner_product(c, theta_sets(c.n_params, 1, seed=2)[0], c,
                                                   theta_sets(c.n_params, 1, seed=3)[0]))
    c = layered_circuit(12, 8)
    terms = C.normalize_terms(tfim(12))
    th = theta_sets(c.n_params, 3, seed=4)
    res = TR.simulate_terms(c, terms, th, 0.0, 4)
    out["trunc_vals"], out["trunc_disc"] = res.values, res.discarded
    v, g = TR.straight_through(c, terms, th, 0.0, 2)
    out["st_vals"], out["st_grad"] = v, g
    return out


def main():
    path = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    print("library:", _lib.LIB_PATH)
    first = cases()
    for k, v in first.items():
        assert np.all(np.isfinite(np.asarray(v))), f"non-finite output {k}"
    for r in range(1, reps):
        again = cases()
        for k in first:
            if not np.array_equal(np.asarray(first[k]), np.asarray(again[k])):
                raise SystemExit(f"repeat {r}: {k} differs (max {np.max(np.abs(np.asarray(first[k]) - np.asarray(again[k])))})")
    np.savez(path, **{k: np.asarray(v) for k, v in first.items()})
    print(f"{len(first)} outputs finite and bitwise identical over {reps} repeats -> {path}")


if __name__ == "__main__":
    main()
