"""RunReport records and the ``bench tfim`` workload on the B200 engine.

The record has the reference's shape (``bench.py:32-51``, schema
``schemas/runreport.schema.json``): ``command``, ``version``, ``seed``, ``inputs``, ``outputs``
and ``measured``.  Everything outside ``measured`` reproduces exactly for a fixed seed.

``measured`` keeps the reference's keys with GPU meaning:
- ``wall_ms`` holds host wall-clock phases, taken after a device synchronize;
- ``peak_bytes`` is the device allocator's high-water mark above the entry level (the
  reference reports host ``tracemalloc`` peaks, which inflate its timings 2.4-3.9x, SURVEY.md
  section 8d);
- ``device`` is extra, and is allowed by the schema.
"""

from __future__ import annotations

import time
from collections import Counter
from dataclasses import dataclass

import numpy as np

from . import __version__
from .circuits import Circuit, standard_gate
from .errors import InputError
from .hamiltonians import tfim


@dataclass(frozen=True)
class RunReport:
    """One CLI / benchmark record (reference bench.py:32-51)."""

    command: str
    seed: int | None
    inputs: dict
    outputs: dict
    measured: dict
    version: str = __version__

    def to_dict(self) -> dict:
        return {"command": self.command, "version": self.version, "seed": self.seed,
                "inputs": dict(self.inputs), "outputs": dict(self.outputs), "measured": dict(self.measured)}


def measure(fn):
    """(result, wall_ms, device peak bytes above entry) of ``fn()``; the device is
    synchronized on both sides so the wall time covers the kernels."""
    import torch

    cuda = torch.cuda.is_available()
    if cuda:
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
    t0 = time.perf_counter_ns()
    out = fn()
    if cuda:
        torch.cuda.synchronize()
    ms = (time.perf_counter_ns() - t0) / 1e6
    peak = max(0, torch.cuda.max_memory_allocated() - base) if cuda else 0
    return out, ms, int(peak)


def device_info() -> dict:
    import torch

    if not torch.cuda.is_available():
        return {"name": None}
    p = torch.cuda.get_device_properties(torch.cuda.current_device())
    return {"name": p.name, "sms": p.multi_processor_count, "engine": "libtq_engine (sm_100a)"}


def tfim_workload(n_qubits: int, n_gates: int) -> Circuit:
    """Brickwork stream cut to exactly ``n_gates`` gates (reference bench.py:70-96).

    Per layer: an ry row, an rz row (all trainable), then a cz line on pairs starting at
    ``layer % 2``.  The stream may stop mid-row."""
    if n_qubits < 1:
        raise InputError("workload needs at least one qubit")
    if n_gates < 0:
        raise InputError("gate count must be non-negative")
    gates, train = [], []
    layer = 0

    def room():
        return len(gates) < n_gates

    while room():
        for rot in ("ry", "rz"):
            q = 0
            while q < n_qubits and room():
                train.append(len(gates))
                gates.append(standard_gate(rot, (q,), 0.0))
                q += 1
        q = layer % 2
        while q < n_qubits - 1 and room():
            gates.append(standard_gate("cz", (q, q + 1)))
            q += 2
        layer += 1
    return Circuit(n_qubits, tuple(gates), tuple(train))


def bond_profile(circuit: Circuit) -> list:
    """Exact bond dimensions over the n+1 cuts of the factored chain (1 at both ends):
    the engine's chi_k = 2^(binary gates straddling cut k)."""
    from . import chain as C

    n = circuit.n_qubits
    bits = np.zeros(n + 1, dtype=np.int64)
    for g in C.time_gates(circuit):
        if g.bits:
            bits[g.lo + 1: g.hi + 1] += g.bits
    return [int(1 << int(b)) for b in bits]


def bench_tfim(n_qubits: int = 500, n_gates: int = 5000, chi_max: int | None = 16, grad: bool = True,
               eps: float = 0.0, j: float = 1.0, h: float = 1.0, seed: int = 0, *,
               dtype: str = "complex128") -> RunReport:
    """TFIM energy (and gradient) of ``tfim_workload`` on the B200 engines
    (reference bench.py:99-156, same inputs/outputs keys).

    The forward phase runs the truncated TT engine (row f3, ``truncated.py``), which repeats
    the reference's simulate_tt with (eps, chi_max).  ``expval``, ``max_bond``,
    ``bond_histogram`` and ``discarded_weight`` therefore follow the reference's semantics.
    The gradient phase is ``grad_expval(eps, chi_max)`` as in the reference: the exact engine
    when (eps, chi_max) truncate nothing, else the reference's straight-through gradient of its
    taped truncated state (``truncated.straight_through``, autodiff.py:10-13,315-363), whose
    ``grad_value`` is the taped construction's energy."""
    from . import autodiff as AD
    from . import chain as C
    from . import truncated as TR
    from .seeding import generator

    wall = {}

    def build():
        circuit = tfim_workload(n_qubits, n_gates)
        return circuit, tfim(n_qubits, j, h), AD.init_params(circuit.n_params, generator(seed))

    (circuit, ham, theta), wall["build"], _ = measure(build)
    terms = C.normalize_terms(ham)

    def forward():
        return TR.simulate_terms(circuit, terms, theta, eps, chi_max, dtype=dtype)

    res, wall["forward"], peak = measure(forward)
    value = res.energy([c for c, _ in terms])[0].real
    bonds = [int(x) for x in res.bonds[0]]
    hist = Counter(bonds)
    outputs = {"gate_count": len(circuit.gates), "n_qubits": n_qubits, "n_params": circuit.n_params,
               "chi_max": chi_max, "expval": float(value), "max_bond": int(max(bonds)),
               "bond_histogram": {str(k): int(v) for k, v in sorted(hist.items())},
               "discarded_weight": float(res.discarded[0])}
    if grad:
        (gval, gvec), wall["gradient"], pk = measure(lambda: AD.grad_expval(circuit, ham, theta, eps=eps,
                                                                            chi_max=chi_max, dtype=dtype))
        peak = max(peak, pk)
        outputs["grad_value"] = float(gval)
        outputs["grad_norm"] = float(np.linalg.norm(gvec))
        outputs["grad_finite"] = bool(np.all(np.isfinite(gvec)))
    inputs = {"n": n_qubits, "gates": n_gates, "chi_max": chi_max, "grad": bool(grad), "eps": eps, "j": j, "h": h}
    return RunReport("bench tfim", seed, inputs, outputs,
                     {"wall_ms": wall, "peak_bytes": int(peak), "device": device_info()})
