"""Synthetic workloads of BASELINE.json (reading-A layer semantics).

A "layer" is one TTCircuit unitary: even layers are a trainable rotation row,
odd layers an entangler line on pairs (q, q+1), q = p (mod 2), with p
alternating 0,1,0,... over successive lines.  Angles come from
``init_params(P, generator(seed))`` / ``spawn`` (reference autodiff.py:609-611,
seeding.py:14-22) and are rounded to float32 once, so every consumer (GPU
engine, CPU oracle) sees identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuits import Circuit, standard_gate
from .hamiltonians import tfim
from .seeding import generator, spawn


def layered_circuit(n: int, layers: int, rot: str = "ry", ent: str = "cz") -> Circuit:
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


def f32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def theta_sets(n_params: int, batch: int, seed: int = 0) -> np.ndarray:
    """[batch, P] float64 holding float32-exact values; set b = init_params(P, spawn(seed, batch)[b])."""
    if batch == 1:
        return f32(generator(seed).uniform(-np.pi, np.pi, size=n_params))[None]
    return np.stack([f32(r.uniform(-np.pi, np.pi, size=n_params)) for r in spawn(seed, batch)])


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    layers: int
    rot: str
    ent: str
    batch: int
    grad: bool
    description: str

    def circuit(self) -> Circuit:
        return layered_circuit(self.n, self.layers, self.rot, self.ent)

    def hamiltonian(self):
        return tfim(self.n)


CONFIGS = {
    "cfg1": Config("cfg1", 10, 4, "ry", "cnot", 256, True,
                   "TTCircuit 10 qubits, 4 layers RotY+CNOT, TFIM energy+gradient"),
    "cfg2": Config("cfg2", 100, 10, "ry", "cz", 256, True,
                   "TTCircuit 100 qubits, 10 layers RotY+CZ, TFIM energy+gradient, 256 parameter sets"),
    "cfg3": Config("cfg3", 1024, 4, "ry+rz", "cz", 8, True,
                   "MBE MaxCut, random 3-regular graph V=2048 (3072 edges), brickwork_ansatz(1024, 4), "
                   "one Adam step (loss + gradient) per restart"),
    "cfg4": Config("cfg4", 1000, 20, "ry", "cz", 64, True,
                   "TTCircuit 1000 qubits, 20 layers RotY+CZ, TFIM energy+gradient"),
    "cfg5": Config("cfg5", 1024, 10, "ry", "cz", 64, False,
                   "TTCircuit 1024*g qubits, 10 layers RotY+CZ, TFIM energy (weak scaling per GPU)"),
}
