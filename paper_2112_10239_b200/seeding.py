"""Deterministic random streams (mirrors reference ``tnsim/seeding.py:14-22``): PCG64
generators and SeedSequence.spawn child streams, so CPU oracle and GPU engine consume
bit-identical angles."""

from __future__ import annotations

import numpy as np


def generator(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def spawn(seed: int, n_children: int) -> list:
    return [np.random.Generator(np.random.PCG64(s)) for s in np.random.SeedSequence(seed).spawn(n_children)]
