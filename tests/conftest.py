import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "golden_small.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_large():
    path = os.path.join(GOLDEN, "golden_large.npz")
    if not os.path.exists(path):
        pytest.skip("golden_large.npz not generated")
    return dict(np.load(path))


def ocircuit(doc):
    from oracle import OCircuit

    return OCircuit(doc["n"], [(g[0], tuple(g[1]), g[2]) for g in doc["gates"]], list(doc["trainable"]))


def oterms(doc):
    return [(complex(re, im), tuple((int(q), l) for q, l in ops)) for re, im, ops in doc]
