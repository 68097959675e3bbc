import itertools
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libkc.so")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# edge-array builders (same graphs as the reference's tests/conftest.py:29-73)
def complete_edges(n):
    return np.array(list(itertools.combinations(range(n), 2)), dtype=np.int64).reshape(-1, 2)


def cycle_edges(n):
    return np.array([(i, (i + 1) % n) for i in range(n)], dtype=np.int64)


def path_edges(n):
    return np.array([(i, i + 1) for i in range(n - 1)], dtype=np.int64).reshape(-1, 2)


def star_edges(leaves):
    return np.array([(leaves, i) for i in range(leaves)], dtype=np.int64)


def bipartite_edges(a, b):
    return np.array([(i, a + j) for i in range(a) for j in range(b)], dtype=np.int64)


def petersen_edges():
    pairs = []
    for i in range(5):
        pairs += [(i, (i + 1) % 5), (i, i + 5), (5 + i, 5 + (i + 2) % 5)]
    return np.array(pairs, dtype=np.int64)


def gnp_edges(n, p, seed):
    rng = np.random.default_rng(seed)
    pairs = complete_edges(n)
    kept = pairs[rng.random(len(pairs)) < p]
    return kept if kept.shape[0] else pairs[:1]


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def kc():
    """The GPU package; gpu tests fail loudly (no skip) when it cannot run."""
    import paper_2104_13209_b200 as pkg
    from paper_2104_13209_b200 import _lib

    _lib.load()
    assert _lib.device_count() > 0, "gpu test without a visible CUDA device"
    return pkg
