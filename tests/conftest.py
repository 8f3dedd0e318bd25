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
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs under gpurun / the round-end GPU tier)")
    config.addinivalue_line("markers", "slow: multi-second CPU work")


@pytest.fixture(scope="session")
def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cfg1_golden():
    return dict(np.load(os.path.join(GOLDEN, "cfg1.npz")))


def parents_to_edges(parents):
    return [(int(parents[v]), v) for v in range(1, len(parents))]


CFG_TEMPLATES = {
    "cfg1": [-1, 0, 1, 1, 3],
    "cfg2": [-1, 0, 0, 1, 1, 2, 2],
    "cfg3": [-1, 0, 1, 2, 0, 4, 4, 6, 0, 8, 9, 9],
    "cfg4": [-1, 0, 1, 2, 3, 0, 5, 6, 0, 8, 8, 10, 10, 12, 13],
    "cfg5": [-1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 11, 0, 14, 15],
}
