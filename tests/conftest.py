import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "golden.json")) as fh:
        meta = json.load(fh)
    return {
        "meta": meta,
        "rng": np.load(os.path.join(d, "rng_construct.npz")),
        "plans": np.load(os.path.join(d, "plans.npz")),
        "adj": np.load(os.path.join(d, "adjacency.npz")),
        "runs": np.load(os.path.join(d, "runs.npz")),
        "big": np.load(os.path.join(d, "big.npz")),
        "bigp": np.load(os.path.join(d, "bigp.npz")) if os.path.exists(os.path.join(d, "bigp.npz")) else {},
    }
