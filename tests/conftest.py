import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def dec(s: str, n: int) -> np.ndarray:
    """Golden matrix string ('0'/'1'/'2' row-major) -> uint8 [n, n] classes."""
    return np.frombuffer(s.encode(), dtype=np.uint8).reshape(n, n) - ord("0")


def centred(a: np.ndarray):
    return [[(-1 if v == 2 else int(v)) for v in row] for row in np.asarray(a)]


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o


@pytest.fixture(scope="session")
def gpu():
    """The product package, after checking a B200 is present (skip otherwise)."""
    import paper_2407_20205_b200 as tp
    from paper_2407_20205_b200 import _kernels

    if _kernels.device_count() < 1:
        pytest.skip("no sm_100 device")
    return tp
