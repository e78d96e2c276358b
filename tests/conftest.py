import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def cfg1_data():
    """BASELINE cfg1 data, regenerated from its seed and checked against the
    digest the reference-run fixture recorded."""
    import hashlib
    from oracle import gen_random_dense
    x = gen_random_dense(10000, 100, 1001)
    g = golden("train.npz")
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(g["cfg1_xsha"])
    return x


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)   # reference conftest.py:47-49
