import os
import sys

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
GOLDEN_F = os.path.join(ROOT, "tests", "golden", "golden_f.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def single_threaded_blas():
    """The reference states every determinism contract for a 1-thread BLAS
    (reference tests/conftest.py:9-18); the oracle runs the same way."""
    with threadpool_limits(limits=1):
        yield


@pytest.fixture(scope="session")
def golden():
    g = np.load(GOLDEN)
    meta = dict(zip(g["meta_keys"].tolist(), g["meta_vals"].tolist()))
    return g, meta


@pytest.fixture(scope="session")
def golden_f():
    """Reference outputs for the §8 (f) rows (tests/golden/make_golden_f.py)."""
    return np.load(GOLDEN_F)


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


GOLDEN_ALG = os.path.join(ROOT, "tests", "golden", "golden_alg.npz")
ALG_CASES = ("f64", "f64c", "f32", "f32c")


@pytest.fixture(scope="session")
def golden_alg():
    """Reference basic_rand_svd / legacy_single_pass outputs (§8 (f) rank 4,
    tests/golden/make_golden_alg.py)."""
    return np.load(GOLDEN_ALG)
