import os
import sys

# BLAS single-threaded like the reference suite (pkg/tests/conftest.py:3-6)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import pytest  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
