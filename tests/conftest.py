"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device and the built libmpmm_cuda.so;
everything else runs on CPU (the oracle, host logic, ABI symbols, gloo
multi-process sharding).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture
def dd():
    from paper_1710_01839_b200 import PrecisionSpec
    return PrecisionSpec.dd()


@pytest.fixture
def qd():
    from paper_1710_01839_b200 import PrecisionSpec
    return PrecisionSpec.qd()


@pytest.fixture
def gpu():
    """Skip-free guard: a gpu-marked test on a box without CUDA fails loudly."""
    import torch
    assert torch.cuda.is_available(), "gpu test collected on a host without CUDA"
    from paper_1710_01839_b200 import _cuda
    _cuda.load()
    return torch.device("cuda", 0)


def random_int_matrix(rng, m, n, prec, bound=8):
    from paper_1710_01839_b200 import DenseMatrix
    return DenseMatrix.from_ints([[rng.randint(-bound, bound) for _ in range(n)]
                                  for _ in range(m)], prec)
