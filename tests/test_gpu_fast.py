"""The opt-in faithful DD mode (mode="fast"): not bit-identical to the
reference by design, so it is checked against the exact rational oracle
at the north_star bound |c - c_exact| <= 4 l u (|A||B|)_ij, u = 2^-104."""

import numpy as np
import pytest

from oracle import exact
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu

DD = mp.PrecisionSpec.dd()
U_EXP_DD = 104          # u = 2^-104 (north_star)


@pytest.mark.parametrize("wide", [False, True])
@pytest.mark.parametrize("n_min", [16, 32, 64, 128, 256])
def test_fast_mode_meets_exact_bound_cfg1(gpu, wide, n_min):
    a, b = inputs.gemm_inputs("dd", 1024, 1024, 1024, seed=0, wide=wide)
    A = DenseMatrix(1024, 1024, DD, a).to_device()
    B = DenseMatrix(1024, 1024, DD, b).to_device()
    c = mp.matmul_block(A, B, n_min, mode="fast").host_array()
    rows, cols = exact.sample_indices(1024, 1024, 5, seed=n_min + wide)
    ratio, n = exact.bound_ratio(a, b, c, rows, cols, U_EXP_DD)
    assert ratio <= 1.0, ratio
    # it differs from the bit-exact product by at most a few ulps of lo
    ref = mp.matmul_block(A, B, n_min).host_array()
    assert np.max(np.abs(c[..., 0] - ref[..., 0])) <= np.max(np.abs(ref[..., 0])) * 2.0 ** -50


def test_fast_mode_cancellation(gpu):
    """Adversarial: rows of A orthogonal-ish to columns of B, so C entries
    cancel to far below |A||B| -- the componentwise bound still holds."""
    rng = np.random.default_rng(3)
    n = 256
    a, b = inputs.gemm_inputs("dd", n, n, n, seed=4)
    b[:, 1::2] = -b[:, 0::2]               # paired columns
    a[:, n // 2:] = a[:, :n // 2]          # repeated halves -> heavy cancellation
    b[n // 2:] = b[:n // 2]
    b[n // 2:, :, :] *= -1.0
    A = DenseMatrix(n, n, DD, np.ascontiguousarray(a)).to_device()
    B = DenseMatrix(n, n, DD, np.ascontiguousarray(b)).to_device()
    c = mp.matmul_block(A, B, 32, mode="fast").host_array()
    ratio, _ = exact.bound_ratio(a, b, c, list(range(0, n, 37)), list(range(0, n, 41)),
                                 U_EXP_DD)
    assert ratio <= 1.0, ratio
    del rng


def test_fast_mode_rejects_qd(gpu):
    x = DenseMatrix.zeros(4, 4, mp.PrecisionSpec.qd())
    with pytest.raises(ValueError):
        mp.matmul_block(x, x, 16, mode="fast")
    with pytest.raises(ValueError):
        mp.matmul_block(DenseMatrix.zeros(4, 4, DD), DenseMatrix.zeros(4, 4, DD), 16,
                        mode="turbo")
