"""The reference's acceptance criteria 3, 4 and 8 (pkg/tests/test_acceptance.py
:91-126, :185-197) on the GPU path, plus the Strassen properties of
test_multiply.py:93-111 at BASELINE config-3 size.

* criterion 3: integer inputs -- simple, blocked (every n_min) and Strassen
  agree exactly; single-block blocked == simple on the paper's test pair;
* criterion 4: rounded inputs -- Strassen within 100 n u and blocked within
  4 n u of simple, normwise (the reference's frobenius_rel_diff);
* criterion 8: the threads argument never changes a bit (here also the
  host-buffer k-panel split and the device-resident path);
* Strassen == blocked when the cutoff covers n; cfg3 (2048) Strassen at
  every BASELINE cutoff within 100 n u of the blocked product.
"""
import random

import numpy as np
import pytest

from conftest import random_int_matrix
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu

DD = mp.PrecisionSpec.dd()
U_DD = 2.0 ** -104


def test_criterion_3_kernel_equivalence_exact(gpu):
    rng = random.Random(3)
    for n in (2, 3, 8, 16, 17):
        a = random_int_matrix(rng, n, n, DD, bound=8)
        b = random_int_matrix(rng, n, n, DD, bound=8)
        ref = mp.matmul_simple(a, b)
        for n_min in (2, 4, n):
            assert mp.matmul_block(a, b, n_min) == ref, (n, n_min)
        assert mp.matmul_strassen(a, b, cutoff=2, leaf_n_min=2) == ref, n
    for n in (8, 64):
        a, b = mp.generate_test_pair(n, DD)
        assert mp.matmul_block(a, b, n) == mp.matmul_simple(a, b), n


def test_criterion_4_kernel_equivalence_rounded(gpu):
    for n in (63, 64, 100, 257):
        a, b = mp.generate_test_pair(n, DD)
        ref = mp.matmul_simple(a, b, threads=2)
        d_str = mp.frobenius_rel_diff(mp.matmul_strassen(a, b, 64, 64, threads=2), ref)
        d_blk = mp.frobenius_rel_diff(mp.matmul_block(a, b, 64, threads=2), ref)
        assert d_str <= 100.0 * U_DD * n, (n, d_str)
        assert d_blk <= 4.0 * n * U_DD, (n, d_blk)


def test_criterion_8_threads_invariance(gpu):
    a, b = mp.generate_test_pair(128, DD)
    base = (mp.matmul_simple(a, b, 1), mp.matmul_block(a, b, 32, 1),
            mp.matmul_strassen(a, b, 64, 32, 1))
    for threads in (2, 4):
        assert mp.matmul_simple(a, b, threads) == base[0]
        assert mp.matmul_block(a, b, 32, threads) == base[1]
        assert mp.matmul_strassen(a, b, 64, 32, threads) == base[2]
    # the same product device-resident, and through every block size
    da, db = a.to_device(), b.to_device()
    assert mp.matmul_block(da, db, 32).to_host() == base[1]
    for n_min in (16, 64, 128, 256):
        assert mp.matmul_block(a, b, n_min) == base[1]


@pytest.mark.parametrize("n,cut", [(64, 64), (100, 128), (257, 257)])
def test_strassen_equals_block_when_cutoff_covers_n(gpu, n, cut):
    a, b = mp.generate_test_pair(n, DD)
    assert mp.matmul_strassen(a, b, cutoff=cut, leaf_n_min=32) == mp.matmul_block(a, b, 32)


@pytest.mark.parametrize("cut", [128, 256, 512])
def test_cfg3_strassen_normwise(gpu, cut):
    """BASELINE config 3: DD 2048^3 Strassen at every cutoff, against the
    blocked product, within the reference's 100 n u normwise budget."""
    n = 2048
    A, B = inputs.gemm_inputs_device("dd", n, n, n, seed=0)
    a, b = DenseMatrix(n, n, DD, A), DenseMatrix(n, n, DD, B)
    blk = mp.matmul_block(a, b, 64).to_host()
    st = mp.matmul_strassen(a, b, cutoff=cut, leaf_n_min=64).to_host()
    d = mp.frobenius_rel_diff(st, blk)
    assert 0.0 < d <= 100.0 * U_DD * n, d
    assert np.isfinite(st.data).all()
