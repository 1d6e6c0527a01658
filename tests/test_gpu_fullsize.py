"""BASELINE configurations at full size on the GPU (configs[2], [3], [4]).

At these sizes a full reference run takes minutes to hours, so parity is
checked the way SURVEY.md s8c prescribes: sampled rows bitwise against the
compiled-C oracle (pinned to the reference by tests/test_oracle_golden.py),
sampled entries against the exact componentwise bound 4 l u (|A||B|)_ij
with the device superaccumulator (csrc/verify.cu), Strassen bitwise against
the oracle's restatement of the reference recursion where the oracle runs
in seconds, and normwise (the reference's 100 n u) where it does not.
"""

import os

import numpy as np
import pytest

import oracle
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
from paper_1710_01839_b200.verify import exact_bound_ratio

pytestmark = pytest.mark.gpu

DD = mp.PrecisionSpec.dd()
QD = mp.PrecisionSpec.qd()
CORES = max(1, len(os.sched_getaffinity(0)))


def dev_pair(tok, m, l, n, seed):
    p = DD if tok == "dd" else QD
    a, b = inputs.gemm_inputs_device(tok, m, l, n, seed=seed)
    return DenseMatrix(m, l, p, a), DenseMatrix(l, n, p, b)


def oracle_rows(a_host, b_host, rows):
    """Rows of the reference product (the oracle's blocked cells over all
    host threads; blocked == simple bitwise)."""
    out = []
    for i in rows:
        out.append(oracle.matmul_block(np.ascontiguousarray(a_host[i:i + 1]), b_host, 64,
                                       threads=CORES)[0])
    return np.stack(out)


def test_cfg2_qd_1024_bitwise_32_rows(gpu):
    A, B = dev_pair("qd", 1024, 1024, 1024, seed=0)
    c = mp.matmul_block(A, B, 64).host_array()
    a, b = A.host_array(), B.host_array()
    rows = list(range(0, 1024, 32))
    assert len(rows) == 32
    assert np.array_equal(c[rows], oracle_rows(a, b, rows))
    worst, _, _ = exact_bound_ratio(A, B, mp.DenseMatrix(1024, 1024, QD, c), samples=4096)
    assert worst <= 1.0


@pytest.mark.parametrize("cut", [128, 256, 512])
def test_cfg3_rectangular_strassen(gpu, cut):
    """BASELINE configs[3] rectangular case, 2048 x 1024 x 4096, uniform
    inputs: normwise against blocked within 100 n u and sampled entries
    within the componentwise bound."""
    A, B = dev_pair("dd", 2048, 1024, 4096, seed=0)
    blk = mp.matmul_block(A, B, 64)
    st = mp.matmul_strassen(A, B, cut, 64, rectangular=True)
    d = mp.frobenius_rel_diff(st.to_host(), blk.to_host())
    assert 0.0 < d <= 100.0 * 4096 * DD.unit_roundoff(), d
    worst, _, _ = exact_bound_ratio(A, B, st, samples=2048)
    assert worst <= 1.0, worst


@pytest.mark.parametrize("tok,n,cut,leaf", [("dd", 512, 128, 64), ("dd", 1024, 256, 32),
                                            ("qd", 256, 64, 16)])
def test_strassen_bitwise_against_reference_recursion(gpu, tok, n, cut, leaf):
    A, B = dev_pair(tok, n, n, n, seed=5)
    c = mp.matmul_strassen(A, B, cut, leaf).host_array()
    assert np.array_equal(c, oracle.strassen(A.host_array(), B.host_array(), cut, leaf))


def test_cfg4_dd_8192(gpu):
    """configs[4] at its largest size: blocked (the bench's kernel) bitwise
    on sampled rows, within the componentwise bound on sampled entries;
    the tuner's Strassen pick within the normwise budget of blocked."""
    n = 8192
    A, B = dev_pair("dd", n, n, n, seed=1)
    C = mp.matmul_block(A, B, 32)
    rows = [0, 4095, 8191]
    a_rows = A.data[rows].cpu().numpy()
    want = np.stack([oracle.matmul_block(np.ascontiguousarray(a_rows[q:q + 1]),
                                         B.host_array(), 64, threads=CORES)[0]
                     for q in range(3)])
    assert np.array_equal(C.data[rows].cpu().numpy(), want)
    worst, _, _ = exact_bound_ratio(A, B, C, samples=4096)
    assert worst <= 1.0, worst
    S = mp.matmul_strassen(A, B, 1024, 32)
    d = mp.frobenius_rel_diff(S.to_host(), C.to_host())
    assert 0.0 < d <= 100.0 * n * DD.unit_roundoff(), d


@pytest.mark.parametrize("n", [4096, 8192])
def test_cfg4_qd(gpu, n):
    """configs[4] QD at 4096 and 8192 (seed 1): sampled entries within
    4 l u (|A||B|), u = 2^-209, and one row bitwise against the oracle."""
    A, B = dev_pair("qd", n, n, n, seed=1)
    C = mp.matmul_block(A, B, 64)
    worst, _, _ = exact_bound_ratio(A, B, C, samples=1024)
    assert worst <= 1.0, worst
    i = n // 3
    a_row = np.ascontiguousarray(A.data[i:i + 1].cpu().numpy())
    want = oracle.matmul_block(a_row, B.host_array(), 64, threads=CORES)
    assert np.array_equal(C.data[i:i + 1].cpu().numpy(), want)
