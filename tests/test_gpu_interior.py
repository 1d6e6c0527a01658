"""The interior-tile path of the blocked kernels (csrc/gemm.cuh
gemm_tile_interior / gemm_tile_sum_interior) against the CPU oracle, bit for
bit.

A CTA takes the interior path when its whole tile lies inside C and l is a
multiple of the k-tile; every other tile of the same launch takes the
general, predicated path.  The shapes here mix both in one launch for every
tile configuration (n_min 16 / 32 / 64 / 128 / 256), with l a multiple of
the k-tile (interior path) and not (general path everywhere), in overwrite
and accumulate mode, on contiguous operands and on strided views (Strassen
quadrants), and in a batched launch.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, inputs

pytestmark = pytest.mark.gpu

NMINS = [16, 32, 64, 128, 256]


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _gemm(comps, n_min, A, B, C, m, l, n, lda, ldb, ldc, accumulate=False):
    s = torch.cuda.current_stream().cuda_stream
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, n_min, m, l, n, A.data_ptr(), lda, B.data_ptr(), ldb,
                   C.data_ptr(), ldc, accumulate, flag.data_ptr(), s)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0


# interior and edge tiles in one launch: 2-3 full tiles of every shape plus a
# ragged rim; l = 96 is a multiple of every k-tile (8, 16, 32), l = 50 of none
@pytest.mark.parametrize("n_min", NMINS)
@pytest.mark.parametrize("shape", [(160, 96, 200), (131, 50, 197), (128, 64, 192)])
def test_dd_interior_and_edge_tiles(gpu, n_min, shape):
    m, l, n = shape
    a, b = inputs.gemm_inputs("dd", m, l, n, seed=11, wide=(l == 96))
    want = oracle.matmul_simple(a, b)
    A, B = _dev(a), _dev(b)
    C = torch.full((m, n, 2), float("nan"), dtype=torch.float64, device="cuda")
    _gemm(2, n_min, A, B, C, m, l, n, l, n, n)
    assert np.array_equal(C.cpu().numpy(), want)


@pytest.mark.parametrize("n_min", [16, 32, 64, 128, 256])
def test_qd_interior_and_edge_tiles(gpu, n_min):
    m, l, n = 72, 48, 80
    a, b = inputs.gemm_inputs("qd", m, l, n, seed=12)
    want = oracle.matmul_simple(a, b)
    C = torch.full((m, n, 4), float("nan"), dtype=torch.float64, device="cuda")
    _gemm(4, n_min, _dev(a), _dev(b), C, m, l, n, l, n, n)
    assert np.array_equal(C.cpu().numpy(), want)


# accumulate mode: C += A2 B2 on top of C = A1 B1 equals the product over the
# concatenated k range (the reference's kb loop, _kernels.pyx:128-184)
@pytest.mark.parametrize("tok,n_min", [("dd", 32), ("dd", 128), ("dd", 64), ("qd", 16)])
def test_accumulate_equals_one_k_range(gpu, tok, n_min):
    comps = 2 if tok == "dd" else 4
    m, n = (96, 128) if tok == "dd" else (48, 64)
    l1, l2 = 64, 32
    a, b = inputs.gemm_inputs(tok, m, l1 + l2, n, seed=13)
    want = oracle.matmul_simple(a, b)
    A, B = _dev(a), _dev(b)
    C = torch.empty((m, n, comps), dtype=torch.float64, device="cuda")
    l = l1 + l2
    # k-panel views: A[:, :l1] has leading dimension l, B[:l1] is contiguous
    _gemm(comps, n_min, A, B, C, m, l1, n, l, n, n, accumulate=False)
    _gemm(comps, n_min, A[:, l1:], B[l1:], C, m, l2, n, l, n, n, accumulate=True)
    assert np.array_equal(C.cpu().numpy(), want)


# strided views of larger buffers (Strassen quadrants): every leading
# dimension differs from the view's width
@pytest.mark.parametrize("n_min", [32, 128])
def test_dd_strided_views(gpu, n_min):
    m, l, n = 64, 64, 128
    rng = np.random.default_rng(14)
    big_a = inputs.dd_random(rng, 2 * m, 2 * l)
    big_b = inputs.dd_random(rng, 2 * l, 2 * n)
    a = np.ascontiguousarray(big_a[m:, l:])
    b = np.ascontiguousarray(big_b[:l, n:])
    want = oracle.matmul_simple(a, b)
    A, B = _dev(big_a), _dev(big_b)
    big_c = torch.zeros((2 * m, 2 * n, 2), dtype=torch.float64, device="cuda")
    _gemm(2, n_min, A[m:, l:], B[:l, n:], big_c[m:, :n], m, l, n, 2 * l, 2 * n, 2 * n)
    got = big_c.cpu().numpy()
    assert np.array_equal(got[m:, :n], want)
    assert not got[:m].any() and not got[m:, n:].any()   # nothing written outside the view


# Strassen with the fused (operand sums in the tile loads) and the
# materialised leaves: 128^3 leaves are all-interior 32x32 tiles, 96^3-padded
# odd sizes take the general path
@pytest.mark.parametrize("n,cutoff", [(256, 128), (256, 64), (200, 50)])
def test_strassen_fused_leaves_interior(gpu, n, cutoff, monkeypatch):
    a, b = inputs.gemm_inputs("dd", n, n, n, seed=15)
    want = oracle.strassen(a, b, cutoff, 32)
    A = mp.DenseMatrix(n, n, mp.PrecisionSpec.dd(), a).to_device()
    B = mp.DenseMatrix(n, n, mp.PrecisionSpec.dd(), b).to_device()
    for fuse in ("1", "0"):
        monkeypatch.setenv("MPMM_STRASSEN_FUSE", fuse)
        got = mp.matmul_strassen(A, B, cutoff, 32).host_array()
        assert np.array_equal(got, want), f"fuse={fuse}"


# --- the speculative dense QD path (ddqd.cuh qd_mul_add_spec) -----------------
# Interior QD tiles run every gate of the multiply-add as "passed" and vote
# once per k-tile on whether one may have failed; a failed vote recomputes the
# tile with the gated sequence.  These operands make gates fail at chosen
# places of an all-interior product: from a later k-tile on, in one tile
# only, in every multiply-add (exact products: zero error terms), and through
# zero limbs; the result must be the oracle's bits every time.

def _qd_product(a, b, n_min):
    m, l, n = a.shape[0], a.shape[1], b.shape[1]
    C = torch.full((m, n, 4), float("nan"), dtype=torch.float64, device="cuda")
    _gemm(4, n_min, _dev(a), _dev(b), C, m, l, n, l, n, n)
    return C.cpu().numpy()


@pytest.mark.parametrize("n_min", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("case", ["late_zeros", "one_tile", "exact_products", "zero_limbs",
                                  "cancel", "bits28", "bits27", "bits26_53"])
def test_qd_speculation_falls_back(gpu, n_min, case):
    m, l, n = 64, 64, 64
    a, b = inputs.gemm_inputs("qd", m, l, n, seed=21)
    rng = np.random.default_rng(22)
    if case == "late_zeros":          # whole elements vanish from the third k-tile on
        a[:, 40:, :] *= (rng.random((m, l - 40, 1)) < 0.7)
    elif case == "one_tile":          # one element of B: only the tiles of column 5 fail
        b[50, 5, :] = 0.0
    elif case == "exact_products":    # powers of two: every TwoProd error is zero
        a = np.ldexp(np.where(rng.random(a.shape) < 0.5, 1.0, -1.0),
                     rng.integers(-8, 8, a.shape) - 55 * np.arange(4))
        b = np.ldexp(np.where(rng.random(b.shape) < 0.5, 1.0, -1.0),
                     rng.integers(-8, 8, b.shape) - 55 * np.arange(4))
    elif case == "zero_limbs":        # double-precision values stored as QD
        a[..., 1:] = 0.0
        b[..., 2:] = 0.0
    elif case in ("bits28", "bits27", "bits26_53"):
        # limbs with exactly 28 significant bits pass the staging test (their
        # products have 55-56 bits: inexact, the speculation must be exact);
        # 27 bits fail it; 26-bit limbs of A against full 53-bit limbs of B
        # fail it although every product is inexact (the test is sufficient,
        # not necessary)
        def limbs(shape, bits):
            mant = rng.integers(1 << (bits - 1), 1 << bits, shape) | 1   # odd, `bits` long
            sign = np.where(rng.random(shape) < 0.5, 1.0, -1.0)
            return np.ldexp(sign * mant.astype(np.float64),
                            rng.integers(-3, 3, shape) - bits - 53 * np.arange(4))
        if case == "bits26_53":
            a = limbs(a.shape, 26)
        else:
            nb = 28 if case == "bits28" else 27
            a, b = limbs(a.shape, nb), limbs(b.shape, nb)
    elif case == "cancel":            # second half of k cancels the first: the sum passes 0
        a[:, 32:, :] = a[:, :32, :]
        b[32:, :, :] = -b[:32, :, :]
    want = oracle.matmul_simple(np.ascontiguousarray(a), np.ascontiguousarray(b))
    got = _qd_product(np.ascontiguousarray(a), np.ascontiguousarray(b), n_min)
    assert np.array_equal(got, want)


def test_qd_speculation_accumulate_from_zero_and_nonzero(gpu):
    # C += A B with C zero (the first step's gate fails -> gated first step)
    # and with C random (speculative from the second step on)
    m, l, n = 32, 32, 48
    a, b = inputs.gemm_inputs("qd", m, 2 * l, n, seed=23)
    want = oracle.matmul_simple(a, b)
    A, B = _dev(a), _dev(b)
    C = torch.zeros((m, n, 4), dtype=torch.float64, device="cuda")
    _gemm(4, 64, A, B, C, m, l, n, 2 * l, n, n, accumulate=True)
    _gemm(4, 64, A[:, l:], B[l:], C, m, l, n, 2 * l, n, n, accumulate=True)
    assert np.array_equal(C.cpu().numpy(), want)


def test_qd_speculation_falls_back_under_streamed_operands(gpu):
    # host operands, k-panel streaming (64-column panels): interior QD tiles
    # whose gates first fail in the LAST k-panel -- the abandoned tile's exact
    # recomputation must wait for the panels like the first attempt did
    from paper_1710_01839_b200.matrix import DenseMatrix
    m, l, n = 64, 512, 64
    a, b = inputs.gemm_inputs("qd", m, l, n, seed=24)
    a[:, 480:, 1:] = 0.0                       # zero limbs from k = 480 on
    want = oracle.matmul_simple(a, b)
    qd = mp.PrecisionSpec.qd()
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
    for n_min in (16, 64):
        A, B = DenseMatrix(m, l, qd, pin(a)), DenseMatrix(l, n, qd, pin(b))
        for _ in range(2):
            assert np.array_equal(mp.matmul_block(A, B, n_min).host_array(), want)


def test_randomised_blocked_parity(gpu):
    # tools/fuzz_gemm.py: random shapes around the tile boundaries, every
    # block size, DD/QD, accumulate, strided views, zero-sprinkled QD operands
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_gemm.py"), "120", "5"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 mismatches" in r.stdout


def test_strassen_driver_regimes(gpu):
    # tools/exp/strassen_fuzz_deep.py: deep recursions with padded levels,
    # fused and materialised last levels, chunked launches (> 1024 parents,
    # > 16384 elementwise problems per level), and the depth-first mode
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("MPMM_STRASSEN_FUSE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "exp",
                                                     "strassen_fuzz_deep.py"), "5"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 mismatches" in r.stdout
