"""The device exact verifier against the Python big-integer oracle, then
full-size exact checks of the BASELINE configs through it."""

import numpy as np
import pytest

from oracle import exact
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
from paper_1710_01839_b200.verify import exact_bound_ratio

pytestmark = pytest.mark.gpu


def M(x, prec):
    return DenseMatrix(x.shape[0], x.shape[1], prec, np.ascontiguousarray(x))


@pytest.mark.parametrize("tok,wide", [("dd", False), ("dd", True), ("qd", False)])
def test_device_verifier_matches_big_integer_oracle(gpu, tok, wide):
    prec = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs(tok, 24, 40, 20, seed=3, wide=wide)
    c = mp.matmul_block(M(a, prec), M(b, prec), 16).data
    rows, cols = list(range(0, 24, 5)), list(range(0, 20, 3))
    want, _ = exact.bound_ratio(a, b, c, rows, cols, 104 if tok == "dd" else 209)
    ii = np.repeat(rows, len(cols))
    jj = np.tile(cols, len(rows))
    got, r, _ = exact_bound_ratio(M(a, prec), M(b, prec), M(c, prec), (ii, jj))
    assert got == pytest.approx(want, rel=1e-9, abs=1e-300)
    # a one-ulp change of a large component is far outside the bound
    bad = c.copy()
    bad[5, 3, 0] = np.nextafter(bad[5, 3, 0], np.inf)
    worst, _, _ = exact_bound_ratio(M(a, prec), M(b, prec), M(bad, prec), ([5], [3]))
    assert worst > 1.0


def test_exact_products_have_zero_error(gpu):
    rng = np.random.default_rng(0)
    a = np.zeros((8, 8, 2))
    b = np.zeros((8, 8, 2))
    a[..., 0] = rng.integers(-8, 9, (8, 8))
    b[..., 0] = rng.integers(-8, 9, (8, 8))
    dd = mp.PrecisionSpec.dd()
    c = mp.matmul_simple(M(a, dd), M(b, dd))
    worst, r, _ = exact_bound_ratio(M(a, dd), M(b, dd), c)
    assert worst == 0.0 and len(r) == 64


@pytest.mark.parametrize("wide", [False, True])
def test_cfg1_full_product_every_entry_within_bound(gpu, wide):
    """Every one of the 1,048,576 entries of BASELINE config 1 (DD 1024^3,
    both input sets) meets 4 l u (|A||B|)_ij exactly -- for the bit-exact
    kernel and for the opt-in fast mode."""
    dd = mp.PrecisionSpec.dd()
    a, b = inputs.gemm_inputs("dd", 1024, 1024, 1024, seed=0, wide=wide)
    A, B = M(a, dd).to_device(), M(b, dd).to_device()
    for mode in ("exact", "fast"):
        c = mp.matmul_block(A, B, 32, mode=mode)
        worst, r, _ = exact_bound_ratio(A, B, c)
        assert len(r) == 1024 * 1024
        print(f"cfg1 wide={wide} mode={mode}: max ratio {worst:.3e}, median {np.median(r):.3e}")
        assert worst <= 1.0


def test_cfg2_qd_and_cfg4_dd8192_sampled(gpu):
    qd = mp.PrecisionSpec.qd()
    a, b = inputs.gemm_inputs("qd", 1024, 1024, 1024, seed=0)
    A, B = M(a, qd).to_device(), M(b, qd).to_device()
    c = mp.matmul_block(A, B, 16)
    worst, r, _ = exact_bound_ratio(A, B, c, samples=16384)
    print(f"cfg2 QD 1024: max ratio {worst:.3e} over {len(r)} entries")
    assert worst <= 1.0
    dd = mp.PrecisionSpec.dd()
    a, b = inputs.gemm_inputs("dd", 8192, 8192, 8192, seed=1)
    A, B = M(a, dd).to_device(), M(b, dd).to_device()
    for algo in ("block", "strassen"):
        c = (mp.matmul_block(A, B, 64) if algo == "block"
             else mp.matmul_strassen(A, B, 2048, 64))
        worst, r, _ = exact_bound_ratio(A, B, c, samples=8192)
        print(f"cfg4 DD 8192 {algo}: max ratio {worst:.3e} over {len(r)} entries")
        assert worst <= 1.0
