"""The streamed host-buffer product (capi.cu host_rows_gemm_streamed): with
page-locked A, B and C, mpmm_gemm_host runs ONE gemm_tiled launch whose
CTAs consume 64-column k-panels as their H2D copies land (flags set by
cuStreamWriteValue32) and write C straight into the page-locked result.

Parity: per element the k order is unchanged, so the result is the
reference's bits -- checked against the oracle (reference
_kernels.pyx:103-186 restated) and against the device-resident product, at
ragged shapes (l not a multiple of the panel), for DD and QD, and with the
streamed path switched off in a child process (MPMM_HOST_STREAMED=0).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, inputs
from paper_1710_01839_b200.errors import RangeError
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pinned(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()


@pytest.mark.parametrize("tok,m,l,n,nmin", [("dd", 96, 200, 72, 32), ("dd", 130, 1000, 70, 16),
                                            ("dd", 256, 128, 256, 128), ("qd", 40, 300, 24, 16),
                                            ("qd", 33, 129, 17, 32)])
def test_streamed_host_product_bit_identical(gpu, tok, m, l, n, nmin):
    prec = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=11)
    want = oracle.matmul_simple(a, b)
    A, B = DenseMatrix(m, l, prec, _pinned(a)), DenseMatrix(l, n, prec, _pinned(b))
    c = mp.matmul_block(A, B, nmin).host_array()
    assert np.array_equal(c, want)
    dev = mp.matmul_block(A.to_device(), B.to_device(), nmin).host_array()
    assert np.array_equal(c, dev)
    # the C ABI entry directly, into a page-locked C
    out = _pinned(np.zeros((m, n, prec.comps)))
    assert _cuda.gemm_host(prec.comps, _cuda.ALGO_BLOCK, nmin, A.data, B.data, out)
    assert np.array_equal(out, want)


def test_streamed_host_product_nonfinite_and_repeat(gpu):
    a, b = inputs.gemm_inputs("dd", 64, 256, 48, seed=12)
    a[5, 100, 0] = 1e300
    b[100, 7, 0] = 1e300
    A = DenseMatrix(64, 256, mp.PrecisionSpec.dd(), _pinned(a))
    B = DenseMatrix(256, 48, mp.PrecisionSpec.dd(), _pinned(b))
    with pytest.raises(RangeError):
        mp.matmul_block(A, B, 32)
    # the next products on the same streams are unaffected
    a2, b2 = inputs.gemm_inputs("dd", 64, 256, 48, seed=13)
    want = oracle.matmul_simple(a2, b2)
    A2 = DenseMatrix(64, 256, mp.PrecisionSpec.dd(), _pinned(a2))
    B2 = DenseMatrix(256, 48, mp.PrecisionSpec.dd(), _pinned(b2))
    for _ in range(3):
        assert np.array_equal(mp.matmul_block(A2, B2, 32).host_array(), want)


_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
a, b = inputs.gemm_inputs("dd", 300, 512, 260, seed=14)
pa, pb = torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(b).pin_memory().numpy()
c = mp.matmul_block(DenseMatrix(300, 512, mp.PrecisionSpec.dd(), pa),
                    DenseMatrix(512, 260, mp.PrecisionSpec.dd(), pb), 32).host_array()
np.save(sys.argv[2], c)
"""


def test_streamed_equals_panelled_path(gpu, tmp_path):
    outs = []
    for k, env in enumerate(({}, {"MPMM_HOST_STREAMED": "0"})):
        path = str(tmp_path / f"c{k}.npy")
        r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, path], cwd=ROOT,
                           env=dict(os.environ, **env), capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


def test_streamed_host_products_from_concurrent_threads(gpu):
    """Four host threads issue streamed products at once (each thread owns
    its streams; the panel flags and buffers are per call): every result
    is the oracle's."""
    from concurrent.futures import ThreadPoolExecutor
    cases = []
    for s in range(4):
        a, b = inputs.gemm_inputs("dd", 96, 256, 80, seed=30 + s)
        cases.append((DenseMatrix(96, 256, mp.PrecisionSpec.dd(), _pinned(a)),
                      DenseMatrix(256, 80, mp.PrecisionSpec.dd(), _pinned(b)),
                      oracle.matmul_simple(a, b)))

    def work(k):
        A, B, want = cases[k % 4]
        return all(np.array_equal(mp.matmul_block(A, B, 32).host_array(), want)
                   for _ in range(5))

    with ThreadPoolExecutor(4) as ex:
        assert all(ex.map(work, range(8)))


@pytest.mark.parametrize("tok,m,l,n,nmin", [("dd", 700, 300, 650, 32), ("dd", 1030, 257, 333, 16),
                                            ("qd", 200, 150, 300, 64), ("dd", 64, 200, 900, 128)])
def test_tile_streamed_host_product(gpu, monkeypatch, tok, m, l, n, nmin):
    """Large host products stream A by row panels and B by column panels in
    the grouped tile raster's order (one wait per tile); forced here at small
    sizes (MPMM_STREAM_TILE_MB=0) with ragged panel counts: the reference's
    bits, also with operands outside the DFMA domain (NaN row, Dekker path)."""
    monkeypatch.setenv("MPMM_STREAM_TILE_MB", "0")
    prec = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=13)
    want = oracle.matmul_simple(a, b)
    out = _pinned(np.zeros((m, n, prec.comps)))
    assert _cuda.gemm_host(prec.comps, _cuda.ALGO_BLOCK, nmin, _pinned(a), _pinned(b), out)
    assert np.array_equal(out, want)
    a[m // 2, l // 3] = 0.0
    a[m // 2, l // 3, 0] = 0.75 * 2.0 ** 1000        # the reference's split overflows
    want = oracle.matmul_simple(a, b)
    out = _pinned(np.zeros((m, n, prec.comps)))
    assert not _cuda.gemm_host(prec.comps, _cuda.ALGO_BLOCK, nmin, _pinned(a), _pinned(b), out)
    from test_oracle_golden import same_bits
    assert same_bits(out, want) and np.isnan(out[m // 2]).all()
