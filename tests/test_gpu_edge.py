"""GPU parity at the reference's EFT-domain edges (eft.py:19-24,
_kernels.pyx:19-29): operands whose split TwoProd overflows (NaN in the
reference, RangeError from matmul_*), products near the subnormal floor,
subnormal operands, signed zeros in every limb, inf and NaN.

Every path a product can take is checked against the reference's own
outputs (tests/golden/edge_*.npz, made by tests/golden/make_golden.py from
the reference), or against the oracle (pinned to those goldens by
tests/test_oracle_golden.py) at sizes that reach the streamed host path:
device-resident simple / blocked / Strassen / batched launches, the
protocol's range kernels on host pointers, and host-buffer products.
"""

import numpy as np
import pytest

import oracle
from conftest import golden
from test_oracle_golden import EDGE, same_bits
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, backend, domain, inputs
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu


def M(arr, prec):
    return DenseMatrix(arr.shape[0], arr.shape[1], prec, np.ascontiguousarray(arr))


def prec_of(a):
    return mp.PrecisionSpec.dd() if a.shape[2] == 2 else mp.PrecisionSpec.qd()


def raw_device(a, b, algo, n_min):
    """C through mpmm_gemm_dev without the finite check (the kernels never
    raise; the reference's kernels return NaN the same way)."""
    import torch
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    m, l, n, comps = a.shape[0], a.shape[1], b.shape[1], a.shape[2]
    C = torch.full((m, n, comps), 7.0, dtype=torch.float64, device="cuda")
    _cuda.gemm_dev(comps, algo, n_min, m, l, n, A.data_ptr(), l, B.data_ptr(), n, C.data_ptr(),
                   n, False, None, torch.cuda.current_stream().cuda_stream)
    return C.cpu().numpy()


@pytest.mark.parametrize("name", EDGE)
def test_edge_device_kernels(gpu, name):
    g = golden(name)
    a, b, want = g["a"], g["b"], g["c"]
    assert same_bits(raw_device(a, b, _cuda.ALGO_SIMPLE, 0), want)
    for n_min in (16, 32, 64, 128, 256):
        assert same_bits(raw_device(a, b, _cuda.ALGO_BLOCK, n_min), want), n_min


@pytest.mark.parametrize("name", EDGE)
def test_edge_public_api_raises_like_the_reference(gpu, name):
    g = golden(name)
    p = prec_of(g["a"])
    A, B = M(g["a"], p), M(g["b"], p)
    for run in (lambda: mp.matmul_simple(A.to_device(), B.to_device()),
                lambda: mp.matmul_block(A.to_device(), B.to_device(), 32),
                lambda: mp.matmul_block(A, B, 64),
                lambda: mp.matmul_simple(A, B)):
        if int(g["raises"]):
            with pytest.raises(mp.RangeError):
                run()
        else:
            c = run()
            assert same_bits(c.host_array(), g["c"])


@pytest.mark.parametrize("name", EDGE)
def test_edge_protocol_range_kernels(gpu, name):
    g = golden(name)
    a, b, want = g["a"], g["b"], g["c"]
    kern = backend.kernels()
    tok = "dd" if a.shape[2] == 2 else "qd"
    m, n = a.shape[0], b.shape[1]
    c = np.zeros_like(want)
    getattr(kern, f"{tok}_simple_rows")(a, b, c, 0, m)
    assert same_bits(c, want)
    n_min = int(g["n_min"])
    cells = (-(-m // n_min)) * (-(-n // n_min))
    c = np.zeros_like(want)
    getattr(kern, f"{tok}_block_cells")(a, b, c, n_min, 0, cells // 2)
    getattr(kern, f"{tok}_block_cells")(a, b, c, n_min, cells // 2, cells)
    assert same_bits(c, want)


def test_edge_strassen(gpu):
    g = golden("edge_dd_strassen_big")
    p = mp.PrecisionSpec.dd()
    import torch
    A, B = torch.from_numpy(g["a"]).cuda(), torch.from_numpy(g["b"]).cuda()
    C = torch.empty_like(A)
    _cuda.strassen_dev(2, 4, 2, 16, 16, 16, A.data_ptr(), 16, B.data_ptr(), 16, C.data_ptr(),
                       16, None, None, torch.cuda.current_stream().cuda_stream)
    assert same_bits(C.cpu().numpy(), g["c"])
    # and it is outside the domain at the Strassen margins (Dekker leaves)
    assert domain.unsafe(g["a"], g["b"], 52, 3)


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_edge_streamed_and_panelled_host_products(gpu, tok):
    """l >= 128 takes the streamed host path (one launch consuming k-panels;
    the domain is checked after the copies and C recomputed with the Dekker
    kernel when needed), pageable operands the panelled path (a scan per
    k-panel)."""
    m, l, n = 96, 320, 80
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=44)
    a0, b0 = a.copy(), b.copy()
    a[5, 200] = 0.0
    a[5, 200, 0] = 0.75 * 2.0 ** 1000           # split overflow: NaN in row 5
    b[17, 3] = np.ldexp(b[17, 3], -1010)       # error underflow in column 3
    want = oracle.matmul_simple(a, b)
    assert domain.unsafe(a, b) and np.isnan(want[5]).all()
    import torch
    pa = torch.from_numpy(a).pin_memory().numpy()
    pb = torch.from_numpy(b).pin_memory().numpy()
    out = torch.empty((m, n, a.shape[2]), dtype=torch.float64, pin_memory=True).numpy()
    assert not _cuda.gemm_host(a.shape[2], _cuda.ALGO_BLOCK, 32, pa, pb, out, accumulate=False)
    assert same_bits(out, want)
    out2 = np.zeros_like(want)
    _cuda.gemm_host(a.shape[2], _cuda.ALGO_BLOCK, 32, a, b, out2, accumulate=False)
    assert same_bits(out2, want)
    # without the injected values the same path stays on the DFMA kernel
    a, b = a0, b0
    assert not domain.unsafe(a, b)
    pa[...] = a
    pb[...] = b
    assert _cuda.gemm_host(a.shape[2], _cuda.ALGO_BLOCK, 32, pa, pb, out, accumulate=False)
    assert np.array_equal(out, oracle.matmul_simple(a, b))


def test_edge_batched_launch(gpu):
    """mpmm_gemm_batched_dev scans every problem of the table."""
    import torch
    g = golden("edge_dd_big1000")
    h = golden("edge_dd_zeros")
    m, l, n = g["a"].shape[0], g["a"].shape[1], g["b"].shape[1]
    A = torch.from_numpy(np.stack([h["a"], g["a"]])).cuda()
    B = torch.from_numpy(np.stack([h["b"], g["b"]])).cuda()
    C = torch.zeros((2, m, n, 2), dtype=torch.float64, device="cuda")
    probs = torch.tensor([[A[i].data_ptr(), B[i].data_ptr(), C[i].data_ptr(), l, n, n]
                          for i in range(2)], dtype=torch.int64, device="cuda")
    _cuda.gemm_batched_dev(2, _cuda.ALGO_BLOCK, 32, 2, m, l, n, probs.data_ptr(), False, None,
                           torch.cuda.current_stream().cuda_stream)
    c = C.cpu().numpy()
    assert same_bits(c[0], h["c"]) and same_bits(c[1], g["c"])
