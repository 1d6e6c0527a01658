"""Native runtime pieces through the C ABI: the Strassen driver
(mpmm_strassen_dev), the single-process multi-GPU runtime (mpmm_init /
mpmm_gemm_multi / mpmm_finalize) and the event timers.

Parity: the reference's Strassen (multiply.py:267-338, oracle.strassen)
bitwise; the multi-GPU runtime bitwise against the single-GPU product
(row sharding + panel broadcast never change an element's k order).
"""
import subprocess
import sys
import os

import numpy as np
import pytest

import oracle
from paper_1710_01839_b200 import _cuda, inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dev(x):
    import torch
    return torch.from_numpy(x).cuda()


def _strassen_native(a, b, cutoff, leaf, stats=False):
    import ctypes
    import torch
    A, B = _dev(a), _dev(b)
    m, l, n = a.shape[0], a.shape[1], b.shape[1]
    C = torch.empty((m, n, a.shape[2]), dtype=torch.float64, device="cuda")
    counts = (ctypes.c_int64 * 2)()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _cuda.strassen_dev(a.shape[2], cutoff, leaf, m, l, n, A.data_ptr(), l, B.data_ptr(), n,
                       C.data_ptr(), n, flag.data_ptr(), counts if stats else None,
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return C.cpu().numpy(), (counts[0], counts[1]), int(flag.item())


@pytest.mark.parametrize("tok,n,cut,leaf", [("dd", 37, 8, 4), ("dd", 64, 16, 8), ("qd", 21, 5, 2),
                                             ("dd", 128, 2, 2)])
def test_native_strassen_matches_oracle(gpu, tok, n, cut, leaf):
    # n=128, cutoff 2: 117649 leaves and 84035 operand sums on one level,
    # more than one launch's batch limit (chunked)
    a, b = inputs.gemm_inputs(tok, n, n, n, seed=3)
    got, counts, flag = _strassen_native(a, b, cut, leaf, stats=True)
    assert flag == 0
    assert np.array_equal(got, oracle.strassen(a, b, cut, leaf))
    nodes, s = 0, n
    level = 1
    while s > cut:
        nodes += level
        level *= 7
        s = (s + (s & 1)) // 2
    assert counts == (7 * nodes, 18 * nodes)


def test_native_strassen_depth_first_budget(gpu):
    """Forcing the depth-first top levels (tiny scratch budget) gives the
    same bits as the level-synchronous run."""
    code = (
        "import numpy as np, torch, sys; sys.path[:0] = ['.', 'tests'];"
        "from paper_1710_01839_b200 import inputs;"
        "from test_gpu_native import _strassen_native as s;"
        "a, b = inputs.gemm_inputs('dd', 96, 96, 96, seed=5);"
        "np.save('/tmp/_mpmm_df.npy', s(a, b, 6, 4)[0])")
    env = dict(os.environ, MPMM_STRASSEN_BUDGET_MB="1")
    subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, check=True)
    a, b = inputs.gemm_inputs("dd", 96, 96, 96, seed=5)
    ref, _, _ = _strassen_native(a, b, 6, 4)
    assert np.array_equal(np.load("/tmp/_mpmm_df.npy"), ref)
    assert np.array_equal(ref, oracle.strassen(a, b, 6, 4))


def test_native_strassen_rectangular_and_nonfinite(gpu):
    a, b = inputs.gemm_inputs("dd", 40, 24, 56, seed=1)
    got, _, flag = _strassen_native(a, b, 8, 4)
    exact = oracle.matmul_block(a, b, 8)
    assert flag == 0
    # same algorithm family, different rounding order: compare to the bound
    err = np.abs((got[..., 0] - exact[..., 0]) + (got[..., 1] - exact[..., 1]))
    assert err.max() <= 1e-25
    a[3, 5, 0] = np.inf
    _, _, flag = _strassen_native(a, b, 8, 4)
    assert flag == 1


@pytest.fixture
def runtime(gpu):
    _cuda.runtime_init(1)
    yield
    _cuda.runtime_finalize()


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_runtime_gemm_multi_bitwise(runtime, tok):
    comps = 2 if tok == "dd" else 4
    a, b = inputs.gemm_inputs(tok, 300, 260, 140, seed=2)
    ref = oracle.matmul_block(a, b, 32)
    assert _cuda.runtime_gpus() == [0]
    for algo, nmin in ((_cuda.ALGO_SIMPLE, 0), (_cuda.ALGO_BLOCK, 32), (_cuda.ALGO_BLOCK, 64)):
        for panels in (0, 1, 3, 7):
            c = np.empty((300, 140, comps))
            bad, ms = _cuda.gemm_multi(comps, algo, nmin, 0, a, b, c, panels)
            assert not bad and ms > 0
            assert np.array_equal(c, ref), (algo, nmin, panels)


def test_runtime_strassen_and_errors(runtime):
    a, b = inputs.gemm_inputs("dd", 64, 64, 64, seed=4)
    c = np.empty((64, 64, 2))
    _cuda.gemm_multi(2, _cuda.ALGO_STRASSEN, 8, 16, a, b, c)
    assert np.array_equal(c, oracle.strassen(a, b, 16, 8))
    with pytest.raises(ValueError):
        _cuda.runtime_init(1)              # already initialized
    a[0, 0, 0] = np.nan
    bad, _ = _cuda.gemm_multi(2, _cuda.ALGO_BLOCK, 16, 0, a, b, c)
    assert bad


def test_runtime_requires_init(gpu):
    a, b = inputs.gemm_inputs("dd", 8, 8, 8, seed=0)
    with pytest.raises(ValueError, match="not initialized"):
        _cuda.gemm_multi(2, _cuda.ALGO_BLOCK, 4, 0, a, b, np.empty((8, 8, 2)))
    with pytest.raises(ValueError):
        _cuda.runtime_init(99)


def test_event_timer(gpu):
    import torch
    t = _cuda.Timer()
    s = torch.cuda.current_stream().cuda_stream
    x = torch.zeros(1 << 22, dtype=torch.float64, device="cuda")
    t.start(s)
    _cuda.fp64_burn_dev(0, 148, 256, 2000, x.data_ptr(), s)
    t.stop(s)
    assert t.elapsed_ms() > 0
