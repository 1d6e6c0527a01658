"""GPU parity: the sm_100a kernels against the reference (golden vectors
from the reference itself) and the CPU oracle, bit for bit.

Every product goes through the drop-in API or the C-ABI (the reference's
kernel-module protocol on host pointers, and the device entry points).
"""

import random

import numpy as np
import pytest

import oracle
from oracle import exact
from conftest import golden, random_int_matrix
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, backend, inputs
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu

DD = mp.PrecisionSpec.dd()
QD = mp.PrecisionSpec.qd()


def M(arr, prec):
    return DenseMatrix(arr.shape[0], arr.shape[1], prec, np.ascontiguousarray(arr))


# --- golden vectors produced by the reference --------------------------------

def test_cfg0_simple_bitwise(gpu):
    g = golden("cfg0_dd_simple_128")
    c = mp.matmul_simple(M(g["a"], DD), M(g["b"], DD))
    assert np.array_equal(c.data, g["c_simple"])


@pytest.mark.parametrize("n_min", [1, 3, 8, 16, 32, 64, 128, 256])
def test_cfg0_blocked_every_nmin(gpu, n_min):
    g = golden("cfg0_dd_simple_128")
    c = mp.matmul_block(M(g["a"], DD), M(g["b"], DD), n_min)
    assert np.array_equal(c.data, g["c_simple"])


@pytest.mark.parametrize("n_min", [1, 3, 8, 16, 64])
def test_ragged_blocked(gpu, n_min):
    g = golden("dd_ragged_37x45x29")
    c = mp.matmul_block(M(g["a"], DD), M(g["b"], DD), n_min)
    assert np.array_equal(c.data, g[f"c_block_{n_min}"])
    assert np.array_equal(mp.matmul_simple(M(g["a"], DD), M(g["b"], DD)).data, g["c_simple"])


def test_wide_exponent(gpu):
    g = golden("dd_wide_32x48x40")
    for n_min in (16, 32, 64):
        assert np.array_equal(mp.matmul_block(M(g["a"], DD), M(g["b"], DD), n_min).data,
                              g["c_simple"])


def test_qd_golden(gpu):
    g = golden("qd_12x10x9")
    assert np.array_equal(mp.matmul_simple(M(g["a"], QD), M(g["b"], QD)).data, g["c_simple"])
    for n_min in (4, 16, 32, 64):
        assert np.array_equal(mp.matmul_block(M(g["a"], QD), M(g["b"], QD), n_min).data,
                              g["c_block_4"])


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_ewise_golden(gpu, tok):
    g = golden(f"{tok}_ewise_7x9")
    p = DD if tok == "dd" else QD
    from paper_1710_01839_b200.multiply import _ewise
    assert np.array_equal(_ewise(M(g["x"], p), M(g["y"], p), False).data, g["add"])
    assert np.array_equal(_ewise(M(g["x"], p), M(g["y"], p), True).data, g["sub"])


@pytest.mark.parametrize("name,prec,cut,leaf", [("dd_strassen_pair33_c8_l4", DD, 8, 4),
                                                ("qd_strassen_pair11_c4_l4", QD, 4, 4),
                                                ("dd_strassen_rand64_c16_l8", DD, 16, 8)])
def test_strassen_golden(gpu, name, prec, cut, leaf):
    g = golden(name)
    c = mp.matmul_strassen(M(g["a"], prec), M(g["b"], prec), cut, leaf)
    assert np.array_equal(c.data, g["c_strassen"])


def test_integer_known_answer(gpu):
    g = golden("dd_int_2x2")
    a, b = M(g["a"], DD), M(g["b"], DD)
    for c in (mp.matmul_simple(a, b), mp.matmul_block(a, b, 1),
              mp.matmul_strassen(a, b, cutoff=2, leaf_n_min=2)):
        assert np.array_equal(c.data, g["c"])


# --- the reference kernel-module protocol through the C-ABI -------------------

@pytest.mark.parametrize("tok,shape", [("dd", (37, 45, 29)), ("qd", (13, 11, 9))])
def test_protocol_functions_match_oracle(gpu, tok, shape):
    m, l, n = shape
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=31)
    kern = backend.kernels()
    assert kern.NAME == "cuda"
    c = np.zeros((m, n, a.shape[2]))
    getattr(kern, f"{tok}_simple_rows")(a, b, c, 3, m - 2)
    want = oracle.matmul_simple(a, b)
    assert np.array_equal(c[3:m - 2], want[3:m - 2]) and not c[:3].any()
    # partial cell ranges accumulate into c, exactly like the reference
    for n_min in (4, 7):
        cells = (-(-m // n_min)) * (-(-n // n_min))
        for lo, hi in ((0, cells), (1, cells - 2), (cells // 2, cells // 2 + 1)):
            got = np.full((m, n, a.shape[2]), 0.0)
            ref = np.full((m, n, a.shape[2]), 0.0)
            got[::2] = ref[::2] = want[::2]          # nonzero starting C
            getattr(kern, f"{tok}_block_cells")(a, b, got, n_min, lo, hi)
            oracle.block_cells(a, b, ref, n_min, lo, hi)
            assert np.array_equal(got, ref), (n_min, lo, hi)
    x, y = a, inputs.gemm_inputs(tok, m, l, n, seed=32)[0]
    for op in ("add", "sub"):
        out = np.zeros_like(x)
        getattr(kern, f"{tok}_ewise_{op}")(x, y, out, 2, m)
        ref = np.zeros_like(x)
        oracle.ewise(x, y, ref, 2, m, op == "sub")
        assert np.array_equal(out, ref)


def test_device_resident_and_host_results_agree(gpu):
    a, b = inputs.gemm_inputs("dd", 100, 70, 90, seed=33)
    A, B = M(a, DD), M(b, DD)
    ch = mp.matmul_block(A, B, 32)
    cd = mp.matmul_block(A.to_device(), B.to_device(), 32)
    assert cd.is_device and not ch.is_device
    assert cd == ch
    assert np.array_equal(ch.data, oracle.matmul_simple(a, b))


def test_nonfinite_raises_range_error(gpu):
    a = np.zeros((4, 4, 2))
    a[:, :, 0] = 1e300
    with pytest.raises(mp.RangeError):
        mp.matmul_block(M(a, DD), M(a, DD), 16)
    with pytest.raises(mp.RangeError):
        mp.matmul_simple(M(a, DD), M(a, DD))


# --- reference unit tests restated on the GPU ---------------------------------

@pytest.mark.parametrize("n", [2, 3, 5, 8, 16, 17])
def test_all_algorithms_exact_on_integers(gpu, n):
    rng = random.Random(0xC0FFEE + n)
    a = random_int_matrix(rng, n, n, DD)
    b = random_int_matrix(rng, n, n, DD)
    ref = mp.matmul_simple(a, b)
    for n_min in (2, 4, n):
        assert mp.matmul_block(a, b, n_min) == ref
    assert mp.matmul_strassen(a, b, cutoff=2, leaf_n_min=2) == ref
    assert np.array_equal(ref.data, oracle.matmul_simple(a.data, b.data))


@pytest.mark.parametrize("prec", [DD, QD])
def test_identity_times_matrix_is_exact(gpu, prec):
    b = M(inputs.gemm_inputs(prec.token, 5, 5, 5, seed=3)[0], prec)
    eye = mp.DenseMatrix.identity(5, prec)
    assert mp.matmul_simple(eye, b) == b
    assert mp.matmul_block(eye, b, 2) == b
    got = mp.matmul_strassen(eye, b, cutoff=2, leaf_n_min=2)
    assert mp.frobenius_rel_diff(got, b) <= 100.0 * 5 * 2.0 ** -prec.bits


def test_strassen_counts_and_odd_padding(gpu):
    rng = random.Random(5)
    a = random_int_matrix(rng, 8, 8, DD)
    b = random_int_matrix(rng, 8, 8, DD)
    st = mp.StrassenStats()
    mp.matmul_strassen(a, b, cutoff=4, leaf_n_min=4, stats=st)
    assert (st.multiplications, st.additions) == (7, 18)
    st = mp.StrassenStats()
    mp.matmul_strassen(a, b, cutoff=2, leaf_n_min=2, stats=st)
    assert (st.multiplications, st.additions) == (7 + 49, 18 + 7 * 18)
    for n, cut in ((7, 2), (9, 4), (17, 4), (20, 4)):
        ga, gb = mp.generate_test_pair(n, DD)
        got = mp.matmul_strassen(ga, gb, cut, 4)
        assert np.array_equal(got.data, oracle.strassen(ga.data, gb.data, cut, 4))
        assert mp.frobenius_rel_diff(got, mp.matmul_simple(ga, gb)) <= 100.0 * n * 2.0 ** -106


def test_run_choice_dispatch(gpu):
    rng = random.Random(9)
    a = random_int_matrix(rng, 6, 6, DD)
    b = random_int_matrix(rng, 6, 6, DD)
    ref = mp.matmul_simple(a, b)
    for tok in ("simple", "block:2", "strassen:2/2"):
        assert mp.run_choice(a, b, mp.AlgorithmChoice.parse(tok)) == ref


def test_backend_registry_with_oracle(gpu):
    """The reference's ext-vs-python equivalence test (test_backend_equiv.py)
    with the CPU oracle registered as a second protocol module."""
    import types
    mod = types.SimpleNamespace(NAME="oracle")
    for tok in ("dd", "qd"):
        setattr(mod, f"{tok}_simple_rows", oracle.simple_rows)
        setattr(mod, f"{tok}_block_cells", oracle.block_cells)
        setattr(mod, f"{tok}_ewise_add", lambda x, y, o, i0, i1: oracle.ewise(x, y, o, i0, i1, False))
        setattr(mod, f"{tok}_ewise_sub", lambda x, y, o, i0, i1: oracle.ewise(x, y, o, i0, i1, True))
    backend.register("oracle", mod)
    try:
        for tok, prec in (("dd", DD), ("qd", QD)):
            a, b = inputs.gemm_inputs(tok, 11, 13, 7, seed=41)
            A, B = M(a, prec), M(b, prec)
            cuda_simple = mp.matmul_simple(A, B, 2)
            cuda_block = mp.matmul_block(A, B, 4, 3)
            prev = backend.use("oracle")
            assert prev == "cuda" and backend.backend_name() == "oracle"
            try:
                assert mp.matmul_simple(A, B) == cuda_simple
                assert mp.matmul_block(A, B, 4, threads=3) == cuda_block
            finally:
                backend.use("cuda")
        with pytest.raises(ValueError):
            backend.use("python")
    finally:
        backend.unregister("oracle")


# --- size-independent properties at full BASELINE sizes ---------------------------

def test_cfg1_blocked_equals_simple_and_meets_exact_bound(gpu):
    """BASELINE config 1 (DD 1024^3, both input sets): blocked == simple
    bitwise for every n_min of the sweep; sampled entries checked against
    the exact rational product at 4 l u (|A||B|), u = 2^-104."""
    for wide in (False, True):
        a, b = inputs.gemm_inputs("dd", 1024, 1024, 1024, seed=0, wide=wide)
        A, B = M(a, DD).to_device(), M(b, DD).to_device()
        ref = mp.matmul_simple(A, B)
        for n_min in (16, 32, 64, 128, 256):
            assert mp.matmul_block(A, B, n_min) == ref
        c = ref.host_array()
        rows, cols = exact.sample_indices(1024, 1024, 6, seed=1)
        ratio, n = exact.bound_ratio(a, b, c, rows, cols, 104)
        assert n >= 16 and ratio <= 1.0, ratio
        # and against the compiled-C oracle on a row sample (bitwise)
        sl = slice(500, 504)
        want = np.zeros((4, 1024, 2))
        oracle.simple_rows(np.ascontiguousarray(a[sl]), b, want, 0, 4)
        assert np.array_equal(c[sl], want)


def test_cfg2_qd_blocked_sampled(gpu):
    """BASELINE config 2 (QD 1024^3): sampled rows bitwise against the
    oracle, sampled entries within 4 l u (|A||B|), u = 2^-209."""
    a, b = inputs.gemm_inputs("qd", 1024, 1024, 1024, seed=0)
    A, B = M(a, QD).to_device(), M(b, QD).to_device()
    c = mp.matmul_block(A, B, 64).host_array()
    rows = [0, 517, 1023]
    for i in rows:
        want = np.zeros((1, 1024, 4))
        oracle.simple_rows(np.ascontiguousarray(a[i:i + 1]), b, want, 0, 1)
        assert np.array_equal(c[i:i + 1], want)
    ratio, _ = exact.bound_ratio(a, b, c, rows, [0, 100, 1023], 209)
    assert ratio <= 1.0


def test_panel_split_invariance(gpu):
    """The k-panel pipelining of shard.broadcast_matmul (world size 1 here)
    is bitwise invariant in the panel size."""
    import torch
    from paper_1710_01839_b200 import shard
    a, b = inputs.gemm_inputs("dd", 256, 300, 200, seed=7)
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    ref = shard.broadcast_matmul(ta, tb, n_min=64).cpu().numpy()
    for panel in (1, 17, 64, 299):
        got = shard.broadcast_matmul(ta, tb, n_min=32, panel_rows=panel).cpu().numpy()
        assert np.array_equal(got, ref), panel
    assert np.array_equal(ref, oracle.matmul_simple(a, b))


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_protocol_reentrant_from_a_thread_pool(gpu, tok):
    """The reference drives its kernel module from a thread pool on disjoint
    ranges (multiply.py:99-112, _run_partitioned): four host threads calling
    the C-ABI cell and row kernels concurrently give the serial result."""
    from concurrent.futures import ThreadPoolExecutor
    m, l, n = 70, 53, 66
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=41)
    kern = backend.kernels()
    want = oracle.matmul_simple(a, b)
    n_min = 8
    cells = (-(-m // n_min)) * (-(-n // n_min))
    bounds = [(q * cells // 4, (q + 1) * cells // 4) for q in range(4)]
    c = np.zeros_like(want)
    with ThreadPoolExecutor(4) as pool:
        list(pool.map(lambda r: getattr(kern, f"{tok}_block_cells")(a, b, c, n_min, *r), bounds))
    assert np.array_equal(c, want)
    rows = [(q * m // 4, (q + 1) * m // 4) for q in range(4)]
    c2 = np.zeros_like(want)
    with ThreadPoolExecutor(4) as pool:
        list(pool.map(lambda r: getattr(kern, f"{tok}_simple_rows")(a, b, c2, *r), rows))
    assert np.array_equal(c2, want)


@pytest.mark.parametrize("shape", [(1, 1, 1), (1, 300, 1), (300, 1, 2), (2, 3, 300)])
@pytest.mark.parametrize("prec", [DD, QD])
def test_degenerate_shapes(gpu, shape, prec):
    """Thin and single-element products on every entry point, bit for bit."""
    m, l, n = shape
    a, b = inputs.gemm_inputs("dd" if prec is DD else "qd", m, l, n, seed=6)
    want = oracle.matmul_simple(a, b)
    A, B = M(a, prec), M(b, prec)
    for c in (mp.matmul_simple(A, B), mp.matmul_block(A, B, 4),
              mp.matmul_block(A.to_device(), B.to_device(), 64).to_host()):
        assert np.array_equal(c.data, want)
    if m == l == n:
        assert np.array_equal(mp.matmul_strassen(A, B, 2, 2).data, want)


@pytest.mark.parametrize("shape", [(0, 5, 3), (4, 0, 3), (4, 5, 0)])
def test_empty_shapes(gpu, shape):
    """The drop-in API rejects empty matrices like the reference
    (matrix.py: ShapeError); the C ABI accepts them: C untouched when
    m or n is 0, zeros when l is 0."""
    import torch
    m, l, n = shape
    with pytest.raises(mp.ShapeError):
        M(np.zeros((m, l, 2)), DD) if m * l == 0 else M(np.zeros((l, n, 2)), DD)
    A = torch.zeros((m, l, 2), dtype=torch.float64, device="cuda")
    B = torch.zeros((l, n, 2), dtype=torch.float64, device="cuda")
    C = torch.full((m, n, 2), 7.0, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for algo in (_cuda.ALGO_SIMPLE, _cuda.ALGO_BLOCK):
        _cuda.gemm_dev(2, algo, 16, m, l, n, A.data_ptr(), max(l, 1), B.data_ptr(), max(n, 1),
                       C.data_ptr(), max(n, 1), False, None, s)
        torch.cuda.synchronize()
        assert (C == 0).all() if l == 0 else (C == 7).all()
