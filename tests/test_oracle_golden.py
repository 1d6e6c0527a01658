"""Pin the CPU oracle against the reference itself (no GPU needed).

Golden vectors in tests/golden/ were produced by the reference package
(tests/golden/make_golden.py); oracle/_ref is the reference's own Cython
kernel module compiled from /root/reference (``make -C oracle ref``).
"""

import numpy as np
import pytest

import oracle
from oracle import exact
from conftest import golden
from paper_1710_01839_b200 import inputs


def test_cfg0_simple_and_blocked():
    g = golden("cfg0_dd_simple_128")
    assert np.array_equal(oracle.matmul_simple(g["a"], g["b"]), g["c_simple"])
    assert np.array_equal(oracle.matmul_block(g["a"], g["b"], 32, threads=4), g["c_simple"])


@pytest.mark.parametrize("n_min", [1, 3, 8, 16, 64])
def test_ragged_blocked_equals_reference(n_min):
    g = golden("dd_ragged_37x45x29")
    assert np.array_equal(oracle.matmul_block(g["a"], g["b"], n_min, threads=3),
                          g[f"c_block_{n_min}"])


def test_wide_exponent():
    g = golden("dd_wide_32x48x40")
    assert np.array_equal(oracle.matmul_simple(g["a"], g["b"]), g["c_simple"])


def test_qd_simple_and_blocked():
    g = golden("qd_12x10x9")
    assert np.array_equal(oracle.matmul_simple(g["a"], g["b"]), g["c_simple"])
    assert np.array_equal(oracle.matmul_block(g["a"], g["b"], 4), g["c_block_4"])


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_ewise(tok):
    g = golden(f"{tok}_ewise_7x9")
    assert np.array_equal(oracle.ewise_new(g["x"], g["y"], False), g["add"])
    assert np.array_equal(oracle.ewise_new(g["x"], g["y"], True), g["sub"])


@pytest.mark.parametrize("name,cut,leaf", [("dd_strassen_pair33_c8_l4", 8, 4),
                                           ("qd_strassen_pair11_c4_l4", 4, 4),
                                           ("dd_strassen_rand64_c16_l8", 16, 8)])
def test_strassen(name, cut, leaf):
    g = golden(name)
    assert np.array_equal(oracle.strassen(g["a"], g["b"], cut, leaf), g["c_strassen"])


def test_compress4_and_vectorised_generator():
    g = golden("qd_compress4_limbs")
    got = np.array([oracle.compress4(r) for r in g["raw"]])
    assert np.array_equal(got, g["out"])
    dense = [i for i in range(len(g["raw"])) if np.all(g["raw"][i] != 0.0)]
    vec = inputs._compress4_dense_vec([g["raw"][dense, q] for q in range(4)])
    assert np.array_equal(vec, g["out"][dense])


def test_integer_known_answer():
    g = golden("dd_int_2x2")
    assert np.array_equal(oracle.matmul_simple(g["a"], g["b"]), g["c"])
    assert g["c"][:, :, 0].tolist() == [[19.0, 22.0], [43.0, 50.0]]


def test_generators_pinned():
    g = golden("cfg0_dd_simple_128")
    a, b = inputs.gemm_inputs("dd", 128, 128, 128, seed=0)
    assert np.array_equal(a, g["a"]) and np.array_equal(b, g["b"])
    for name, args in (("dd_wide_32x48x40", ("dd", 32, 48, 40, 12, True)),
                       ("qd_12x10x9", ("qd", 12, 10, 9, 13, False))):
        g = golden(name)
        a, b = inputs.gemm_inputs(args[0], *args[1:4], seed=args[4], wide=args[5])
        assert np.array_equal(a, g["a"]) and np.array_equal(b, g["b"])


def test_eft_known_answers():
    # reference tests/test_eft.py:16-39
    p, e = oracle.two_prod(2.0 ** 27 + 1, 2.0 ** 27 + 1)
    assert (p, e) == (2.0 ** 54 + 2.0 ** 28, 1.0)


def test_exact_checker_on_reference_outputs():
    # the reference meets the north_star bound
    g = golden("cfg0_dd_simple_128")
    rows, cols = exact.sample_indices(128, 128, 6)
    ratio, n = exact.bound_ratio(g["a"], g["b"], g["c_simple"], rows, cols, 104)
    assert n > 0 and ratio < 1e-2
    g = golden("qd_12x10x9")
    ratio, _ = exact.bound_ratio(g["a"], g["b"], g["c_simple"], range(12), range(9), 209)
    assert ratio < 1e-2
    # and it detects a one-ulp perturbation of the low limb of a large entry
    bad = g["c_simple"].copy()
    bad[0, 0, 0] = np.nextafter(bad[0, 0, 0], np.inf)
    ratio, _ = exact.bound_ratio(g["a"], g["b"], bad, [0], [0], 209)
    assert ratio > 1.0


ref = oracle.ref_kernels()


@pytest.mark.skipif(ref is None, reason="oracle/_ref not built (make -C oracle ref)")
@pytest.mark.parametrize("tok,shape,n_min", [("dd", (23, 31, 17), 5), ("qd", (9, 7, 11), 3),
                                             ("dd", (64, 64, 64), 16)])
def test_oracle_matches_compiled_reference(tok, shape, n_min):
    m, l, n = shape
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=21)
    assert np.array_equal(oracle.matmul_simple(a, b), oracle.matmul_simple(a, b, kernels=ref))
    assert np.array_equal(oracle.matmul_block(a, b, n_min),
                          oracle.matmul_block(a, b, n_min, kernels=ref))
    out = np.zeros_like(a)
    getattr(ref, f"{tok}_ewise_sub")(a, a[::-1].copy(), out, 0, m)
    assert np.array_equal(out, oracle.ewise_new(a, a[::-1].copy(), True))


EDGE = ["edge_dd_big995", "edge_dd_big996", "edge_dd_big997", "edge_dd_big1000",
        "edge_dd_big996_9", "edge_dd_tiny969", "edge_dd_tiny1000", "edge_dd_tiny1040",
        "edge_dd_subnormal", "edge_dd_zeros", "edge_dd_inf_nan", "edge_dd_overflow",
        "edge_qd_zeros", "edge_qd_big997", "edge_qd_tiny"]


def same_bits(x, y):
    """Bitwise equal, except that any NaN matches any NaN (payloads are
    platform-dependent: x86 and the GPU produce different default NaNs)."""
    nx, ny = np.isnan(x), np.isnan(y)
    if not np.array_equal(nx, ny):
        return False
    return np.array_equal(np.where(nx, 0, x.view(np.int64)), np.where(ny, 0, y.view(np.int64)))


@pytest.mark.parametrize("name", EDGE)
def test_edge_goldens(name):
    """EFT-domain edges (eft.py:19-24): the oracle's Dekker TwoProd gives the
    reference's results, NaN where the reference's split overflows."""
    g = golden(name)
    n_min = int(g["n_min"])
    assert same_bits(oracle.matmul_simple(g["a"], g["b"]), g["c"])
    assert same_bits(oracle.matmul_block(g["a"], g["b"], n_min), g["c"])
    assert bool(g["raises"]) == (not np.isfinite(g["c"]).all())


def test_edge_strassen_golden():
    g = golden("edge_dd_strassen_big")
    assert same_bits(oracle.strassen(g["a"], g["b"], 4, 2), g["c"])


def test_edge_goldens_leave_the_dfma_domain():
    """The edge set is not vacuous: several cases are outside the domain
    where a DFMA TwoProd equals Dekker's (the GPU must take its Dekker path
    there) -- checked with the host restatement of the domain test."""
    from paper_1710_01839_b200 import domain
    outside = [n for n in EDGE if domain.unsafe(golden(n)["a"], golden(n)["b"])]
    assert {"edge_dd_big1000", "edge_dd_inf_nan", "edge_dd_subnormal",
            "edge_dd_tiny1040", "edge_qd_big997"} <= set(outside)
    assert "edge_dd_zeros" not in outside and "edge_qd_zeros" not in outside
