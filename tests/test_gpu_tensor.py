"""The exact int8 tensor-core mode: exact product, correctly rounded."""

from fractions import Fraction

import numpy as np
import pytest

from oracle import exact
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
from paper_1710_01839_b200.tensor import matmul_exact, plan
from paper_1710_01839_b200.verify import exact_bound_ratio

pytestmark = pytest.mark.gpu


def M(x, prec):
    return DenseMatrix(x.shape[0], x.shape[1], prec, np.ascontiguousarray(x))


def _exact_entry(a, b, i, j):
    return sum(sum(Fraction(float(v)) for v in a[i, k]) * sum(Fraction(float(v)) for v in b[k, j])
               for k in range(a.shape[1]))


def _rn_expansion(x, comps):
    out = []
    for _ in range(comps):
        d = float(x)          # Fraction -> nearest double
        out.append(d)
        x -= Fraction(d)
    return out


@pytest.mark.parametrize("tok,shape,wide", [("dd", (20, 33, 17), False), ("dd", (9, 64, 11), True),
                                            ("qd", (12, 10, 9), False)])
def test_exact_and_correctly_rounded(gpu, tok, shape, wide):
    prec = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs(tok, *shape, seed=7, wide=wide)
    c = matmul_exact(M(a, prec), M(b, prec)).data
    for i, j in ((0, 0), (shape[0] - 1, shape[2] - 1), (3, 5)):
        want = _rn_expansion(_exact_entry(a, b, i, j), prec.comps)
        assert list(c[i, j]) == want, (i, j)


def test_plan_splits_wide_and_qd(gpu):
    import torch
    a, b = inputs.gemm_inputs("dd", 64, 64, 64, seed=1)
    pl = plan(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert len(pl.jobs) == 1 and pl.jobs[0][2] <= 54
    a, b = inputs.gemm_inputs("qd", 32, 32, 32, seed=1)
    pl = plan(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert len(pl.jobs) in (2, 4)     # hi/lo of one operand, or of both
    cover = sorted((x, y) for ia, ib, _ in pl.jobs for x in range(*pl.ranges_a[ia])
                   for y in range(*pl.ranges_b[ib]))
    assert cover == [(x, y) for x in range(4) for y in range(4)]


def test_speculative_plan_reuse_and_replan(gpu):
    """Same shape, wider data: the cached plan no longer fits, the product
    is replanned and still exact; narrower data afterwards drops it."""
    import torch
    from paper_1710_01839_b200 import tensor
    a, b = inputs.gemm_inputs("dd", 12, 40, 10, seed=2)
    wa, wb = inputs.gemm_inputs("dd", 12, 40, 10, seed=3, wide=True)
    for x, y in ((a, b), (a, b), (wa, wb), (wa, wb), (a, b)):
        c = tensor.matmul_exact_tensors(torch.from_numpy(x).cuda(),
                                        torch.from_numpy(y).cuda()).cpu().numpy()
        for i, j in ((0, 0), (11, 9), (5, 3)):
            assert list(c[i, j]) == _rn_expansion(_exact_entry(x, y, i, j), 2), (i, j)


def test_integers_and_zero_rows(gpu):
    dd = mp.PrecisionSpec.dd()
    a = np.zeros((6, 5, 2))
    b = np.zeros((5, 4, 2))
    a[1:, :, 0] = np.arange(25).reshape(5, 5) - 12
    b[..., 0] = np.arange(20).reshape(5, 4) % 7
    c = matmul_exact(M(a, dd), M(b, dd)).data
    assert np.array_equal(c[..., 0], a[..., 0] @ b[..., 0]) and not c[..., 1].any()


@pytest.mark.parametrize("wide", [False, True])
def test_cfg1_every_entry_and_speed(gpu, wide):
    import torch
    dd = mp.PrecisionSpec.dd()
    A, B = inputs.gemm_inputs_device("dd", 1024, 1024, 1024, seed=0, wide=wide)
    Am, Bm = DenseMatrix(1024, 1024, dd, A), DenseMatrix(1024, 1024, dd, B)
    c = matmul_exact(Am, Bm)
    worst, r, _ = exact_bound_ratio(Am, Bm, c)
    ref = mp.matmul_block(Am, Bm, 32)
    worst_ref, _, _ = exact_bound_ratio(Am, Bm, ref)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        matmul_exact(Am, Bm)
    e.record()
    e.synchronize()
    t = s.elapsed_time(e) / 3e3
    print(f"tensor mode DD 1024^3 wide={wide}: max ratio {worst:.3e} (mirror {worst_ref:.3e}), "
          f"{t*1e3:.3f} ms, {2*1024**3/t/1e9:.1f} G 2mnl/s")
    assert worst <= worst_ref and worst <= 1e-3


@pytest.mark.parametrize("tok,wide", [("dd", False), ("dd", True), ("qd", False),
                                      ("qd", True)])
def test_every_entry_correctly_rounded(gpu, tok, wide):
    """All entries (not a sample) against exact rational arithmetic: the
    DD fast rounding path (128-bit window + sticky) and the limb paths must
    both give the nearest expansion."""
    prec = mp.PrecisionSpec.parse(tok)
    m, l, n = (16, 24, 12) if tok == "dd" else (6, 8, 5)
    a, b = inputs.gemm_inputs(tok, m, l, n, seed=11, wide=wide and tok == "dd")
    if wide and tok == "qd":       # the spec's wide set is DD-only: scale QD entries by 2^k
        rng = np.random.default_rng(12)
        a = np.ldexp(a, rng.integers(-30, 31, a.shape[:2])[..., None])
        b = np.ldexp(b, rng.integers(-30, 31, b.shape[:2])[..., None])
    # cancellation-heavy rows: the remainder after hi can be tiny
    a[0, :, :] = a[1, :, :]
    a[0, ::2, :] *= -1
    c = matmul_exact(M(a, prec), M(b, prec)).data
    for i in range(m):
        for j in range(n):
            want = _rn_expansion(_exact_entry(a, b, i, j), prec.comps)
            assert list(c[i, j]) == want, (i, j)


def test_graph_replay_same_operands_and_in_place_change(gpu):
    """Same operands three times: the third product replays the captured
    graph; then the operands change in place (same addresses, wider data):
    the replay's width check sends it back to the eager path, still exact."""
    import torch
    from paper_1710_01839_b200 import tensor
    a, b = inputs.gemm_inputs("dd", 12, 40, 10, seed=5)
    wa, wb = inputs.gemm_inputs("dd", 12, 40, 10, seed=6, wide=True)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    outs = [tensor.matmul_exact_tensors(A, B).cpu().numpy() for _ in range(4)]
    for c in outs[1:]:
        assert np.array_equal(c, outs[0])
    for i, j in ((0, 0), (11, 9)):
        assert list(outs[-1][i, j]) == _rn_expansion(_exact_entry(a, b, i, j), 2)
    A.copy_(torch.from_numpy(wa))
    B.copy_(torch.from_numpy(wb))
    c = tensor.matmul_exact_tensors(A, B).cpu().numpy()
    for i, j in ((0, 0), (11, 9), (4, 4)):
        assert list(c[i, j]) == _rn_expansion(_exact_entry(wa, wb, i, j), 2), (i, j)


@pytest.mark.parametrize("tok,n", [("dd", 4096), ("qd", 2048), ("dd", 1000)])
def test_large_and_unaligned_sampled_exact(gpu, tok, n):
    """Large sizes (DD 4096: cluster-pair tcgen05 residue GEMMs)
    and with padded tiles (1000 is no multiple of 128/256): sampled entries
    against the exact superaccumulator verifier; a correctly rounded
    result uses at most ~2^-104 / (4 l 2^-104) of the bound."""
    prec = mp.PrecisionSpec.parse(tok)
    A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    Am, Bm = DenseMatrix(n, n, prec, A), DenseMatrix(n, n, prec, B)
    c = matmul_exact(Am, Bm)
    worst, _, _ = exact_bound_ratio(Am, Bm, c, samples=2000)
    assert worst <= 1e-3, worst


def test_nonfinite_and_empty(gpu):
    import torch
    from paper_1710_01839_b200 import tensor
    from paper_1710_01839_b200.errors import RangeError
    a, b = inputs.gemm_inputs("dd", 9, 7, 5, seed=3)
    a[2, 3, 0] = np.inf
    with pytest.raises(RangeError):
        tensor.matmul_exact_tensors(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    b[1, 1, 1] = np.nan
    a[2, 3, 0] = 1.0
    with pytest.raises(RangeError):
        tensor.matmul_exact_tensors(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    z = tensor.matmul_exact_tensors(torch.zeros((4, 0, 2), dtype=torch.float64, device="cuda"),
                                    torch.zeros((0, 3, 2), dtype=torch.float64, device="cuda"))
    assert z.shape == (4, 3, 2) and not z.any()
    # after the errors the same shapes work again
    a, b = inputs.gemm_inputs("dd", 9, 7, 5, seed=4)
    c = tensor.matmul_exact_tensors(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert list(c.cpu().numpy()[0, 0]) == _rn_expansion(_exact_entry(a, b, 0, 0), 2)


_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1710_01839_b200 import inputs, tensor
tok, n, out = sys.argv[2], int(sys.argv[3]), sys.argv[4]
A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=5)
np.save(out, tensor.matmul_exact_tensors(A, B).cpu().numpy())
"""


@pytest.mark.parametrize("env", [{"MPMM_EXACT_GEMM": "lt"}, {"MPMM_COMBINE": "cuda"},
                                 {"MPMM_EXACT_GEMM": "lt", "MPMM_COMBINE": "cuda"}])
@pytest.mark.parametrize("tok,n", [("dd", 512), ("qd", 256)])
def test_fallback_paths_bit_identical(gpu, tmp_path, env, tok, n):
    """The default path (tcgen05 residue GEMMs, byte residues, tensor-core
    CRT sums) and the fallbacks (cuBLASLt int32 residue products; CUDA-core
    CRT sums), forced in child processes: all return the exact product
    rounded once, so the same bits."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for k, e in enumerate(({}, env)):
        path = str(tmp_path / f"c{k}.npy")
        r = subprocess.run([sys.executable, "-c", _CHILD, root, tok, str(n), path], cwd=root,
                           env=dict(os.environ, **e), capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


def _exact_scaled(x_comps, shift):
    """sum of the components times 2^shift as an exact integer"""
    from fractions import Fraction
    v = sum(Fraction(float(c)) for c in x_comps) * (Fraction(2) ** shift)
    assert v.denominator == 1
    return v.numerator


@pytest.mark.parametrize("by_cols", [0, 1])
@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_residue_kernels_exact(gpu, by_cols, tok):
    """mpmm_oz_residues_dev (the residue kernels) against exact
    big-integer residues, centred into int8, for a ragged operand with
    signs, zeros and a wide exponent spread: every byte."""
    import torch
    from paper_1710_01839_b200 import _cuda
    from paper_1710_01839_b200.tensor import MODULI
    comps = 2 if tok == "dd" else 4
    rows, cols = 37, 150
    a, _ = inputs.gemm_inputs(tok, rows, cols, 3, seed=21)
    a[3, 7] = 0.0
    a[5] *= 2.0 ** 40
    a[:, 11] *= -1.0
    X = torch.from_numpy(a).cuda()
    # the shift makes every entry of a row (column) an integer: -min low bit
    odim = cols if by_cols else rows
    shifts = []
    for o in range(odim):
        vals = a[:, o] if by_cols else a[o]
        low = min((int(np.frexp(v)[1]) - 53 for e in vals for v in e if v != 0.0), default=0)
        shifts.append(-low)
    sh = torch.tensor(shifts, dtype=torch.int32, device="cuda")
    ints = [[_exact_scaled(a[r, c], shifts[c if by_cols else r]) for c in range(cols)]
            for r in range(rows)]
    bits = max(abs(v).bit_length() for row in ints for v in row) + 1
    words = (bits + 31) // 32
    N = 39
    if by_cols:
        R = torch.zeros((N, cols, rows + 11), dtype=torch.int8, device="cuda")   # pitch 48
        rp, rpl = rows + 11, cols * (rows + 11)
    else:
        R = torch.zeros((N, rows, cols + 10), dtype=torch.int8, device="cuda")
        rp, rpl = cols + 10, rows * (cols + 10)
    _cuda.oz_residues_dev(by_cols, comps, 0, comps, rows, cols, X.data_ptr(), cols, sh.data_ptr(),
                          N, words, R.data_ptr(), rp, rpl)
    torch.cuda.synchronize()
    got = R.cpu().numpy()
    for t in range(N):
        p = MODULI[t]
        for r in range(rows):
            for c in range(cols):
                v = ints[r][c] % p
                if v > p // 2:
                    v -= p
                if v > 127:
                    v -= p
                g = got[t, c, r] if by_cols else got[t, r, c]
                assert g == v, (t, r, c, g, v)
