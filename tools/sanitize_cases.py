#!/usr/bin/env python3
"""Small cases through every entry point, for compute-sanitizer runs.

Exercises: simple and every blocked tile (DD/QD), the fast DD mode, ragged
and degenerate shapes, accumulate, cell ranges, the host protocol, the
pipelined host product, batched GEMM and elementwise kernels (Strassen,
odd sizes, rectangular), the finite check and the FP64 burn kernel.
Exits non-zero on any mismatch with the oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import _cuda, backend, inputs  # noqa: E402
from paper_1710_01839_b200.matrix import DenseMatrix  # noqa: E402


def check(cond, what):
    if not cond:
        print("MISMATCH:", what)
        sys.exit(1)


def main():
    kern = backend.kernels()
    for tok in ("dd", "qd"):
        prec = mp.PrecisionSpec.parse(tok)
        for (m, l, n) in ((1, 1, 1), (3, 5, 2), (17, 9, 33), (70, 65, 67)):
            a, b = inputs.gemm_inputs(tok, m, l, n, seed=m + l + n)
            want = oracle.matmul_simple(a, b)
            A, B = DenseMatrix(m, l, prec, a), DenseMatrix(l, n, prec, b)
            check(np.array_equal(mp.matmul_simple(A, B).data, want), f"{tok} simple {m,l,n}")
            dA, dB = A.to_device(), B.to_device()
            for n_min in (1, 16, 32, 64, 128, 256):
                got = mp.matmul_block(dA, dB, n_min).host_array()
                check(np.array_equal(got, want), f"{tok} block {n_min} {m,l,n}")
                check(np.array_equal(mp.matmul_block(A, B, n_min).data, want), "host path")
            if tok == "dd":
                f = mp.matmul_block(dA, dB, 64, mode="fast").host_array()
                check(np.allclose(f[..., 0], want[..., 0], rtol=1e-14, atol=1e-300), "fast")
            c = np.zeros((m, n, prec.comps))
            cells = (-(-m // 7)) * (-(-n // 7))
            kern.__dict__[f"{tok}_block_cells"](a, b, c, 7, 1, max(1, cells - 1))
            ref = np.zeros_like(c)
            oracle.block_cells(a, b, ref, 7, 1, max(1, cells - 1))
            check(np.array_equal(c, ref), f"{tok} cells")
            for sub in (False, True):
                out = np.zeros_like(a)
                kern.__dict__[f"{tok}_ewise_{'sub' if sub else 'add'}"](a, a, out, 0, m)
                check(np.array_equal(out, oracle.ewise_new(a, a, sub)), "ewise")
        for n, cut in ((7, 2), (12, 4), (33, 8)):
            ga, gb = mp.generate_test_pair(n, prec)
            got = mp.matmul_strassen(ga, gb, cut, 4)
            check(np.array_equal(got.data, oracle.strassen(ga.data, gb.data, cut, 4)),
                  f"{tok} strassen {n}")
        a, b = inputs.gemm_inputs(tok, 40, 24, 56, seed=3)
        got = mp.matmul_strassen(DenseMatrix(40, 24, prec, a), DenseMatrix(24, 56, prec, b),
                                 4, 4, rectangular=True)
        check(got.data.shape == (40, 56, prec.comps), "rect shape")
    bad = np.zeros((4, 4, 2))
    bad[:, :, 0] = 1e300
    try:
        mp.matmul_block(DenseMatrix(4, 4, mp.PrecisionSpec.dd(), bad),
                        DenseMatrix(4, 4, mp.PrecisionSpec.dd(), bad), 16)
        check(False, "range error not raised")
    except mp.RangeError:
        pass
    # the exact tensor mode (residues, tcgen05 residue GEMMs, tensor-core CRT)
    from paper_1710_01839_b200.tensor import matmul_exact
    from oracle import exact
    for tok, (m, l, n) in (("dd", (40, 72, 36)), ("qd", (17, 33, 20))):
        prec = mp.PrecisionSpec.parse(tok)
        a, b = inputs.gemm_inputs(tok, m, l, n, seed=6)
        c = matmul_exact(DenseMatrix(m, l, prec, a).to_device(),
                         DenseMatrix(l, n, prec, b).to_device()).host_array()
        ratio, _ = exact.bound_ratio(a, b, c, range(0, m, 5), range(0, n, 7),
                                     104 if tok == "dd" else 209)
        check(ratio <= 1.0, f"{tok} exact mode bound")
    # page-locked host operands: the streamed single-launch product (under a
    # tool that serialises kernels it times out once and falls back)
    a, b = inputs.gemm_inputs("dd", 48, 160, 40, seed=7)
    pa = torch.from_numpy(a).pin_memory().numpy()
    pb = torch.from_numpy(b).pin_memory().numpy()
    c = mp.matmul_block(DenseMatrix(48, 160, mp.PrecisionSpec.dd(), pa),
                        DenseMatrix(160, 40, mp.PrecisionSpec.dd(), pb), 32).host_array()
    check(np.array_equal(c, oracle.matmul_simple(a, b)), "streamed host product")
    s = torch.zeros(64, dtype=torch.float64, device="cuda")
    _cuda.fp64_burn_dev(0, 4, 64, 10, s.data_ptr())
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
