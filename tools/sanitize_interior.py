#!/usr/bin/env python3
"""Interior-tile and speculative-QD paths on small all-interior products, for
compute-sanitizer where it is available (memcheck, racecheck: the one-barrier
k-tile pipeline and the vote barriers; the tool is closed on the round's GPU
pool, where this runs as a plain parity check).  Exits non-zero on any
mismatch with the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import _cuda, inputs  # noqa: E402


def gemm(comps, n_min, a, b):
    m, l, n = a.shape[0], a.shape[1], b.shape[1]
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    C = torch.empty((m, n, comps), dtype=torch.float64, device="cuda")
    _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, n_min, m, l, n, A.data_ptr(), l, B.data_ptr(), n,
                   C.data_ptr(), n, False, None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def main():
    for tok, comps, shape in (("dd", 2, (64, 64, 128)), ("qd", 4, (32, 48, 64))):
        m, l, n = shape
        a, b = inputs.gemm_inputs(tok, m, l, n, seed=3)
        want = oracle.matmul_simple(a, b)
        for n_min in (16, 32, 64, 128, 256):
            if not np.array_equal(gemm(comps, n_min, a, b), want):
                print("MISMATCH", tok, n_min)
                sys.exit(1)
    # speculative QD: a gate fails in the second k-tile -> fallback
    a, b = inputs.gemm_inputs("qd", 32, 48, 32, seed=4)
    a[:, 20:, 2:] = 0.0
    want = oracle.matmul_simple(a, b)
    for n_min in (16, 64):
        if not np.array_equal(gemm(4, n_min, a, b), want):
            print("MISMATCH qd fallback", n_min)
            sys.exit(1)
    # Strassen with fused leaves (sum-interior path)
    n = 128
    a, b = inputs.gemm_inputs("dd", n, n, n, seed=5)
    dd = mp.PrecisionSpec.dd()
    got = mp.matmul_strassen(mp.DenseMatrix(n, n, dd, a).to_device(),
                             mp.DenseMatrix(n, n, dd, b).to_device(), 64, 32).host_array()
    if not np.array_equal(got, oracle.strassen(a, b, 64, 32)):
        print("MISMATCH strassen")
        sys.exit(1)
    print("sanitize_interior ok")


if __name__ == "__main__":
    main()
