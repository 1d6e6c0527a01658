#!/usr/bin/env python3
"""Randomised parity of the blocked kernels against the CPU oracle: random
shapes around the tile and k-tile boundaries (interior and edge tiles mixed),
every block size, both precisions, overwrite / accumulate, contiguous and
strided operands, zero-sprinkled QD operands (speculation fallback).
usage: fuzz_gemm.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1710_01839_b200 import _cuda, inputs  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    stream = torch.cuda.current_stream().cuda_stream
    bad = 0
    for it in range(cases):
        tok = "dd" if rng.random() < 0.6 else "qd"
        comps = 2 if tok == "dd" else 4
        big = 192 if tok == "dd" else 80
        m, n = (int(rng.choice([16, 32, 48, 64, 96, 128, big, int(rng.integers(1, big))]))
                for _ in range(2))
        l = int(rng.choice([8, 16, 32, 48, 64, 96, int(rng.integers(1, 100))]))
        n_min = int(rng.choice([16, 32, 64, 128, 256]))
        a, b = inputs.gemm_inputs(tok, m, l, n, seed=int(rng.integers(1 << 30)))
        if tok == "qd" and rng.random() < 0.4:      # gates fail somewhere
            mask = rng.random((m, l, 1)) < 0.97
            a = a * mask
        accumulate = rng.random() < 0.3
        pad = int(rng.integers(0, 3)) * 8            # strided views
        A = torch.zeros((m, l + pad, comps), dtype=torch.float64, device="cuda")
        B = torch.zeros((l, n + pad, comps), dtype=torch.float64, device="cuda")
        C = torch.zeros((m, n + pad, comps), dtype=torch.float64, device="cuda")
        A[:, :l] = torch.from_numpy(a).cuda()
        B[:, :n] = torch.from_numpy(b).cuda()
        want = oracle.matmul_simple(np.ascontiguousarray(a), b)
        if accumulate:
            c0, _ = inputs.gemm_inputs(tok, m, 1, n, seed=int(rng.integers(1 << 30)))
            c0 = np.ascontiguousarray(np.broadcast_to(c0[:, :1, :], (m, n, comps)))
            C[:, :n] = torch.from_numpy(c0).cuda()
            want = oracle.matmul_block(np.ascontiguousarray(a), b, 1 << 20, c=c0.copy())
        _cuda.gemm_dev(comps, _cuda.ALGO_BLOCK, n_min, m, l, n, A.data_ptr(), l + pad,
                       B.data_ptr(), n + pad, C.data_ptr(), n + pad, accumulate, None, stream)
        torch.cuda.synchronize()
        got = C[:, :n].cpu().numpy()
        ok = np.array_equal(got, want) and not C[:, n:].any().item()
        if not ok:
            bad += 1
            print(f"MISMATCH {tok} m={m} l={l} n={n} n_min={n_min} acc={accumulate} pad={pad}")
    print(f"fuzz_gemm: {cases} cases, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
