#!/usr/bin/env python3
"""Randomised parity of the other callers of the blocked kernels against the
CPU oracle: Strassen (materialised and fused leaves, odd sizes, DD/QD), and
host-buffer products in both streaming orders (k-panels, tile order) with
zero-sprinkled QD operands.  usage: fuzz_paths.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import inputs  # noqa: E402
from paper_1710_01839_b200.matrix import DenseMatrix  # noqa: E402


def pin(x):
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 9)
    bad = 0
    for it in range(cases):
        tok = "dd" if rng.random() < 0.6 else "qd"
        prec = mp.PrecisionSpec.parse(tok)
        # Strassen
        n = int(rng.choice([64, 96, 128, 130, 200, 256])) if tok == "dd" else \
            int(rng.choice([32, 48, 64, 66]))
        cutoff = int(rng.choice([16, 32, 64, 128]))
        leaf = int(rng.choice([16, 32, 64]))
        a, b = inputs.gemm_inputs(tok, n, n, n, seed=int(rng.integers(1 << 30)))
        want = oracle.strassen(a, b, cutoff, leaf)
        A, B = DenseMatrix(n, n, prec, a).to_device(), DenseMatrix(n, n, prec, b).to_device()
        for fuse in ("1", "0"):
            os.environ["MPMM_STRASSEN_FUSE"] = fuse
            got = mp.matmul_strassen(A, B, cutoff, leaf).host_array()
            if not np.array_equal(got, want):
                bad += 1
                print(f"MISMATCH strassen {tok} n={n} cutoff={cutoff} leaf={leaf} fuse={fuse}")
        os.environ.pop("MPMM_STRASSEN_FUSE", None)
        # host-buffer product, both streaming orders
        m, l, nn = (int(rng.choice([32, 64, 96, 128, int(rng.integers(1, 160))])),
                    int(rng.choice([128, 192, 256, 320, int(rng.integers(128, 400))])),
                    int(rng.choice([32, 64, 128, int(rng.integers(1, 160))])))
        if tok == "qd":
            m, nn = min(m, 64), min(nn, 64)
        a, b = inputs.gemm_inputs(tok, m, l, nn, seed=int(rng.integers(1 << 30)))
        if tok == "qd" and rng.random() < 0.5:
            a = a * (rng.random((m, l, 1)) < 0.98)
        want = oracle.matmul_simple(np.ascontiguousarray(a), b)
        n_min = int(rng.choice([16, 32, 64, 128, 256]))
        for tile_mb in ("0", "1000000"):
            os.environ["MPMM_STREAM_TILE_MB"] = tile_mb
            Ah, Bh = DenseMatrix(m, l, prec, pin(a)), DenseMatrix(l, nn, prec, pin(b))
            got = mp.matmul_block(Ah, Bh, n_min).host_array()
            if not np.array_equal(got, want):
                bad += 1
                print(f"MISMATCH host {tok} m={m} l={l} n={nn} n_min={n_min} tile_mb={tile_mb}")
        os.environ.pop("MPMM_STREAM_TILE_MB", None)
    print(f"fuzz_paths: {cases} cases, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
