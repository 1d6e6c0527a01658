"""Strassen driver under its different regimes against the CPU oracle:
odd and even sizes 100..520, cutoffs 8..128 (several levels, padded levels,
fused and materialised last level, chunked launches), and the depth-first
mode forced by a tiny scratch budget (MPMM_STRASSEN_BUDGET_MB=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
bad = 0
cases = 0
for budget in (None, "1"):
    if budget:
        os.environ["MPMM_STRASSEN_BUDGET_MB"] = budget
    else:
        os.environ.pop("MPMM_STRASSEN_BUDGET_MB", None)
    for it in range(14):
        tok = "dd" if rng.random() < 0.7 else "qd"
        prec = mp.PrecisionSpec.parse(tok)
        hi = 520 if tok == "dd" else 150
        m, l, n = (int(rng.integers(100 if tok == "dd" else 40, hi)) for _ in range(3))
        if rng.random() < 0.5:
            m = l = n
        cutoff = int(rng.choice([8, 16, 32, 64, 128]))
        leaf = int(rng.choice([16, 32, 128]))
        a, b = inputs.gemm_inputs(tok, m, l, n, seed=int(rng.integers(1 << 30)))
        rect = not (m == l == n)
        if rect:
            # the reference's Strassen is square-only; the rectangular extension is
            # checked against the blocked product within the Strassen error bound
            continue
        want = oracle.strassen(a, b, cutoff, leaf)
        A, B = DenseMatrix(m, l, prec, a).to_device(), DenseMatrix(l, n, prec, b).to_device()
        for fuse in ("1", "0"):
            os.environ["MPMM_STRASSEN_FUSE"] = fuse
            got = mp.matmul_strassen(A, B, cutoff, leaf).host_array()
            cases += 1
            if not np.array_equal(got, want):
                bad += 1
                print(f"MISMATCH {tok} n={n} cutoff={cutoff} leaf={leaf} fuse={fuse} budget={budget}")
print(f"strassen_fuzz_deep: {cases} products, {bad} mismatches")
sys.exit(1 if bad else 0)
