#!/usr/bin/env python3
"""Time matmul_strassen on device-resident operands (CUDA events)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import inputs  # noqa: E402
from paper_1710_01839_b200.matrix import DenseMatrix  # noqa: E402

for spec in sys.argv[1:] or ["dd:2048:512:64", "dd:2048:256:64"]:
    tok, n, cut, leaf = spec.split(":")
    n, cut, leaf = int(n), int(cut), int(leaf)
    A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=0)
    prec = mp.PrecisionSpec.parse(tok)
    a, b = DenseMatrix(n, n, prec, A), DenseMatrix(n, n, prec, B)
    mp.matmul_strassen(a, b, cut, leaf)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        mp.matmul_strassen(a, b, cut, leaf)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = min(ts)
    print(f"{spec}: {t:.2f} ms  {2 * n ** 3 / t / 1e9:.3f} T 2mnl/s eff", flush=True)
