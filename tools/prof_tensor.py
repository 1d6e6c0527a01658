#!/usr/bin/env python3
"""Run the exact tensor mode a few times (for ncu launch lists)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1710_01839_b200 import inputs  # noqa: E402
from paper_1710_01839_b200.tensor import matmul_exact_tensors  # noqa: E402

tok = sys.argv[1] if len(sys.argv) > 1 else "dd"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=0)
for _ in range(3):
    matmul_exact_tensors(A, B)
torch.cuda.synchronize()
import time  # noqa: E402
t0 = time.perf_counter()
for _ in range(5):
    matmul_exact_tensors(A, B)
torch.cuda.synchronize()
print(f"{tok} {n}: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per product (wall)")
