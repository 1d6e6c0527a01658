#!/usr/bin/env python3
"""Break down the host-buffer (end-to-end) product path on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import _cuda, inputs  # noqa: E402
from paper_1710_01839_b200.matrix import DenseMatrix  # noqa: E402

n = int(os.environ.get("N", "1024"))
a, b = inputs.gemm_inputs("dd", n, n, n, seed=0)
pa = torch.from_numpy(a).pin_memory().numpy()
pb = torch.from_numpy(b).pin_memory().numpy()
A = DenseMatrix(n, n, mp.PrecisionSpec.dd(), pa)
B = DenseMatrix(n, n, mp.PrecisionSpec.dd(), pb)
Ap = DenseMatrix(n, n, mp.PrecisionSpec.dd(), a)
Bp = DenseMatrix(n, n, mp.PrecisionSpec.dd(), b)
for name, (X, Y) in (("pinned", (A, B)), ("pageable", (Ap, Bp))):
    for _ in range(3):
        mp.matmul_block(X, Y, 32)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        mp.matmul_block(X, Y, 32)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{name}: matmul_block(host, host) min {ts[0]*1e3:.3f} med {ts[5]*1e3:.3f} ms")
for _ in range(3):
    out = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    out = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
    ts.append(time.perf_counter() - t0)
print(f"pinned alloc med {sorted(ts)[5]*1e3:.3f} ms")
c = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    _cuda.gemm_host(2, 1, 32, pa, pb, c)
    ts.append(time.perf_counter() - t0)
print(f"gemm_host reuse-out med {sorted(ts)[5]*1e3:.3f} ms")
