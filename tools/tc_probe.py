#!/usr/bin/env python3
"""Time the tcgen05 residue GEMM against cuBLASLt's int8 GEMM (same shapes).
usage: tc_probe.py m n k batch"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1710_01839_b200 import _cuda  # noqa: E402

m, n, k, b = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 1024, 1024, 39)))
A = torch.randint(-128, 128, (b, m, k), dtype=torch.int8, device="cuda")
B = torch.randint(-128, 128, (b, n, k), dtype=torch.int8, device="cuda")
R = torch.empty((b, m, n), dtype=torch.uint8, device="cuda")
G = torch.empty((b, m, n), dtype=torch.int32, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def tc():
    _cuda.residue_gemm_dev(m, n, k, b, A.data_ptr(), B.data_ptr(), R.data_ptr(), s)


def lt():
    _cuda.int8_gemm_batched_dev(m, n, k, b, A.data_ptr(), B.data_ptr(), G.data_ptr(),
                                ws.data_ptr(), 64 << 20, s)


for name, fn in (("tcgen05 residue", tc), ("cuBLASLt int32", lt)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f"{name:16s} {m}x{n}x{k} x{b}: {t * 1e3:.1f} us  {2 * m * n * k * b / t / 1e9:.0f} TOPS",
          flush=True)
