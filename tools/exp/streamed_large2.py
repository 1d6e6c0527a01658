"""Steady-state host products at large sizes (page-locked results cached after warm-up)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
for tok, n, nmin in (("dd", 4096, 32), ("qd", 2048, 16)):
    prec = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs(tok, n, n, n, seed=2)
    pa, pb = torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(b).pin_memory().numpy()
    A, B = DenseMatrix(n, n, prec, pa), DenseMatrix(n, n, prec, pb)
    c = None
    t00 = time.perf_counter()
    for _ in range(3):
        c = mp.matmul_block(A, B, nmin)
    tw = (time.perf_counter() - t00) / 3
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); c = mp.matmul_block(A, B, nmin); ts.append(time.perf_counter() - t0)
    Ad, Bd = A.to_device(), B.to_device()
    mp.matmul_block(Ad, Bd, nmin); torch.cuda.synchronize()
    t1 = time.perf_counter(); d = mp.matmul_block(Ad, Bd, nmin); torch.cuda.synchronize(); td = time.perf_counter() - t1
    print(f"{tok} {n}: host warm-up mean {tw*1e3:.1f} ms, steady {min(ts)*1e3:.1f} ms, device {td*1e3:.1f} ms", flush=True)
