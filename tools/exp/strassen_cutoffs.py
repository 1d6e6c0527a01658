"""Strassen by cutoff (32 ... 512) at DD 2048/4096/8192 and QD 2048/4096:
device time (events, min of 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
for tok, n, cuts in (("dd", 2048, (32, 64, 128, 256)), ("dd", 4096, (32, 64, 128, 256)),
                     ("dd", 8192, (32, 64, 128, 256)), ("qd", 2048, (32, 64, 128, 256)),
                     ("qd", 4096, (64, 128, 256))):
    p = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
    for cut in cuts:
        try:
            mp.matmul_strassen(A, B, cut, 128); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); mp.matmul_strassen(A, B, cut, 128); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            print(f"{tok} n={n} cutoff={cut}: {min(ts):.2f} ms  ({2.0 * n ** 3 / min(ts) / 1e9:.3f} T eff.)", flush=True)
        except Exception as ex:
            print(f"{tok} n={n} cutoff={cut}: {type(ex).__name__} {ex}", flush=True)
    del A, B, a, b
    torch.cuda.empty_cache()
