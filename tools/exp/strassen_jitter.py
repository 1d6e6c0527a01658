"""DD 8192^3 Strassen at cutoff 128 / 256 (and QD 2048^3 at 256): five
repetitions in one process -- device time by CUDA events and the host's
wall time of the call (a call that returns late is planning on the host)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
for tok, n, cuts in (("dd", 8192, (128, 256)), ("dd", 2048, (128,)), ("qd", 2048, (256,))):
    p = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
    for cut in cuts:
        c = mp.matmul_strassen(A, B, cut, 128); torch.cuda.synchronize()
        ts, hs = [], []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(); c = mp.matmul_strassen(A, B, cut, 128); e1.record()
            hs.append(round((time.perf_counter() - t0) * 1e3, 1))
            e1.synchronize()
            ts.append(round(e0.elapsed_time(e1), 1))
        print(f"{tok} n={n} cutoff={cut}: device ms {ts}  host call ms {hs}", flush=True)
    del A, B, a, b
