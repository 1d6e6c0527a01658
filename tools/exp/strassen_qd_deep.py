import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
for tok, n, cuts in (("qd", 2048, (16, 32)), ("qd", 4096, (16, 32)), ("qd", 8192, (32, 64))):
    p = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
    for cut in cuts:
        mp.matmul_strassen(A, B, cut, 64); torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); mp.matmul_strassen(A, B, cut, 64); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{tok} n={n} cutoff={cut}: {min(ts):.1f} ms ({2.0 * n ** 3 / min(ts) / 1e9:.4f} T eff.)", flush=True)
    del A, B, a, b
    torch.cuda.empty_cache()
