"""Strassen with the last level's operand sums folded into the leaf tile
loads (MPMM_STRASSEN_FUSE=1, default) vs materialised by ewise launches
(=0): device time (CUDA events, min of 3) and bitwise agreement."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix

cases = [("dd", 2048, 128, 32), ("dd", 2048, 256, 32), ("dd", 2048, 512, 32),
         ("dd", 4096, 512, 32), ("dd", 8192, 1024, 32), ("qd", 1024, 128, 16),
         ("qd", 2048, 256, 16)]
for tok, n, cut, leaf in cases:
    p = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
    res, outs = {}, {}
    for fuse in ("0", "1"):
        os.environ["MPMM_STRASSEN_FUSE"] = fuse
        c = mp.matmul_strassen(A, B, cut, leaf)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c = mp.matmul_strassen(A, B, cut, leaf)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[fuse] = min(ts)
        outs[fuse] = c.data
    same = torch.equal(outs["0"], outs["1"])
    print(f"{tok} n={n} cutoff={cut}: materialised {res['0']:.2f} ms, fused {res['1']:.2f} ms "
          f"({res['0'] / res['1']:.3f}x), bitwise {'equal' if same else 'DIFFERENT'}", flush=True)
    del A, B, a, b, outs
    torch.cuda.empty_cache()
