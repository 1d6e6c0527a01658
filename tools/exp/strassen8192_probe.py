import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
p = mp.PrecisionSpec.parse("dd")
n = 8192
a, b = inputs.gemm_inputs_device("dd", n, n, n, seed=1)
A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
for cut, leaf in ((128, 32), (128, 128), (256, 32), (256, 128), (512, 128)):
    for fuse in ("0", "1"):
        os.environ["MPMM_STRASSEN_FUSE"] = fuse
        mp.matmul_strassen(A, B, cut, leaf); torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); c = mp.matmul_strassen(A, B, cut, leaf); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"dd 8192 cutoff={cut} leaf n_min={leaf} fuse={fuse}: {min(ts):.1f} ms", flush=True)
