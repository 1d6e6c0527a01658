import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
p = mp.PrecisionSpec.parse("dd")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cut = int(sys.argv[2]) if len(sys.argv) > 2 else 128
a, b = inputs.gemm_inputs_device("dd", n, n, n, seed=1)
A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
c = mp.matmul_strassen(A, B, cut, 32)
torch.cuda.synchronize()
print("done")
