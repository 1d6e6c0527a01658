#!/usr/bin/env python3
"""cProfile of the exact tensor mode's host side (where the wall time that
is not kernel time goes).  usage: host_profile_tensor.py dd|qd n"""
import cProfile
import os
import pstats
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1710_01839_b200 import inputs  # noqa: E402
from paper_1710_01839_b200.tensor import matmul_exact_tensors  # noqa: E402

tok, n = sys.argv[1], int(sys.argv[2])
A, B = inputs.gemm_inputs_device(tok, n, n, n, seed=0)
for _ in range(3):
    matmul_exact_tensors(A, B)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    matmul_exact_tensors(A, B)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
