"""Per-call times of matmul_block(host, host) before/after the bench's other phases."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, inputs
from paper_1710_01839_b200.matrix import DenseMatrix
n = 1024
a, b = inputs.gemm_inputs("dd", n, n, n, seed=0)
prec = mp.PrecisionSpec.dd()
pa, pb = torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(b).pin_memory().numpy()
Ah, Bh = DenseMatrix(n, n, prec, pa), DenseMatrix(n, n, prec, pb)

def e2e(tag):
    for _ in range(3):
        mp.matmul_block(Ah, Bh, 32)
    torch.cuda.synchronize()
    ts = []
    t00 = time.perf_counter()
    for _ in range(20):
        t0 = time.perf_counter()
        ch = mp.matmul_block(Ah, Bh, 32)
        ts.append((time.perf_counter() - t0) * 1e3)
    tot = (time.perf_counter() - t00) * 1e3 / 20
    print(f"{tag}: per call min {min(ts):.3f} med {statistics.median(ts):.3f} max {max(ts):.3f} mean-of-loop {tot:.3f} ms", flush=True)

e2e("cold process")
A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(10):
    flush.zero_(); torch.cuda._sleep(10_000_000)
    C = torch.empty((n, n, 2), dtype=torch.float64, device="cuda")
    _cuda.gemm_dev(2, _cuda.ALGO_BLOCK, 32, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, False, None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
e2e("after device GEMMs + sleeps")
from paper_1710_01839_b200.tensor import matmul_exact_tensors
for _ in range(8):
    matmul_exact_tensors(A, B)
torch.cuda.synchronize()
e2e("after tensor mode")
