"""e2e A/B: fresh page-locked result per call (the API's pattern) vs a reused one."""
import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, inputs
from paper_1710_01839_b200.matrix import DenseMatrix
n = 1024
a, b = inputs.gemm_inputs("dd", n, n, n, seed=0)
pa, pb = torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(b).pin_memory().numpy()
A, B = DenseMatrix(n, n, mp.PrecisionSpec.dd(), pa), DenseMatrix(n, n, mp.PrecisionSpec.dd(), pb)
def run(tag, fn, reps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{tag}: med {statistics.median(ts):.3f} min {min(ts):.3f} ms", flush=True)
state = {}
def api():
    state["c"] = mp.matmul_block(A, B, 32)      # keeps the previous result alive, like bench
c = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
ring = [torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
k = [0]
def reuse():
    _cuda.gemm_host(2, 1, 32, pa, pb, c)
def rotate():
    k[0] = (k[0] + 1) % 4
    _cuda.gemm_host(2, 1, 32, pa, pb, ring[k[0]])
for r in range(2):
    run(f"[{os.environ.get('MPMM_HOST_STREAMED', 'default')}] api (fresh result)", api)
    run(f"[{os.environ.get('MPMM_HOST_STREAMED', 'default')}] reuse one out", reuse)
    run(f"[{os.environ.get('MPMM_HOST_STREAMED', 'default')}] rotate 4 outs", rotate)
