"""Achieved HBM bandwidth of the ewise kernel (Strassen operand sums and
quadrant combinations): DD/QD, 1-op and 3-op chains, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1710_01839_b200 import _cuda

_cuda.load()
n = int(os.environ.get("N", "4096"))
for comps in (2, 4):
    X, Y, Z, W = (torch.rand((n, n, comps), dtype=torch.float64, device="cuda") for _ in range(4))
    O = torch.empty_like(X)
    s = torch.cuda.current_stream().cuda_stream
    for nops in (1, 3):
        def run():
            _cuda.ewise_dev(comps, n, n, O.data_ptr(), n, X.data_ptr(), n, Y.data_ptr(), n, 1,
                            Z.data_ptr() if nops == 3 else None, n, -1,
                            W.data_ptr() if nops == 3 else None, n, 1, s)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / reps
        byts = (nops + 2) * n * n * comps * 8
        print(f"comps={comps} nops={nops} n={n}: {t*1e6:.1f} us, {byts/t/1e9:.0f} GB/s "
              f"({byts/t/6440.7e9:.2f} of 6440.7)", flush=True)
