"""End-to-end host product at DD 8192^3 (and 4096^3): the streamed
single-launch path with k-panel streaming (MPMM_STREAM_TILE_MB=-1) vs
tile-order streaming (A row panels, B column panels; the default from
128 MiB of operands), against the device-resident kernel time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import _cuda, inputs
from paper_1710_01839_b200.matrix import DenseMatrix

for n in (int(x) for x in os.environ.get("SIZES", "4096,8192").split(",")):
    prec = mp.PrecisionSpec.dd()
    a, b = inputs.gemm_inputs_device("dd", n, n, n, seed=1)
    C = torch.empty_like(a)
    s = torch.cuda.current_stream().cuda_stream
    run = lambda: _cuda.gemm_dev(2, _cuda.ALGO_BLOCK, 32, n, n, n, a.data_ptr(), n, b.data_ptr(),
                                 n, C.data_ptr(), n, False, None, s)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); e1.synchronize()
    dev = e0.elapsed_time(e1) / 1e3
    ha, hb = a.cpu().pin_memory().numpy(), b.cpu().pin_memory().numpy()
    want = C.cpu().numpy()
    A, B = DenseMatrix(n, n, prec, ha), DenseMatrix(n, n, prec, hb)
    for mode in ("-1", "128"):
        os.environ["MPMM_STREAM_TILE_MB"] = mode
        c = mp.matmul_block(A, B, 32)
        c = mp.matmul_block(A, B, 32)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            c = mp.matmul_block(A, B, 32)
            ts.append(time.perf_counter() - t0)
        same = np.array_equal(c.data, want)
        print(f"n={n} mode={'k-panels' if mode == '-1' else 'tile order'}: e2e {min(ts)*1e3:.1f} ms "
              f"(device {dev*1e3:.1f} ms, overhead {(min(ts)-dev)*1e3:.1f} ms), bitwise "
              f"{'equal' if same else 'DIFFERENT'}", flush=True)
    del a, b, C, ha, hb, A, B, c
    torch.cuda.empty_cache()
