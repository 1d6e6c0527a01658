"""Device time of the blocked DD kernel (n_min 32) at 8192^3 and 1024^3 for
the library in MPMM_LIB_PATH (tile-raster group variants)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1710_01839_b200 import _cuda, inputs

for n, reps in ((1024, 20), (8192, 2)):
    a, b = inputs.gemm_inputs_device("dd", n, n, n, seed=1)
    c = torch.empty_like(a)
    s = torch.cuda.current_stream().cuda_stream
    run = lambda: _cuda.gemm_dev(2, _cuda.ALGO_BLOCK, 32, n, n, n, a.data_ptr(), n, b.data_ptr(),
                                 n, c.data_ptr(), n, False, None, s)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record(); e1.synchronize()
    print(f"{os.environ.get('MPMM_LIB_PATH', 'default (group 16)')}: n={n} "
          f"{e0.elapsed_time(e1) / reps:.3f} ms", flush=True)
