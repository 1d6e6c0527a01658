"""Blocked QD kernel time per block size (events, L2 flushed), with a hash
of the 512^3 result (variants must agree bit for bit)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1710_01839_b200 import _cuda, inputs

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
lib = os.path.basename(os.environ.get("MPMM_LIB_PATH", "default"))
for n, reps in ((512, 5), (1024, 5), (2048, 2)):
    a, b = inputs.gemm_inputs_device("qd", n, n, n, seed=1)
    c = torch.empty_like(a)
    s = torch.cuda.current_stream().cuda_stream
    for nm in (16, 32, 64, 128, 256):
        run = lambda: _cuda.gemm_dev(4, _cuda.ALGO_BLOCK, nm, n, n, n, a.data_ptr(), n,
                                     b.data_ptr(), n, c.data_ptr(), n, False, None, s)
        run(); torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(); e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        t = min(x.elapsed_time(y) for x, y in ts)
        frac = 796 * n ** 3 / (t / 1e3) / 1e12 / 37.22496
        h = hashlib.sha1(c.cpu().numpy().tobytes()).hexdigest()[:12] if n == 512 else ""
        print(f"{lib}: qd n={n} n_min={nm} {t:.3f} ms frac {frac:.4f} {h}", flush=True)
