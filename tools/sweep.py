#!/usr/bin/env python3
"""Per-config measurements for BASELINE.json configs 0-4 on one B200.

For every config: device time (CUDA events, min of N after warm-up),
2mnl/s, fraction of the FP64 roofline, and for the blocked sweeps the
wave-aware predicted time next to the measured one (paper Table 1 columns
(a)-(e)).  Writes one JSON document (default gpurun_out/sweep.json).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1710_01839_b200 as mp  # noqa: E402
from paper_1710_01839_b200 import _cuda, inputs  # noqa: E402
from paper_1710_01839_b200.matrix import DenseMatrix  # noqa: E402
from paper_1710_01839_b200.predict import select_block_size  # noqa: E402

F = {"dd": 53, "qd": 796}


def ev_time(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def gemm_fn(tok, algo, n_min, A, B, C):
    comps = 2 if tok == "dd" else 4
    m, l, n = A.shape[0], A.shape[1], B.shape[1]
    s = torch.cuda.current_stream().cuda_stream
    return lambda: _cuda.gemm_dev(comps, algo, n_min, m, l, n, A.data_ptr(), l, B.data_ptr(),
                                  n, C.data_ptr(), n, False, None, s)


def rec(tok, m, l, n, t, peak, **kw):
    madds = float(m) * l * n
    d = {"prec": tok, "m": m, "l": l, "n": n, "seconds": t, "2mnl_per_s": 2 * madds / t,
         "fp64_tflops": F[tok] * madds / t / 1e12, "roofline_frac": F[tok] * madds / t / 1e12 / peak}
    d.update(kw)
    print(json.dumps(d), flush=True)
    return d


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default="gpurun_out/sweep.json")
    p.add_argument("--max-n", type=int, default=8192)
    p.add_argument("--qd-max-n", type=int, default=4096)
    p.add_argument("--only", default="0,1,2,3,4")
    a = p.parse_args()
    only = set(a.only.split(","))
    dev = torch.device("cuda", 0)
    # FP64 peak
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    scratch = torch.zeros(4096, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    iters = 20000
    t = ev_time(lambda: _cuda.fp64_burn_dev(0, sms * 8, 256, iters, scratch.data_ptr(), s))
    peak = sms * 8 * 256 * 8 * iters * 2 / t / 1e12
    out = {"device": torch.cuda.get_device_name(0), "sms": sms, "fp64_peak_tflops": peak,
           "records": []}
    R = out["records"]
    DD, QD = mp.PrecisionSpec.dd(), mp.PrecisionSpec.qd()

    if "0" in only:  # cfg0 DD simple 128^3
        x, y = inputs.gemm_inputs("dd", 128, 128, 128, seed=0)
        A, B = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        C = torch.empty_like(A)
        for algo, name in ((_cuda.ALGO_SIMPLE, "simple"), (_cuda.ALGO_BLOCK, "block:16")):
            R.append(rec("dd", 128, 128, 128, ev_time(gemm_fn("dd", algo, 16, A, B, C), 10),
                         peak, config=0, algo=name))

    if "1" in only or "2" in only:  # cfg1 DD 1024 sweep x2 input sets; cfg2 QD 1024
        sets = []
        if "1" in only:
            sets += [("dd", False), ("dd", True)]
        if "2" in only:
            sets += [("qd", False)]
        for tok, wide in sets:
            x, y = inputs.gemm_inputs(tok, 1024, 1024, 1024, seed=0, wide=wide)
            prec = DD if tok == "dd" else QD
            Am = DenseMatrix(1024, 1024, prec, x).to_device()
            Bm = DenseMatrix(1024, 1024, prec, y).to_device()
            C = torch.empty_like(Am.data)
            pol = mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min")
            t0 = time.perf_counter()
            best, recs = select_block_size(Am, Bm, [16, 32, 64, 128, 256], policy=pol)
            pred_phase = time.perf_counter() - t0
            for r in recs:
                t = ev_time(gemm_fn(tok, _cuda.ALGO_BLOCK, r.n_min, Am.data, Bm.data, C))
                R.append(rec(tok, 1024, 1024, 1024, t, peak, config=1 if tok == "dd" else 2,
                             algo=f"block:{r.n_min}", wide=wide, slice_rows=r.slice_rows,
                             slice_s=r.slice_time_s, predicted_s=r.predicted_full_s,
                             rel_diff=mp.rel_diff(r.predicted_full_s, t),
                             chosen=(r.n_min == best), prediction_phase_wall_s=pred_phase))
            t = ev_time(gemm_fn(tok, _cuda.ALGO_SIMPLE, 0, Am.data, Bm.data, C), 2)
            R.append(rec(tok, 1024, 1024, 1024, t, peak, config=1 if tok == "dd" else 2,
                         algo="simple", wide=wide))

    if "3" in only:  # cfg3 DD Strassen 2048^3 + rectangular
        for (m, l, n) in ((2048, 2048, 2048), (2048, 1024, 4096)):
            x, y = inputs.gemm_inputs("dd", m, l, n, seed=0)
            Am = DenseMatrix(m, l, DD, x).to_device()
            Bm = DenseMatrix(l, n, DD, y).to_device()
            C = torch.empty((m, n, 2), dtype=torch.float64, device=dev)
            t = ev_time(gemm_fn("dd", _cuda.ALGO_BLOCK, 64, Am.data, Bm.data, C))
            R.append(rec("dd", m, l, n, t, peak, config=3, algo="block:64"))
            for cut in (128, 256, 512):
                fn = lambda: mp.matmul_strassen(Am, Bm, cut, 64, rectangular=(m != n or m != l))  # noqa
                t = ev_time(fn, 2)
                R.append(rec("dd", m, l, n, t, peak, config=3, algo=f"strassen:{cut}/64",
                             note="effective 2mnl/s; flops use the classical count"))

    if "4" in only:  # cfg4 sizes, blocked + best strassen, seed 1
        for tok in ("dd", "qd"):
            prec = DD if tok == "dd" else QD
            for n in (512, 1024, 2048, 4096, 8192):
                if n > (a.max_n if tok == "dd" else a.qd_max_n):
                    continue
                x, y = inputs.gemm_inputs(tok, n, n, n, seed=1)
                Am = DenseMatrix(n, n, prec, x).to_device()
                Bm = DenseMatrix(n, n, prec, y).to_device()
                C = torch.empty_like(Am.data)
                reps = 1 if n >= 4096 else 3
                t = ev_time(gemm_fn(tok, _cuda.ALGO_BLOCK, 64, Am.data, Bm.data, C), reps)
                R.append(rec(tok, n, n, n, t, peak, config=4, algo="block:64"))
                if n >= 1024:
                    cut = n // 4 if tok == "dd" else n // 2
                    t = ev_time(lambda: mp.matmul_strassen(Am, Bm, cut, 64), reps)
                    R.append(rec(tok, n, n, n, t, peak, config=4, algo=f"strassen:{cut}/64"))
                del Am, Bm, C
                torch.cuda.empty_cache()

    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fp:
        json.dump(out, fp, indent=1)


if __name__ == "__main__":
    main()
