"""The block-size predictor with its refinement of near-tied candidates, DD
8192^3 (seed 1), four repetitions: pick, predictions, what the phase cost."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix
p = mp.PrecisionSpec.dd(); n = 8192
a, b = inputs.gemm_inputs_device("dd", n, n, n, seed=1)
A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
pol = mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min")
for refine in (False, True, True, True, True):
    t0 = time.perf_counter()
    best, recs = mp.select_block_size(A, B, [16, 32, 64, 128, 256], policy=pol, refine=refine)
    wall = time.perf_counter() - t0
    print(f"refine={refine}: pick {best}; " + ", ".join(f"{r.n_min}:{r.predicted_full_s*1e3:.1f}ms(rows {r.slice_rows})" for r in recs)
          + f"; timed {sum(r.phase_time_s for r in recs):.2f} s, wall {wall:.2f} s", flush=True)
