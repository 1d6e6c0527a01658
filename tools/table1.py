#!/usr/bin/env python3
"""The paper's Table 1 on one B200 (PAPER.md:105-142 columns (a)-(e)).

Runs the tuner (tune_sweep: wave-aware prediction, blocked, simple up to
simple_limit, Strassen over a cutoff list) on the paper's own test pair
(generate_test_pair, matrix.py:168-200) and prints, per precision and n:
(a) chosen n_min, (b) blocked time, (c) prediction-phase slice time of
the chosen candidate, (d) predicted time, rel.diff, (e) Strassen time,
plus the winner.  Saves the mpmmtune table next to the JSON summary.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1710_01839_b200 as mp  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--prec", default="dd,qd")
    p.add_argument("--dims", default="512,1024,2048")
    p.add_argument("--nmin", default="16,32,64,128,256")
    p.add_argument("--cutoffs", default="256,512,1024")
    p.add_argument("--out", default="gpurun_out/table1")
    a = p.parse_args()
    cfg = mp.TuningConfig(
        precisions=[mp.PrecisionSpec.parse(t) for t in a.prec.split(",")],
        dims=[int(x) for x in a.dims.split(",")],
        block_candidates=[int(x) for x in a.nmin.split(",")],
        thread_counts=[1], strassen_cutoffs=[int(x) for x in a.cutoffs.split(",")],
        timing=mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min"),
        out_path=a.out + ".tbl")
    table = mp.tune_sweep(cfg)
    rows = []
    print(f"{'prec':>4} {'n':>5} {'(a)':>5} {'(b) block s':>12} {'(c) slice s':>12} "
          f"{'(d) pred s':>11} {'rel':>7} {'simple s':>10} {'(e) strassen s':>14}  winner")
    for r in table.rows:
        print(f"{r.prec.token:>4} {r.n:>5} {r.best_n_min:>5} {r.block_time_s:>12.5f} "
              f"{r.selection_time_s:>12.5f} {r.predicted_s:>11.5f} {r.rel_diff:>7.2%} "
              f"{(r.simple_time_s or float('nan')):>10.5f} {r.strassen_time_s:>14.5f}  "
              f"{r.winner.token}")
        rows.append({"prec": r.prec.token, "n": r.n, "a_n_min": r.best_n_min,
                     "b_block_s": r.block_time_s, "c_slice_s": r.selection_time_s,
                     "d_predicted_s": r.predicted_s, "rel_diff": r.rel_diff,
                     "simple_s": r.simple_time_s, "e_strassen_s": r.strassen_time_s,
                     "winner": r.winner.token,
                     "block_2mnl_per_s": 2.0 * r.n ** 3 / r.block_time_s,
                     "strassen_eff_2mnl_per_s": 2.0 * r.n ** 3 / r.strassen_time_s})
    for f in table.failures:
        print("FAILED", f)
    summary = {"rows": rows, "thresholds": {f"{k[0].token}/threads={k[1]}": v
                                            for k, v in table.thresholds.items()},
               "total_tuning_s": table.total_tuning_time_s,
               "prediction_phase_s": table.prediction_total_s,
               "failures": [vars(f) | {"prec": f.prec.token} for f in table.failures]}
    with open(a.out + ".json", "w") as fp:
        json.dump(summary, fp, indent=1)


if __name__ == "__main__":
    main()
