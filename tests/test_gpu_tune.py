"""Predictor and tuner on the GPU (reference test_predict.py, test_tune.py,
acceptance criteria 6/7 as soft reports)."""

import numpy as np
import pytest

import oracle
import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import inputs
from paper_1710_01839_b200.matrix import DenseMatrix

pytestmark = pytest.mark.gpu

DD = mp.PrecisionSpec.dd()


def test_select_block_size_on_device(gpu):
    a, b = mp.generate_test_pair(256, DD)
    A, B = a.to_device(), b.to_device()
    best, records = mp.select_block_size(A, B, [16, 32, 64], policy=mp.TimingPolicy())
    assert [r.n_min for r in records] == [16, 32, 64] and best in (16, 32, 64)
    for r in records:
        assert r.slice_time_s > 0 and r.slice_rows <= A.rows and r.predicted_full_s > 0


def test_time_slice_and_reference_mode(gpu):
    a, b = mp.generate_test_pair(32, DD)
    elapsed, rows = mp.time_slice(a, b, n_min=4, policy=mp.TimingPolicy())
    assert rows == 8 and elapsed > 0
    best, recs = mp.select_block_size(a, b, [8, 16], policy=mp.TimingPolicy(),
                                      wave_aware=False)
    for r in recs:
        assert r.predicted_full_s == r.slice_time_s * r.scale_factor


def test_prediction_accuracy_report(gpu):
    """Wave-aware prediction vs measured full runs at 1024 (soft: report)."""
    a, b = inputs.gemm_inputs("dd", 1024, 1024, 1024, seed=1)
    A = DenseMatrix(1024, 1024, DD, a).to_device()
    B = DenseMatrix(1024, 1024, DD, b).to_device()
    pol = mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min")
    best, recs = mp.select_block_size(A, B, [16, 32, 64, 128, 256], policy=pol)
    from paper_1710_01839_b200.tune import _measure_block
    for r in recs:
        full = _measure_block(A, B, r.n_min, 1, pol)
        print(f"n_min={r.n_min} slice_rows={r.slice_rows} slice={r.slice_time_s*1e3:.3f}ms "
              f"pred={r.predicted_full_s*1e3:.3f}ms full={full*1e3:.3f}ms "
              f"rel={mp.rel_diff(r.predicted_full_s, full):.1%}")
        assert full > 0


def test_tune_one_and_sweep(gpu, tmp_path):
    cfg = mp.TuningConfig(precisions=[DD, mp.PrecisionSpec.qd()], dims=[16, 24],
                          block_candidates=[4, 8], thread_counts=[1], strassen_cutoff=8,
                          out_path=str(tmp_path / "t.tbl"))
    r = mp.tune_one(DD, 16, 1, cfg)
    assert r.best_n_min in (4, 8)
    assert r.rel_diff == mp.rel_diff(r.predicted_s, r.block_time_s)
    times = {mp.Algorithm.BLOCK: r.block_time_s, mp.Algorithm.STRASSEN: r.strassen_time_s,
             mp.Algorithm.SIMPLE: r.simple_time_s}
    assert times[r.winner.kind] == min(times.values())
    table = mp.tune_sweep(cfg)
    assert len(table.rows) == 4 and not table.failures
    assert mp.load_table(str(tmp_path / "t.tbl")) == table


def test_tune_one_tie_breaks_to_block(gpu):
    state = {"t": 0.0}

    def clock():
        state["t"] += 1.0
        return state["t"]
    cfg = mp.TuningConfig(precisions=[DD], dims=[16], block_candidates=[4, 8],
                          thread_counts=[1], strassen_cutoff=8,
                          timing=mp.TimingPolicy(clock=clock), predict=False)
    r = mp.tune_one(DD, 16, 1, cfg)
    assert r.block_time_s == r.strassen_time_s == r.simple_time_s
    assert r.winner.kind is mp.Algorithm.BLOCK


def test_strassen_cutoff_sweep_cfg3_rectangular(gpu):
    """BASELINE config 3 rectangular case (scaled to keep the oracle check
    fast): rectangular Strassen vs blocked within the normwise bound."""
    a, b = inputs.gemm_inputs("dd", 256, 128, 512, seed=0)
    A = DenseMatrix(256, 128, DD, a).to_device()
    B = DenseMatrix(128, 512, DD, b).to_device()
    ref = mp.matmul_block(A, B, 64)
    for cut in (16, 32, 64):
        got = mp.matmul_strassen(A, B, cut, 32, rectangular=True)
        assert mp.frobenius_rel_diff(got, ref) <= 100.0 * 512 * 2.0 ** -106
    # square inputs: rectangular mode is the reference algorithm bit for bit
    s, t = inputs.gemm_inputs("dd", 96, 96, 96, seed=2)
    S, T = DenseMatrix(96, 96, DD, s), DenseMatrix(96, 96, DD, t)
    assert mp.matmul_strassen(S, T, 16, 8, rectangular=True) == mp.matmul_strassen(S, T, 16, 8)
    assert np.array_equal(mp.matmul_strassen(S, T, 16, 8).data, oracle.strassen(s, t, 16, 8))


def test_tune_one_with_exact_candidate_and_run_choice(gpu, tmp_path):
    """The opt-in exact tensor-core candidate: timed, ranked last on ties,
    written as a v3 table; run_choice on its token returns the exact mode's
    product (the exact product rounded once, within the north_star bound)."""
    from paper_1710_01839_b200.tensor import matmul_exact
    cfg = mp.TuningConfig(precisions=[DD], dims=[512], block_candidates=[32, 64],
                          thread_counts=[1], strassen_cutoff=128, exact=True,
                          out_path=str(tmp_path / "t3.tbl"))
    r = mp.tune_one(DD, 512, 1, cfg)
    assert r.exact_time_s is not None and r.exact_time_s > 0
    times = {mp.Algorithm.BLOCK: r.block_time_s, mp.Algorithm.STRASSEN: r.strassen_time_s,
             mp.Algorithm.SIMPLE: r.simple_time_s, mp.Algorithm.EXACT: r.exact_time_s}
    assert times[r.winner.kind] == min(times.values())
    table = mp.tune_sweep(cfg)
    assert open(cfg.out_path).read().startswith("mpmmtune v3")
    assert mp.load_table(cfg.out_path) == table
    a, b = inputs.gemm_inputs("dd", 96, 80, 72, seed=3)
    A = DenseMatrix(96, 80, DD, a).to_device()
    B = DenseMatrix(80, 72, DD, b).to_device()
    c = mp.run_choice(A, B, mp.AlgorithmChoice.parse("exact/32")).host_array()
    assert np.array_equal(c, matmul_exact(A, B).host_array())
    from oracle import exact
    ratio, _ = exact.bound_ratio(a, b, c, range(0, 96, 7), range(0, 72, 5), 104)
    assert ratio <= 1.0
