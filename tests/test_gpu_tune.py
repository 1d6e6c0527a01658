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


@pytest.mark.parametrize("tok,n", [("dd", 4096), ("qd", 2048)])
def test_acceptance_criteria_6_7_on_the_gpu(gpu, tok, n):
    """The reference's acceptance criteria 6 and 7 (test_acceptance.py:
    141-182) for the GPU predictor, at configs[4] sizes where the slices
    are a fraction of the product: every candidate's prediction within
    15 % of its measured time, the chosen candidate within 10 % of the
    fastest measured one, and the prediction phase (both slices of every
    candidate) at most 0.7 x the exhaustive search."""
    from paper_1710_01839_b200.tune import _measure_block
    p = mp.PrecisionSpec.parse(tok)
    a, b = inputs.gemm_inputs_device(tok, n, n, n, seed=1)
    A, B = DenseMatrix(n, n, p, a), DenseMatrix(n, n, p, b)
    pol = mp.TimingPolicy(warmup_runs=1, measured_runs=3, aggregator="min")
    cands = [16, 32, 64, 128, 256]
    best, recs = mp.select_block_size(A, B, cands, policy=pol)
    full = {c: _measure_block(A, B, c, 1, pol) for c in cands}
    phase = sum(r.phase_time_s for r in recs)
    for r in recs:
        err = mp.rel_diff(r.predicted_full_s, full[r.n_min])
        print(f"{tok} n={n} n_min={r.n_min} predicted={r.predicted_full_s * 1e3:.2f} ms "
              f"measured={full[r.n_min] * 1e3:.2f} ms err={err:.2%}")
        assert err <= 0.15, (r.n_min, err)
    assert full[best] <= 1.10 * min(full.values()), (best, full)
    assert phase <= 0.7 * sum(full.values()), (phase, sum(full.values()))


def test_tune_over_gpu_counts(gpu, tmp_path):
    """gpus > 1 points: the largest row block's product measured on this
    GPU plus the modelled broadcast; more GPUs -> a smaller block time."""
    cfg = mp.TuningConfig(precisions=[DD], dims=[512], block_candidates=[32, 64],
                          thread_counts=[1], strassen_cutoffs=[128], gpu_counts=[1, 2, 8],
                          inputs="seeded", out_path=str(tmp_path / "g.tbl"))
    table = mp.tune_sweep(cfg)
    rows = {r.gpus: r for r in table.rows}
    assert sorted(rows) == [1, 2, 8] and not table.failures
    assert not rows[1].gpus_modelled and rows[2].gpus_modelled and rows[8].gpus_modelled
    assert rows[8].block_time_s < rows[2].block_time_s < rows[1].block_time_s
    assert open(cfg.out_path).read().startswith("mpmmtune v2")
    assert mp.load_table(cfg.out_path) == table


def test_gpus_argument(gpu):
    """gpus= on the public API: Strassen's seven top-level products spread
    over a device list (the same device twice here) give the one-GPU bits;
    row sharding needs distinct devices."""
    a, b = inputs.gemm_inputs("dd", 300, 300, 300, seed=6)
    A = DenseMatrix(300, 300, DD, a).to_device()
    B = DenseMatrix(300, 300, DD, b).to_device()
    one = mp.matmul_strassen(A, B, 64, 32)
    st1, st2 = mp.StrassenStats(), mp.StrassenStats()
    assert mp.matmul_strassen(A, B, 64, 32, stats=st1) == one
    two = mp.matmul_strassen(A, B, 64, 32, gpus=[0, 0], stats=st2)
    assert two == one and two.is_device
    assert (st1.multiplications, st1.additions) == (st2.multiplications, st2.additions)
    assert np.array_equal(one.host_array(), oracle.strassen(a, b, 64, 32))
    choice = mp.AlgorithmChoice.parse("strassen:64/32")
    assert mp.run_choice(A, B, choice, gpus=[0, 0]) == one
    with pytest.raises(ValueError):
        mp.matmul_block(A, B, 32, gpus=[0, 0])
    with pytest.raises(ValueError):
        mp.matmul_block(A, B, 32, gpus=0)
    assert mp.matmul_block(A, B, 32, gpus=1) == mp.matmul_block(A, B, 32)
