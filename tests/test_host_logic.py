"""Host-side logic of the drop-in (no GPU): choices, validation, partition,
prediction arithmetic, timing policy, tuning tables, wave model, shards.
Mirrors the reference's unit tests (tests/test_multiply.py, test_predict.py,
test_tune.py, test_acceptance.py criteria 5 and 9)."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1710_01839_b200 as mp
from paper_1710_01839_b200 import shard
from paper_1710_01839_b200.errors import MeasurementError, ShapeError, TableFormatError
from paper_1710_01839_b200.multiply import _split_range
from paper_1710_01839_b200.predict import (WaveModel, fit_two_slices, gpu_slice_rows,
                                           predict_full_time_waves)

DD = mp.PrecisionSpec.dd()
QD = mp.PrecisionSpec.qd()


def test_algorithm_choice_tokens():
    for tok in ("simple", "block:64", "strassen:64/32", "exact", "exact/32"):
        assert mp.AlgorithmChoice.parse(tok).token == tok
    with pytest.raises(ValueError):
        mp.AlgorithmChoice.parse("winograd")
    with pytest.raises(ValueError):
        mp.AlgorithmChoice(mp.Algorithm.BLOCK)
    with pytest.raises(ValueError):
        mp.AlgorithmChoice(mp.Algorithm.STRASSEN, n_min=8, cutoff=1)


def test_precision_tokens_and_bounds():
    assert mp.PrecisionSpec.parse("dd") == DD and DD.comps == 2 and QD.comps == 4
    assert DD.gemm_bound_u == 2.0 ** -104 and QD.gemm_bound_u == 2.0 ** -209
    assert mp.PrecisionSpec.parse("ap:128").bits == 128
    with pytest.raises(ValueError):
        mp.PrecisionSpec.parse("fp128")


def test_shape_and_prec_errors():
    a = mp.DenseMatrix.zeros(3, 4, DD)
    with pytest.raises(ShapeError):
        mp.matmul_simple(a, mp.DenseMatrix.zeros(3, 4, DD))
    with pytest.raises(mp.PrecisionMismatchError):
        mp.matmul_simple(mp.DenseMatrix.zeros(3, 3, DD), mp.DenseMatrix.zeros(3, 3, QD))
    with pytest.raises(ShapeError):
        mp.matmul_strassen(a, a)
    sq = mp.DenseMatrix.zeros(4, 4, DD)
    with pytest.raises(ValueError):
        mp.matmul_strassen(sq, sq, cutoff=1)
    with pytest.raises(ValueError):
        mp.matmul_simple(sq, sq, threads=0)
    with pytest.raises(ValueError):
        mp.matmul_block(sq, sq, 0)
    with pytest.raises(ShapeError):
        mp.DenseMatrix(0, 3, DD, np.zeros((0, 3, 2)))


def test_split_range_and_partition():
    assert _split_range(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert _split_range(2, 8) == [(0, 1), (1, 2)]
    p = mp.make_partition(100, 64, 33, 32)
    assert p.row_extents == (32, 32, 32, 4) and p.inner_extents == (32, 32)
    assert p.col_extents == (32, 1) and p.n_blocks == 2


def test_leading_rows_shares_storage():
    m = mp.DenseMatrix.zeros(5, 3, DD)
    s = mp.leading_rows(m, 2)
    s.data[0, 0, 0] = 7.0
    assert m.data[0, 0, 0] == 7.0
    with pytest.raises(ShapeError):
        mp.leading_rows(m, 6)


def test_from_ints_and_identity_are_exact():
    a = mp.DenseMatrix.from_ints([[1, 2], [3, 2 ** 60 + 1]], DD)
    assert a.data[1, 1, 0] + a.data[1, 1, 1] == 2 ** 60 + 1
    assert int(a.data[1, 1, 0]) + int(a.data[1, 1, 1]) == 2 ** 60 + 1
    e = mp.DenseMatrix.identity(3, QD)
    assert e.data[:, :, 0].tolist() == np.eye(3).tolist()


# --- prediction (reference test_predict.py, acceptance criterion 5) --------

def fake_clock(deltas):
    state = {"t": 0.0, "i": 0}

    def clock():
        t = state["t"]
        state["t"] += deltas[state["i"] % len(deltas)]
        state["i"] += 1
        return t
    return clock


def test_measure_aggregators():
    for agg, want in (("median", 2.0), ("min", 1.0), ("mean", 2.0)):
        pol = mp.TimingPolicy(measured_runs=3, aggregator=agg,
                              clock=fake_clock([1.0, 0.0, 2.0, 0.0, 3.0, 0.0]))
        assert mp.measure(lambda: None, pol) == want


def test_measure_rejects_zero_and_validates():
    with pytest.raises(MeasurementError):
        mp.measure(lambda: None, mp.TimingPolicy(clock=lambda: 1.0))
    with pytest.raises(ValueError):
        mp.TimingPolicy(measured_runs=0)
    with pytest.raises(ValueError):
        mp.TimingPolicy(aggregator="max")
    calls = []
    mp.measure(lambda: None, mp.TimingPolicy(measured_runs=3, warmup_runs=1,
                                             clock=fake_clock([0.5])),
               setup=lambda: calls.append(1))
    assert len(calls) == 4


def test_slice_rows_and_published_values():
    assert mp.slice_rows_for(64, 1024) == 128
    assert mp.slice_rows_for(512, 1024) == 1024
    assert mp.slice_rows_for(64, 1024, slice_multiplier=4) == 256
    assert mp.predict_full_time(5.77, 1024, 64) == pytest.approx(46.16, abs=1e-12)
    assert mp.predict_full_time(32.5, 1024, 128) == pytest.approx(130.0, abs=1e-12)
    assert round(100 * mp.rel_diff(46.1, 45.97), 2) == 0.28
    assert round(100 * mp.rel_diff(13.8, 14.66), 2) == 5.87
    with pytest.raises(ValueError):
        mp.predict_full_time(0.0, 100, 8)
    with pytest.raises(ValueError):
        mp.slice_rows_for(0, 10)


@settings(max_examples=200, deadline=None)
@given(st.floats(min_value=1e-6, max_value=1e6), st.integers(1, 10000), st.integers(1, 4096))
def test_predict_linearity(t, m, n_min):
    if 2 * n_min <= m:
        assert mp.predict_full_time(t, 2 * m, n_min) == 2.0 * mp.predict_full_time(t, m, n_min)


def test_choose_best_tie_break():
    rec = lambda n, p: mp.PredictionRecord(n, 1, 1, p, p)  # noqa: E731
    assert mp.choose_best([rec(64, 10.0), rec(128, 9.0), rec(256, 9.0)]) == 128


def test_wave_model():
    wm = WaveModel(tile_m=64, tile_n=64, ctas_per_sm=1, sm_count=148)
    assert wm.ctas(1024, 1024) == 256 and wm.waves(1024, 1024) == 2
    assert wm.load(1024, 1024) == 2
    rows = gpu_slice_rows(wm, 64, 1024, 1024)
    assert rows % 64 == 0 and wm.ctas(rows, 1024) >= 148
    assert predict_full_time_waves(1.0, wm, rows, 1024, 1024) == \
        pytest.approx(wm.load(1024, 1024) / wm.load(rows, 1024))
    assert gpu_slice_rows(wm, 64, 100, 1024) == 100
    lpt = WaveModel(64, 64, 1, 148, balanced=True)
    assert lpt.load(1024, 1024) == pytest.approx(256 / 148)
    # two-point fit recovers alpha + beta * load exactly
    t = lambda r: 0.5 + 2.0 * wm.load(r, 4096)  # noqa: E731
    assert fit_two_slices(wm, 640, t(640), 1280, t(1280), 8192, 4096) == \
        pytest.approx(t(8192))


# --- tuning tables (reference test_tune.py, acceptance criterion 9) --------

def mk_row(prec, n, threads, strassen, best=8, t=1.0, gpus=1):
    win = (mp.AlgorithmChoice(mp.Algorithm.STRASSEN, n_min=best, cutoff=64) if strassen
           else mp.AlgorithmChoice(mp.Algorithm.BLOCK, n_min=best))
    return mp.TuningResult(prec=prec, n=n, threads=threads, best_n_min=best, block_time_s=t,
                           selection_time_s=t / 4, predicted_s=t * 1.01, rel_diff=0.01,
                           simple_time_s=t * 2, strassen_time_s=t * (0.5 if strassen else 2.0),
                           winner=win, gpus=gpus)


def test_threshold_rules():
    rows = [mk_row(DD, n, 1, s) for n, s in ((64, False), (128, True), (256, True), (512, True))]
    assert mp.extract_threshold(rows, DD, 1) == 128
    assert mp.extract_threshold([mk_row(DD, n, 1, False) for n in (64, 128)], DD, 1) is None
    assert mp.extract_threshold([mk_row(QD, n, 1, True) for n in (63, 64, 128)], QD, 1) == 63
    rows = [mk_row(DD, 64, 1, True), mk_row(DD, 64, 2, False)]
    assert mp.extract_threshold(rows, DD, 2) is None


def test_reference_fixture_round_trips_byte_for_byte(tmp_path):
    # the v1 fixture of the reference's acceptance criterion 9
    fixture = "\n".join([
        "mpmmtune v1",
        "total " + (45.97).hex(),
        "predtotal " + (5.77).hex(),
        f"dd,106 1024 1 64 {(45.97).hex()} {(5.77).hex()} {(46.1).hex()} "
        f"{(0.0028).hex()} - {(25.54).hex()} strassen:64/64",
        f"ap,128 1024 2 32 {(67.72).hex()} {(4.43).hex()} {(70.8).hex()} "
        f"{(0.0455).hex()} - {(88.15).hex()} block:32",
        "threshold dd,106 1 64",
    ]) + "\n"
    p = tmp_path / "f.tbl"
    p.write_text(fixture)
    t = mp.load_table(str(p))
    assert t.rows[0].block_time_s == 45.97 and t.rows[0].winner.kind is mp.Algorithm.STRASSEN
    assert t.thresholds[(DD, 1)] == 64
    q = tmp_path / "g.tbl"
    mp.save_table(t, str(q))
    assert q.read_text() == fixture


def test_v2_table_with_gpus(tmp_path):
    t = mp.TuningTable(rows=[mk_row(DD, 1024, 1, False, gpus=8), mk_row(QD, 512, 1, True)],
                       thresholds={(QD, 1): 512, (DD, 1, 8): 2048}, total_tuning_time_s=3.5,
                       prediction_total_s=0.25,
                       failures=[mp.TuningFailure(DD, 64, 1, "gap here", gpus=2)])
    p = tmp_path / "v2.tbl"
    mp.save_table(t, str(p))
    assert p.read_text().startswith("mpmmtune v2")
    assert mp.load_table(str(p)) == t
    assert mp.lookup_best(t, DD, 1024, 1, gpus=8) == (t.rows[0].winner, "exact")
    assert mp.lookup_best(t, DD, 4096, 1, gpus=8)[1] == "nearest"


def test_v3_table_with_exact_candidate(tmp_path):
    ex = mk_row(DD, 2048, 1, False)
    ex.exact_time_s = 0.125
    ex.winner = mp.AlgorithmChoice(mp.Algorithm.EXACT, n_min=ex.best_n_min)
    t = mp.TuningTable(rows=[mk_row(DD, 1024, 1, True), ex], thresholds={},
                       total_tuning_time_s=2.0, prediction_total_s=0.5)
    p = tmp_path / "v3.tbl"
    mp.save_table(t, str(p))
    text = p.read_text()
    assert text.startswith("mpmmtune v3") and " exact/8" in text
    assert mp.load_table(str(p)) == t
    assert mp.lookup_best(t, DD, 2048, 1) == (ex.winner, "exact")
    assert mp.lookup_best(t, DD, 4096, 1) == (ex.winner, "nearest")
    # no exact column / winner: the reference's v1 format, unchanged
    t1 = mp.TuningTable(rows=[mk_row(DD, 1024, 1, True)], thresholds={})
    mp.save_table(t1, str(p))
    assert p.read_text().startswith("mpmmtune v1")


def test_pick_winner_with_exact_candidate():
    from paper_1710_01839_b200.tune import _pick_winner
    w = _pick_winner(2.0, 3.0, None, 32, 64, exact_time=1.0)
    assert w.kind is mp.Algorithm.EXACT and w.n_min == 32
    # ties go to the reference's algorithms first
    assert _pick_winner(1.0, 1.0, 1.0, 32, 64, exact_time=1.0).kind is mp.Algorithm.BLOCK
    assert _pick_winner(2.0, 1.0, None, 32, 64, exact_time=1.0).kind is mp.Algorithm.STRASSEN
    assert _pick_winner(2.0, None, None, 32, 64).kind is mp.Algorithm.BLOCK


def test_table_errors(tmp_path):
    p = tmp_path / "bad.tbl"
    p.write_text("mpmmtune v9\n")
    with pytest.raises(TableFormatError):
        mp.load_table(str(p))
    p.write_text("")
    with pytest.raises(TableFormatError):
        mp.load_table(str(p))
    p.write_text("mpmmtune v1\ndd,106 1 2 3\n")
    with pytest.raises(TableFormatError):
        mp.load_table(str(p))


def test_lookup_fallbacks():
    t = mp.TuningTable(rows=[mk_row(DD, 128, 1, True)], thresholds={(DD, 1): 128})
    assert mp.lookup_best(t, DD, 128, 1)[1] == "exact"
    assert mp.lookup_best(t, DD, 200, 1)[1] == "nearest"
    assert mp.lookup_best(t, DD, 64, 1)[1] == "default"
    t2 = mp.TuningTable(rows=[], thresholds={(DD, 1): 128})
    assert mp.lookup_best(t2, DD, 256, 1)[1] == "threshold"


def test_tuning_config_validation():
    with pytest.raises(ValueError):
        mp.TuningConfig(precisions=[DD], dims=[], block_candidates=[4], thread_counts=[1])
    with pytest.raises(ValueError):
        mp.TuningConfig(precisions=[DD], dims=[1, 16], block_candidates=[4], thread_counts=[1])
    cfg = mp.TuningConfig(precisions=[DD], dims=[16], block_candidates=[8, 4], thread_counts=[1])
    assert cfg.block_candidates == [4, 8]


def test_tune_sweep_records_failures(monkeypatch):
    import paper_1710_01839_b200.tune as tune_mod

    def flaky(prec, n, threads, cfg, _accum=None, gpus=1):
        if n == 24:
            raise RuntimeError("injected fault")
        return mk_row(prec, n, threads, False)

    monkeypatch.setattr(tune_mod, "tune_one", flaky)
    monkeypatch.setattr(tune_mod, "_device_pair",
                        lambda n, prec: (mp.DenseMatrix.zeros(n, n, prec),) * 2)
    monkeypatch.setattr(tune_mod, "_block_into", lambda *a, **k: None)
    cfg = mp.TuningConfig(precisions=[DD], dims=[16, 24], block_candidates=[4, 8],
                          thread_counts=[1])
    table = mp.tune_sweep(cfg)
    assert len(table.rows) == 1 and len(table.failures) == 1
    assert "injected" in table.failures[0].message


def test_tune_sweep_over_gpu_counts(monkeypatch, tmp_path):
    """gpu_counts is swept like thread_counts (reference tune.py:173-213):
    one row per (prec, n, threads, gpus), thresholds per gpus series, and
    the modelled rows survive a save/load round trip as "G~"."""
    import paper_1710_01839_b200.tune as tune_mod
    seen = []

    def fake(prec, n, threads, cfg, _accum=None, gpus=1):
        seen.append((n, gpus))
        _accum["selection"] = _accum.get("selection", 0.0) + 0.5
        r = mk_row(prec, n, threads, n >= 32 and gpus == 1)
        r.gpus, r.gpus_modelled = gpus, gpus > 1
        return r

    monkeypatch.setattr(tune_mod, "tune_one", fake)
    monkeypatch.setattr(tune_mod, "_warm", lambda *a: None)
    cfg = mp.TuningConfig(precisions=[DD], dims=[16, 32, 64], block_candidates=[8],
                          thread_counts=[1], gpu_counts=[8, 1, 2],
                          out_path=str(tmp_path / "g.tbl"))
    table = mp.tune_sweep(cfg)
    assert seen == [(n, g) for n in (16, 32, 64) for g in (1, 2, 8)]
    assert table.prediction_total_s == 0.5 * 9
    assert table.thresholds == {(DD, 1): 32}
    text = open(tmp_path / "g.tbl").read()
    assert text.startswith("mpmmtune v2") and " 8~ " in text and " 1 " in text
    back = mp.load_table(str(tmp_path / "g.tbl"))
    assert sorted((r.n, r.gpus, r.gpus_modelled) for r in back.rows) == \
        sorted((n, g, g > 1) for n in (16, 32, 64) for g in (1, 2, 8))
    with pytest.raises(ValueError):
        mp.TuningConfig(precisions=[DD], dims=[16], block_candidates=[8], thread_counts=[1],
                        gpu_counts=[0])


def test_shard_model_geometry():
    """The G-GPU point tunes the largest row block's product; the exposed
    broadcast is one k-panel (blocked/simple) or all of B (Strassen)."""
    from paper_1710_01839_b200.tune import _Shard
    cfg = mp.TuningConfig(precisions=[DD], dims=[16], block_candidates=[8], thread_counts=[1],
                          bcast_bytes_per_s=1e9, bcast_panels=8)
    s1 = _Shard(8192, 1, 2, cfg)
    assert s1.rows == 8192 and s1.full_s == 0.0 and s1.panel_s == 0.0
    s3 = _Shard(8192, 3, 2, cfg)
    assert s3.rows == 2752                       # ceil(8192/3) -> 64-row multiple
    assert s3.full_s == 16.0 * 8192 * 8192 / 1e9 and s3.panel_s == s3.full_s / 8


# --- sharding -----------------------------------------------------------------

def test_row_shards_cover_exactly():
    for m, world, align in ((1024, 8, 64), (1000, 3, 16), (5, 8, 1), (0, 2, 1)):
        parts = shard.row_shards(m, world, align)
        assert len(parts) == world
        covered = [i for lo, hi in parts for i in range(lo, hi)]
        assert covered == list(range(m))
        for lo, hi in parts:
            assert lo % align == 0 or lo == m
    assert shard.panel_bounds(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert shard.panel_bounds(10, None) == [(0, 10)]


# --- tensor mode host tables ----------------------------------------------------

def test_tensor_moduli_and_crt_tables():
    import math
    import random
    from paper_1710_01839_b200 import tensor
    mods = tensor.MODULI
    assert len(mods) == 54 and all(math.gcd(a, b) == 1 for i, a in enumerate(mods)
                                   for b in mods[:i])
    assert all(p <= 256 for p in mods)
    assert tensor.moduli_count(300) is not None and tensor.moduli_count(400) is None
    N = tensor.moduli_count(250)
    words, K = tensor.crt_table(N)
    limbs = lambda q: sum(int(words[q * K + t]) << (32 * t) for t in range(K))  # noqa: E731
    P, W = limbs(0), [limbs(1 + t) for t in range(N)]
    assert P == math.prod(mods[:N]) and P > 1 << 250
    rng = random.Random(1)
    for _ in range(20):
        x = rng.randrange(-(P // 2), P // 2)
        r = [x % p for p in mods[:N]]
        X = sum(ri * wi for ri, wi in zip(r, W)) % P
        assert (X if X <= P // 2 else X - P) == x
    padded, K2 = tensor.crt_table(N, K + 2)
    assert K2 == K + 2 and int(padded[K2 * 1 + K]) == 0



def test_native_tensor_planner():
    """mpmm_oz_plan (host-only C++): feasibility, cost choice and shifts."""
    from paper_1710_01839_b200 import _cuda, tensor
    E_, L_ = tensor.EMPTY_E, tensor.EMPTY_L
    # DD, 3 rows: hi spans [2^-52, 2^0), lo down to 2^-105; row 2 empty
    ea = np.array([0, -3, E_, -53, -60, E_, -52, -10, L_, -105, -70, L_], dtype=np.int32)
    eb = ea.copy()
    jobs, ra, sa, rb, sb = _cuda.oz_plan(2, 3, 3, 64, ea, eb)
    assert len(jobs) == 1 and tuple(ra[0]) == (0, 2)
    beta = (0 + 105) + 1 + 1
    N, K, wa, wb, ba, bb = jobs[0][2:]
    assert (ba, bb) == (beta, beta) and wa == wb == (beta + 33) // 32
    assert N == tensor.moduli_count(2 * beta + 6 + 1) and K == tensor.crt_limbs(N)
    assert list(sa[0]) == [105, 70, 0]
    # a wide row: the 1-job plan no longer fits 54 moduli -> a split
    ea2 = ea.copy()
    ea2[9] = -250
    jobs, ra, sa, rb, sb = _cuda.oz_plan(2, 3, 3, 64, ea2, eb)
    assert len(jobs) > 1
    cover = sorted((x, y) for j in jobs for x in range(*ra[j[0]]) for y in range(*rb[j[1]]))
    assert cover == [(0, 0), (0, 1), (1, 0), (1, 1)]
    # hopeless: a single component spanning 2^400
    ea3 = ea.copy()
    ea3[6] = -400
    assert _cuda.oz_plan(2, 3, 3, 64, ea3, eb) is None


def test_matrix_dump_round_trip_and_reference_format():
    """write_matrix / read_matrix (reference matrix.py:318-354): exact hex
    components, one row per line; malformed dumps raise TableFormatError."""
    import io
    from paper_1710_01839_b200 import inputs
    for tok in ("dd", "qd"):
        a, _ = inputs.gemm_inputs(tok, 3, 4, 2, seed=9)
        m = mp.DenseMatrix(3, 4, mp.PrecisionSpec.parse(tok), a)
        buf = io.StringIO()
        mp.write_matrix(m, buf)
        text = buf.getvalue()
        assert text.splitlines()[0] == f"3 4 {tok}"
        assert text.splitlines()[1].split()[0] == ",".join(x.hex() for x in a[0, 0])
        assert mp.read_matrix(io.StringIO(text)) == m
    for bad in ("3 4\n", "1 2 dd\n0x1p+0,0x0p+0\n", "1 1 dd\n0x1p+0\n", "x y dd\n"):
        with pytest.raises(TableFormatError):
            mp.read_matrix(io.StringIO(bad))


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_scalar_algebra_matches_the_reference(tok):
    """Scalar and scalar_* (reference scalar.py:95-251 over ddqd.py): add,
    sub, mul, div, sqrt and the literal constructors, bit for bit against
    outputs of the reference itself (tests/golden/scalar_ops.npz)."""
    from conftest import golden
    g = golden("scalar_ops")
    prec = mp.PrecisionSpec.parse(tok)
    xs = [mp.Scalar(prec, r) for r in g[f"{tok}_x"]]
    ys = [mp.Scalar(prec, r) for r in g[f"{tok}_y"]]
    ops = {"add": lambda x, y: x + y, "sub": mp.scalar_sub, "mul": lambda x, y: x * y,
           "div": lambda x, y: x / y}
    for name, fn in ops.items():
        got = np.array([fn(x, y).payload for x, y in zip(xs, ys)])
        assert np.array_equal(got, g[f"{tok}_{name}"]), name
    got = np.array([mp.scalar_sqrt(x if x.payload[0] >= 0 else -x).payload for x in xs])
    assert np.array_equal(got, g[f"{tok}_sqrt"])
    lits = [mp.Scalar.from_str("0.1", prec), mp.Scalar.from_str(
        "-3.14159265358979323846264338327950288", prec),
        mp.Scalar.from_int(2 ** 60 + 1, prec), mp.Scalar.from_int(-(3 ** 70), prec)]
    assert np.array_equal(np.array([s.payload for s in lits]), g[f"{tok}_lits"])
    z = mp.Scalar.zero(prec)
    assert z.is_zero() and (xs[0] - xs[0]).is_zero() and -(-xs[1]) == xs[1]
    with pytest.raises(ZeroDivisionError):
        xs[0] / z
    with pytest.raises(mp.PrecisionMismatchError):
        mp.Scalar.zero(mp.PrecisionSpec.dd()) + mp.Scalar.zero(mp.PrecisionSpec.qd())
    m = mp.DenseMatrix(1, 2, prec, np.stack([g[f"{tok}_x"][:2]]))
    assert m.get(0, 1) == xs[1]
