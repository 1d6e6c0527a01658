"""CLI (reference tests/test_cli.py): report formats, usage/lock exit codes
on CPU; tune/verify/predict end to end on the GPU."""

import csv
import io
import os
import tempfile

import pytest

import paper_1710_01839_b200 as mp
from paper_1710_01839_b200.cli import (EX_IO, EX_MEASURE, EX_OK, EX_USAGE, EX_VERIFY, LOCK_NAME,
                                       main)

DD = mp.PrecisionSpec.dd()
QD = mp.PrecisionSpec.qd()


def _row(prec, n, threads, strassen, gpus=1):
    win = (mp.AlgorithmChoice(mp.Algorithm.STRASSEN, n_min=32, cutoff=256) if strassen
           else mp.AlgorithmChoice(mp.Algorithm.BLOCK, n_min=32))
    return mp.TuningResult(prec, n, threads, 32, 1.0, 0.25, 1.01, 0.01, None,
                           0.5 if strassen else 2.0, win, gpus)


def _table(tmp_path, rows):
    t = mp.TuningTable(rows=rows, thresholds={})
    p = tmp_path / "t.tbl"
    mp.save_table(t, str(p))
    return str(p)


def test_report_csv_and_winners(tmp_path, capsys):
    path = _table(tmp_path, [_row(DD, 1024, 1, False), _row(QD, 1024, 1, True),
                             _row(DD, 2048, 1, True), _row(DD, 2048, 1, True, gpus=8)])
    assert main(["report", "--in", path, "--format", "csv"]) == EX_OK
    text = capsys.readouterr().out
    rows = list(csv.DictReader(io.StringIO("".join(
        ln + "\n" for ln in text.splitlines() if not ln.startswith("#")))))
    assert len(rows) == 4 and rows[0]["prec"] == "dd" and "gpus" in rows[0]
    assert main(["report", "--in", path, "--format", "winners"]) == EX_OK
    grid = capsys.readouterr().out
    assert "winners for threads=1\n" in grid and "winners for threads=1 gpus=8" in grid
    assert "B@32" in grid and "S" in grid and "?" in grid


def test_usage_and_io_errors(tmp_path, capsys):
    assert main(["frobnicate"]) == EX_USAGE
    assert main(["report", "--in", str(tmp_path / "missing.tbl")]) == EX_IO
    bad = tmp_path / "bad.tbl"
    bad.write_text("not a table\n")
    assert main(["report", "--in", str(bad)]) == EX_IO


def test_lock_excludes_concurrent_timed_runs(tmp_path):
    lock = os.path.join(tempfile.gettempdir(), LOCK_NAME)
    with open(lock, "w") as fp:
        fp.write("12345")
    try:
        rc = main(["tune", "--prec", "dd", "--dims", "16", "--nmin", "4", "--threads", "1",
                   "--out", str(tmp_path / "t.tbl")])
        assert rc == EX_MEASURE
    finally:
        os.unlink(lock)


def test_threads_env_cap(monkeypatch):
    from paper_1710_01839_b200.cli import _cap_threads
    monkeypatch.setenv("MPMM_THREADS_MAX", "2")
    assert _cap_threads([1, 2, 4, 8]) == [1, 2]


@pytest.mark.gpu
def test_tune_grid_and_report(gpu, tmp_path, capsys):
    out = tmp_path / "t.tbl"
    rc = main(["tune", "--prec", "dd,qd", "--dims", "16,24", "--nmin", "4,8", "--threads", "1",
               "--out", str(out), "--cutoffs", "4,8"])
    assert rc == EX_OK
    table = mp.load_table(str(out))
    assert len(table.rows) == 4
    assert os.path.exists(str(out) + ".csv")
    assert main(["report", "--in", str(out), "--format", "winners"]) == EX_OK
    assert "?" not in capsys.readouterr().out


@pytest.mark.gpu
def test_tune_exact_mode_v3_table_and_report(gpu, tmp_path, capsys):
    out = tmp_path / "x.tbl"
    rc = main(["tune", "--prec", "dd", "--dims", "128,256", "--nmin", "16,32", "--threads", "1",
               "--out", str(out), "--cutoffs", "64", "--exact-mode", "--warmup", "1"])
    assert rc == EX_OK
    assert open(out).read().startswith("mpmmtune v3")
    table = mp.load_table(str(out))
    assert len(table.rows) == 2 and all(r.exact_time_s > 0 for r in table.rows)
    with open(str(out) + ".csv") as fp:
        hdr = next(ln for ln in fp if not ln.startswith("#"))
    assert "exact_s" in hdr
    assert main(["report", "--in", str(out), "--format", "winners"]) == EX_OK
    assert "?" not in capsys.readouterr().out


@pytest.mark.gpu
def test_verify_ok_and_detects_injected_fault(gpu, monkeypatch, capsys):
    assert main(["verify", "--prec", "dd,qd", "--dims", "17,32", "--nmin", "8", "--cutoff", "8",
                 "--exact"]) == EX_OK
    import paper_1710_01839_b200.cli as cli_mod
    real = cli_mod.matmul_strassen

    def broken(a, b, *args, **kw):
        c = real(a, b, *args, **kw)
        c.data[0, 0, 0] *= 1.0 + 1e-10
        return c
    monkeypatch.setattr(cli_mod, "matmul_strassen", broken)
    assert main(["verify", "--prec", "dd", "--dims", "16", "--nmin", "8",
                 "--cutoff", "8"]) == EX_VERIFY


@pytest.mark.gpu
def test_predict_layout(gpu, capsys):
    assert main(["predict", "--prec", "dd", "--dim", "256", "--nmin", "16,32,64"]) == EX_OK
    out = capsys.readouterr().out
    assert "best n_min=" in out and out.count("\n") >= 5


@pytest.mark.gpu
def test_tune_gpu_sweep_seeded_inputs(gpu, tmp_path, capsys):
    """tune --gpus 1,2,8 --inputs seeded: rows per GPU count (G > 1 from the
    shard product plus the broadcast model, 'G~' in the v2 table), the
    gpus_source CSV column, a winners grid per GPU count."""
    out = tmp_path / "g.tbl"
    rc = main(["tune", "--prec", "dd", "--dims", "256", "--nmin", "16,32", "--threads", "1",
               "--gpus", "1,2,8", "--cutoffs", "64", "--inputs", "seeded", "--seed", "1",
               "--out", str(out)])
    assert rc == EX_OK
    text = open(out).read()
    assert text.startswith("mpmmtune v2") and " 2~ " in text and " 8~ " in text
    rows = [ln for ln in open(str(out) + ".csv") if not ln.startswith("#")]
    assert rows[0].startswith("prec,bits,n,threads,gpus,gpus_source,")
    assert len(rows) == 4 and "shard+bcast model" in rows[3]
    assert main(["report", "--in", str(out), "--format", "winners"]) == EX_OK
    grid = capsys.readouterr().out
    assert "gpus=2" in grid and "gpus=8" in grid and "?" not in grid
