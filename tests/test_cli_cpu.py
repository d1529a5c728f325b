"""CLI, matrix generation and Matrix Market format on CPU (no device calls).

Contracts follow the reference's tests/test_cli.py and tests/test_varray.py;
the byte fixtures were written by the unmodified reference
(tests/golden/make_mtx.py)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2507_07788_b200 import cli, matgen, mmio

from conftest import Golden

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# reference cli.py:23-62
REF_CSV_HEADER = ["algorithm", "backend", "m", "n", "log10_cond", "rep", "runtime_s", "loo", "rrr", "rcr", "iters",
                  "shifts", "flops", "status"]
REF_FLOPS_HEADER = ["algorithm", "backend", "m", "n", "log10_cond", "panels", "outer_iters", "gemm_measured",
                    "gemm_predicted", "trmm_measured", "trmm_predicted", "potrf_measured", "potrf_predicted",
                    "trtri_measured", "trtri_predicted", "fro_norm_measured", "fro_norm_predicted",
                    "eig_est_measured", "eig_est_predicted", "total_measured", "total_predicted", "match",
                    "ratio_measured", "ratio_predicted"]


def test_csv_schemas_match_reference():
    assert cli.CSV_HEADER == REF_CSV_HEADER
    assert cli.FLOPS_HEADER == REF_FLOPS_HEADER
    assert cli.STATUSES == ("ok", "breakdown", "iter_limit", "oom")


def _rec(**kw):
    base = dict(algorithm="rscholqr", backend="cuda", m=10, n=2, log10_cond=0.0, rep=0, runtime_s=0.1, loo=None,
                rrr=None, rcr=None, iters=None, shifts=None, flops=None, status="ok")
    base.update(kw)
    return cli.BenchRecord(**base)


def test_bench_record_validation():
    with pytest.raises(ValueError, match="status"):
        _rec(status="exploded")
    with pytest.raises(ValueError, match="runtime"):
        _rec(runtime_s=-1.0)


def test_bench_record_round_trips():
    rec = _rec(runtime_s=None, status="oom", log10_cond=2.5, rep=3, m=100, n=5)
    row = rec.to_row()
    assert row[6] == "" and row[4] == "2.5"
    assert cli.BenchRecord.from_row(row) == rec
    full = _rec(loo=1.5e-15, rrr=2e-16, rcr=3e-17, iters=3, shifts=1, flops=12345)
    assert cli.BenchRecord.from_row(full.to_row()) == full
    with pytest.raises(ValueError, match="cells"):
        cli.BenchRecord.from_row(full.to_row()[:-1])


def test_parse_errors_and_exit_codes(tmp_path, capsys):
    with pytest.raises(SystemExit):
        cli.main(["polish"])
    assert cli.main(["bench", "-m", "60", "-n", "4", "--reps", "0"]) == 2
    assert "--reps" in capsys.readouterr().err
    assert cli.main(["bench", "-m", "60", "-n", "4", "--axis", "m"]) == 2
    assert "--points is required" in capsys.readouterr().err
    assert cli.main(["bench", "-m", "60", "-n", "4", "--points", "1:2"]) == 2
    assert "start:stop:count" in capsys.readouterr().err
    assert cli.main(["bench", "-m", "60", "-n", "4", "--gnuplot", "x.gp"]) == 2
    assert "--gnuplot needs -o" in capsys.readouterr().err
    assert cli.main(["flops", "-m", "50", "-n", "3", "--algs", "mgs"]) == 2
    assert "flop prediction covers" in capsys.readouterr().err
    assert cli.main(["gen", "-m", "3", "-n", "5", "-o", str(tmp_path / "x.mtx")]) == 2
    assert "error:" in capsys.readouterr().err
    assert cli.main(["qr", "rscholqr", str(tmp_path / "x.mtx"), "--threads", "0"]) == 2
    assert "thread count" in capsys.readouterr().err
    with pytest.raises(cli.CLIError, match="unknown algorithm"):
        cli._runner("qrqr")
    with pytest.raises(cli.CLIError, match="panel count"):
        cli._runner("pncholqr:0")


def test_threads_env(monkeypatch, capsys, tmp_path):
    for var in cli.THREAD_ENV:   # restored by monkeypatch afterwards
        monkeypatch.setenv(var, os.environ.get(var, "1"))
    monkeypatch.setenv("CHOLQR_THREADS", "many")
    assert cli.main(["qr", "rscholqr", str(tmp_path / "x.mtx")]) == 2
    assert "CHOLQR_THREADS" in capsys.readouterr().err
    monkeypatch.setenv("CHOLQR_THREADS", "3")
    cli._export_threads(None)
    assert os.environ["OPENBLAS_NUM_THREADS"] == "3"


def test_sweep_points():
    args = cli.build_parser().parse_args(["bench", "-m", "1000", "-n", "8", "--axis", "m", "--points", "100:10000:3"])
    assert [p["m"] for p in cli.sweep_points(args)] == [100, 1000, 10000]
    args = cli.build_parser().parse_args(["bench", "-m", "1000", "-n", "8"])
    pts = cli.sweep_points(args)
    assert len(pts) == 21 and pts[0]["log10_cond"] == 0.0 and pts[-1]["log10_cond"] == 20.0
    args = cli.build_parser().parse_args(["bench", "-m", "1000", "-n", "8", "--axis", "backend"])
    assert [p["backend"] for p in cli.sweep_points(args)] == ["cuda"]


def test_gnuplot_script(tmp_path):
    path = tmp_path / "p.gp"
    cli.write_gnuplot(str(path), "b.csv", "cond", ["rscholqr", "cholqr2"], ["cuda"])
    text = path.read_text()
    assert "set xlabel 'log10 condition number'" in text
    assert text.count("with points") == 2 and "'b.csv' using 5:" in text


def test_matgen_matches_reference_bitwise():
    g = Golden()
    block, sigma = matgen.generate_host(matgen.MatrixSpec(300, 10, 6.0, 0))
    np.testing.assert_array_equal(block, g.arrays["matgen_300_10_c6_s0"])
    block, _ = matgen.generate_host(matgen.MatrixSpec(50, 1, 0.0, 0))
    np.testing.assert_array_equal(block, g.arrays["matgen_50_1_c0_s0"])
    meta = json.loads(open(os.path.join(HERE, "ref_gen.mtx.json")).read())
    spec = matgen.MatrixSpec(40, 3, 2.5, 9)
    assert matgen.effective_seed(spec) == meta["effective_seed"]
    assert matgen.SEED_MIXING == meta["seed_mixing"]
    block, sigma = matgen.generate_host(spec)
    assert [float(s) for s in sigma] == meta["singular_values"]
    np.testing.assert_array_equal(block, mmio.load_block(os.path.join(HERE, "ref_gen.mtx")))


def test_matgen_spec_validation():
    with pytest.raises(ValueError):
        matgen.MatrixSpec(3, 5, 1.0)
    with pytest.raises(ValueError):
        matgen.MatrixSpec(5, 3, -1.0)
    with pytest.raises(ValueError):
        matgen.MatrixSpec(5, 3, 1.0, seed=-1)


@pytest.mark.parametrize("name", ["ref_block.mtx", "ref_gen.mtx"])
def test_matrix_market_bytes_match_reference(tmp_path, name):
    src = os.path.join(HERE, name)
    block = mmio.load_block(src)
    out = tmp_path / "again.mtx"
    mmio.save_matrix_market(block, str(out))
    assert out.read_bytes() == open(src, "rb").read()


def test_matrix_market_edge_values_round_trip(tmp_path):
    block = np.array([[1.0 / 3.0, -0.0], [5e-324, np.inf], [-np.inf, 1e308]])
    path = tmp_path / "e.mtx"
    mmio.save_matrix_market(block, str(path))
    back = mmio.load_block(str(path))
    np.testing.assert_array_equal(back, block)
    assert np.signbit(back[0, 1])


def test_matrix_market_validation(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2\n1.0\n")
    with pytest.raises(ValueError, match="header"):
        mmio.load_block(str(bad))
    bad.write_text("%%MatrixMarket matrix array real general\n% comment\n2 2\n1.0\n")
    with pytest.raises(ValueError, match="expected 4 values"):
        mmio.load_block(str(bad))
    bad.write_text("%%MatrixMarket matrix array real general\n2 2 2\n")
    with pytest.raises(ValueError, match="size line"):
        mmio.load_block(str(bad))
    bad.write_text("%%MatrixMarket matrix array real general\n")
    with pytest.raises(ValueError, match="missing size"):
        mmio.load_block(str(bad))
    bad.write_text("%%MatrixMarket matrix array real general\n1 1\nabc\n")
    with pytest.raises(ValueError):
        mmio.load_block(str(bad))
