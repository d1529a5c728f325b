"""The cholqr-compatible CLI and Matrix Market I/O through device arrays
(reference tests/test_cli.py, tests/test_varray.py:215-238)."""

from __future__ import annotations

import csv
import io
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cq():
    import paper_2507_07788_b200 as cq

    return cq


def _gen(tmp_path, name="a.mtx", m=80, n=5, cond=2.0, seed=0):
    from paper_2507_07788_b200.cli import main

    path = tmp_path / name
    assert main(["gen", "-m", str(m), "-n", str(n), "--log10-cond", str(cond), "--seed", str(seed),
                 "-o", str(path)]) == 0
    return path


def _csv(text):
    rows = list(csv.reader(io.StringIO(text)))
    return rows[0], rows[1:]


def test_gen_writes_matrix_and_sidecar(tmp_path):
    cq = _cq()
    path = _gen(tmp_path, m=60, n=4, cond=3.0, seed=7)
    meta = json.loads((tmp_path / "a.mtx.json").read_text())
    assert (meta["m"], meta["n"], meta["log10_cond"], meta["seed"]) == (60, 4, 3.0, 7)
    assert meta["backend"] == "cuda" and meta["seed_mixing"]
    loaded = cq.load_matrix_market(str(path))
    direct, sigma = cq.generate(cq.MatrixSpec(60, 4, 3.0, seed=7))
    np.testing.assert_array_equal(cq.to_dense_block(loaded), cq.to_dense_block(direct))
    assert meta["singular_values"] == [float(s) for s in sigma]


def test_gen_matches_reference_file_bytes(tmp_path):
    path = _gen(tmp_path, m=40, n=3, cond=2.5, seed=9)
    assert path.read_bytes() == open(os.path.join(HERE, "ref_gen.mtx"), "rb").read()
    assert _gen(tmp_path, name="b.mtx", m=40, n=3, cond=2.5, seed=9).read_bytes() == path.read_bytes()


def test_matrix_market_round_trip_through_device(tmp_path):
    cq = _cq()
    rng = np.random.default_rng(11)
    block = rng.standard_normal((9, 4))
    block[0, 0] = 1.0 / 3.0
    block[1, 1] = -0.0
    first, second = tmp_path / "first.mtx", tmp_path / "second.mtx"
    cq.save_matrix_market(cq.CudaVectorArray.from_numpy(block), str(first))
    loaded = cq.load_matrix_market(str(first))
    np.testing.assert_array_equal(cq.to_dense_block(loaded), block)
    cq.save_matrix_market(loaded, str(second))
    assert first.read_bytes() == second.read_bytes()
    ref = cq.load_matrix_market(os.path.join(HERE, "ref_block.mtx"))
    cq.save_matrix_market(ref, str(second))
    assert second.read_bytes() == open(os.path.join(HERE, "ref_block.mtx"), "rb").read()


def test_matrix_market_wide_array_streams_column_blocks(tmp_path):
    cq = _cq()
    block = np.random.default_rng(5).standard_normal((33, 130))
    path = tmp_path / "w.mtx"
    cq.save_matrix_market(cq.CudaVectorArray.from_numpy(block), str(path))
    np.testing.assert_array_equal(cq.to_dense_block(cq.load_matrix_market(str(path))), block)


def test_qr_happy_path(tmp_path, capsys):
    cq = _cq()
    from paper_2507_07788_b200.cli import main

    path = _gen(tmp_path)
    assert main(["qr", "rscholqr", str(path)]) == 0
    out = capsys.readouterr().out.strip().splitlines()[-1]
    assert "algorithm=rscholqr" in out and "backend=cuda" in out and "status=ok" in out
    q = cq.load_matrix_market(str(tmp_path / "a.q.mtx"))
    r = cq.to_dense_block(cq.load_matrix_market(str(tmp_path / "a.r.mtx")))
    assert cq.loss_of_orthogonality(q) <= 1e-12
    np.testing.assert_array_equal(np.tril(r, -1), 0.0)
    block = cq.to_dense_block(cq.load_matrix_market(str(path)))
    np.testing.assert_allclose(cq.to_dense_block(q) @ r, block, rtol=0, atol=1e-10)


def test_qr_output_prefix_and_algorithms(tmp_path):
    from paper_2507_07788_b200.cli import main

    path = _gen(tmp_path)
    for alg in ("cholqr2", "scholqr3", "ischolqr", "pncholqr:2"):
        assert main(["qr", alg, str(path), "-o", str(tmp_path / alg.replace(":", "_"))]) == 0
        assert (tmp_path / (alg.replace(":", "_") + ".q.mtx")).exists()


def test_qr_exit_codes(tmp_path, capsys):
    cq = _cq()
    from paper_2507_07788_b200.cli import main

    path = _gen(tmp_path, name="ill.mtx", m=300, n=10, cond=12.0)
    assert main(["qr", "cholqr", str(path)]) == 3
    assert "cholesky breakdown" in capsys.readouterr().err
    block = cq.to_dense_block(cq.generate(cq.MatrixSpec(80, 5, 1.0, seed=3))[0])
    block[:, 2] = 0.0
    deg = tmp_path / "degenerate.mtx"
    cq.save_matrix_market(block, str(deg))
    code = main(["qr", "rscholqr", str(deg), "--max-iter", "3"])
    cap = capsys.readouterr()
    assert code == 4 and "status=iter_limit" in cap.out and "iteration cap" in cap.err
    assert main(["qr", "rscholqr", str(tmp_path / "nope.mtx")]) == 2
    assert "cannot read" in capsys.readouterr().err


def test_bench_csv_contract(tmp_path):
    from paper_2507_07788_b200.cli import CSV_HEADER, BenchRecord, main

    out = tmp_path / "bench.csv"
    assert main(["bench", "-m", "60", "-n", "4", "--points", "0:2:2", "--algs", "cholqr,rscholqr", "--reps", "2",
                 "-o", str(out), "--gnuplot", str(tmp_path / "b.gp")]) == 0
    header, rows = _csv(out.read_text())
    assert header == CSV_HEADER
    assert len(rows) == 2 * 2 * 2
    for row in rows:
        rec = BenchRecord.from_row(row)
        assert rec.status == "ok" and rec.backend == "cuda"
        assert rec.runtime_s > 0 and rec.loo is not None and rec.flops > 0 and rec.iters >= 0
    assert (tmp_path / "b.gp").exists()


def test_bench_size_axis_to_stdout(capsys):
    from paper_2507_07788_b200.cli import main

    assert main(["bench", "-m", "60", "-n", "4", "--axis", "m", "--points", "40:400:2", "--reps", "1"]) == 0
    header, rows = _csv(capsys.readouterr().out)
    assert [int(r[2]) for r in rows] == [40, 400]


def test_flops_csv_contract(tmp_path):
    from paper_2507_07788_b200.cli import FLOPS_HEADER, main

    out = tmp_path / "flops.csv"
    assert main(["flops", "-m", "120", "-n", "6", "--points", "0:6:2", "--algs", "rscholqr,pncholqr:2,pncholqr:3",
                 "-o", str(out)]) == 0
    header, rows = _csv(out.read_text())
    assert header == FLOPS_HEADER
    assert len(rows) == 2 * 3
    for row in rows:
        rec = dict(zip(header, row))
        assert rec["match"] == "true"
        assert int(rec["total_measured"]) == int(rec["total_predicted"])
        if rec["algorithm"].startswith("pncholqr"):
            assert float(rec["ratio_measured"]) > 0 and float(rec["ratio_predicted"]) > 0
