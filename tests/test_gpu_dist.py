"""Row-sharded runs (world size 2) of the device path on the GPU.

The gpurun box has one B200, so both ranks run on cuda:0 with the gloo backend
(host-staged allreduce of CUDA tensors).  No kernel of one rank waits on the
other: the one exchange per pass is the host-mediated Gram allreduce, exactly
where the NCCL allreduce sits at N > 1 on a multi-GPU box.  This exercises the
product's sharded control flow end to end on real kernels:
  * rank r factors rows [r m / 2, (r+1) m / 2) (paper_2507_07788_b200.dist.row_range);
  * every k x k stage runs redundantly on the allreduced Gram with the GLOBAL m
    in the shift rule (reference kernels.py:181-194), so both ranks take the
    same decisions;
  * the gated one-pass-ahead host loop (rs_chol_qr, chol_qr_update) and the
    fixed schedules (chol_qr2, s_chol_qr3) run unchanged.
The sharded result is compared with the single-process run of the same input
and with the CPU oracle (R within 1e-10 relative for well-conditioned input,
LOO_F / RRR_F within 10x).
"""

from __future__ import annotations

import math
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U = 1.11e-16
WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    """(name, builder) pairs; every rank rebuilds the same host input from a seed."""
    from paper_2507_07788_b200.workloads import host_gaussian, host_svd_matrix

    return {
        "rs_kappa12": lambda: host_svd_matrix(24_002, 64, 12.0, seed=11),
        "rs_kappa15_k128": lambda: host_svd_matrix(30_000, 128, 15.0, seed=5, u_from="cholqr2"),
        "cqr2_k128": lambda: host_gaussian(40_001, 128, seed=3),
        "s3_kappa12": lambda: host_svd_matrix(20_000, 64, 12.0, seed=0),
    }


def _run(cq, name, x):
    a = cq.CudaVectorArray.from_numpy(x)
    algo = {"rs": cq.rs_chol_qr, "cqr2": cq.chol_qr2, "s3": cq.s_chol_qr3}[name.split("_")[0]]
    res = algo(a)
    loo = cq.loss_of_orthogonality(res.q, norm="frobenius")
    rrr = cq.reconstruction_residual(a, res.q, res.r, norm="frobenius")
    return {"r": np.asarray(res.r), "attempts": list(res.shift_attempts), "shifts": list(res.shifts_applied),
            "iterations": res.iterations, "loo": loo, "rrr": rrr}


def _run_update(cq, seed=7, m=20_001, p=16, blocks=4):
    """Initial rs_chol_qr on p columns, then `blocks` appended blocks A_j = Q C + 1e-8 G (config 4's construction)."""
    from paper_2507_07788_b200.workloads import host_gaussian, next_block

    rng = np.random.default_rng(seed)
    x0 = host_gaussian(m, p, seed)
    res = cq.rs_chol_qr(cq.CudaVectorArray.from_numpy(x0))
    q, r = res.q, res.r
    full = [x0]
    attempts = []
    for _ in range(blocks):
        blk = next_block(q.to_numpy(), rng, p=p)
        full.append(blk)
        up = cq.chol_qr_update(q, r, cq.CudaVectorArray.from_numpy(blk))
        attempts.append(list(up.shift_attempts))
        q, r = up.q, up.r
    a = cq.CudaVectorArray.from_numpy(np.hstack(full))
    return {"r": np.asarray(r), "attempts": attempts,
            "loo": cq.loss_of_orthogonality(q, norm="frobenius"),
            "rrr": cq.reconstruction_residual(a, q, r, norm="frobenius")}


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD),
                      LOCAL_RANK="0")   # one GPU on the box: both ranks on cuda:0
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2507_07788_b200 as cq
        from paper_2507_07788_b200._device import ctx

        assert ctx().world == WORLD and ctx().rank == rank
        out = {}
        for name, build in _cases().items():
            out[name] = _run(cq, name, build())
        out["update"] = _run_update(cq)
        out["again"] = _run(cq, "rs_kappa15_k128", _cases()["rs_kappa15_k128"]())
        out["rows"] = ctx().row_range(24_002)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array(out, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded(tmp_path_factory):
    import torch.multiprocessing as mp

    out_dir = str(tmp_path_factory.mktemp("dist"))
    mp.start_processes(_worker, args=(_free_port(), out_dir), nprocs=WORLD, join=True, start_method="spawn")
    return [np.load(os.path.join(out_dir, f"rank{r}.npy"), allow_pickle=True).item() for r in range(WORLD)]


def test_ranks_own_disjoint_rows(sharded):
    assert sharded[0]["rows"] == (0, 12_001) and sharded[1]["rows"] == (12_001, 24_002)


def test_ranks_agree_bitwise(sharded):
    """Both ranks factor the same reduced Grams: R, decisions and shifts identical."""
    a, b = sharded
    for name in list(_cases()) + ["update"]:
        assert np.array_equal(a[name]["r"], b[name]["r"]), name
        assert a[name]["attempts"] == b[name]["attempts"], name
        if "shifts" in a[name]:
            assert a[name]["shifts"] == b[name]["shifts"], name


def test_sharded_runs_are_deterministic(sharded):
    """Two sharded runs of the same input give bitwise the same R and shifts:
    the cross-rank sum is an all-gather plus an in-order device sum, so the
    collective's algorithm cannot change a bit (reference
    tests/test_algorithms.py:107-113)."""
    for rank in sharded:
        assert np.array_equal(rank["again"]["r"], rank["rs_kappa15_k128"]["r"])
        assert rank["again"]["shifts"] == rank["rs_kappa15_k128"]["shifts"]


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("name", ["rs_kappa12", "rs_kappa15_k128", "cqr2_k128", "s3_kappa12"])
def test_sharded_matches_single_process_and_oracle(sharded, name):
    import paper_2507_07788_b200 as cq
    from oracle import cholqr_oracle as co

    x = _cases()[name]()
    one = _run(cq, name, x)
    two = sharded[0][name]
    k = x.shape[1]
    ref = {"rs": co.rs_chol_qr, "cqr2": co.chol_qr2, "s3": co.s_chol_qr3}[name.split("_")[0]](x)
    floor = 10 * U * math.sqrt(k)
    for mine in (one, two):
        assert mine["loo"] <= 10 * max(co.loo_fro(ref.q), floor), (name, mine["loo"])
        assert mine["rrr"] <= 10 * max(co.rrr_fro(x, ref.q, ref.r), floor), (name, mine["rrr"])
    if name == "cqr2_k128":   # well-conditioned: R within 1e-10 of the oracle and of the 1-rank run
        assert _rel(two["r"], ref.r) < 1e-10
        assert _rel(two["r"], one["r"]) < 1e-10
    if name == "s3_kappa12":   # the unconditional first shift uses the global m
        assert two["shifts"][0] == pytest.approx(ref.shifts_applied[0], rel=1e-6)
        assert two["shifts"][0] == pytest.approx(one["shifts"][0], rel=1e-6)
    if name == "rs_kappa15_k128":   # structural breakdowns (kappa 1e15): the first pass shifts on both
        assert two["attempts"][0] >= 1 and one["attempts"][0] >= 1


def test_sharded_update_chain(sharded):
    import paper_2507_07788_b200 as cq

    one = _run_update(cq)
    two = sharded[0]["update"]
    assert two["attempts"] == one["attempts"]
    assert _rel(two["r"], one["r"]) < 1e-10
    assert np.all(np.tril(two["r"], -1) == 0.0)
    floor = 10 * U * math.sqrt(two["r"].shape[0])
    assert two["loo"] <= 10 * max(one["loo"], floor)
    assert two["rrr"] <= 10 * max(one["rrr"], floor)


@pytest.mark.parametrize("config,rows", [(3, 400_000), (4, 200_000)])
def test_bench_two_ranks_plumbing(config, rows, tmp_path):
    """bench.py's N > 1 path (torchrun, row sharding, max-over-ranks timing,
    e2e, the update chain) end to end with two ranks on cuda:0 and gloo
    (CQR_BENCH_ONE_GPU_RANKS): one JSON line from rank 0 with n_gpus = 2."""
    import json
    import subprocess

    env = dict(os.environ, CQR_BENCH_ONE_GPU_RANKS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", str(config), "--steps", "2", "--warmup", "1", "--rows", str(rows), "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    if config != 4:   # the update chain reports no e2e
        assert line["e2e"]["value"] > 0
    assert line["config"]["rows"] == rows
