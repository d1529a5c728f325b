"""Multi-rank (world size 2, gloo, CPU) checks of the row-sharded decomposition.

The GPU box gives one device per call, so the N > 1 data path is exercised
here with the product's own sharding helpers (`paper_2507_07788_b200.dist`):
each rank owns rows [r m / P, (r+1) m / P), forms its local Gram (NumPy
stands in for the K1 kernel), the Grams are summed with `reduce_ranks_`
(all-gather + in-order sum: deterministic and bit-symmetric),
and every rank runs the k x k stage of the oracle on the reduced matrix with
the GLOBAL m in the shift rule.  The sharded run must reproduce the
single-process oracle's decisions and factor, and both ranks must hold
bit-identical Grams and decisions.
"""

from __future__ import annotations

import os
import socket
import warnings

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_07788_b200.dist import reduce_ranks_, row_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_rs(x, rank, world):
    """rs_chol_qr with row-sharded tall work and allreduced Grams (mirrors
    paper_2507_07788_b200.algorithms.rs_chol_qr's control flow)."""
    from oracle import cholqr_oracle as co

    m, n = x.shape
    lo, hi = row_range(m, rank, world)
    q = np.asfortranarray(x[lo:hi])
    cfg = co.default_cfg()

    def gram(qloc):
        g = qloc.T @ qloc
        g = torch.from_numpy((g + g.T) / 2.0)   # bit-symmetric local partial, as the Gram kernels write it
        reduce_ranks_(g)
        return g.numpy()

    g = gram(q)
    r = np.eye(n)
    attempts, shifts, grams = [], [], [g.copy()]
    its = 0
    err = co.identity_distance(g)
    while not err < cfg["tol"]:
        assert its < cfg["max_iter"]
        try:
            rk = co.cholesky_upper(g)
            attempts.append(0)
        except co.OracleBreakdown:
            rk, tries, _ = co._recomputed_shift_attempts(g, m, n, cfg, shifts)   # GLOBAL m
            attempts.append(tries)
        q = co.lincomb(q, co.tri_inverse(rk))
        r = co.tri_mult(rk, r)
        g = gram(q)
        grams.append(g.copy())
        its += 1
        err = co.identity_distance(g)
    return q, r, attempts, shifts, grams


def _worker(rank, world, port, x, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            q, r, attempts, shifts, grams = _sharded_rs(x, rank, world)
            q2, r2, _, shifts2, grams2 = _sharded_rs(x, rank, world)
        # run-to-run determinism at world size > 1 (reference test_algorithms.py:107-113)
        np.testing.assert_array_equal(r, r2)
        np.testing.assert_array_equal(q, q2)
        assert shifts == shifts2
        for g in grams:
            np.testing.assert_array_equal(g, g.T)   # bit-symmetric after the cross-rank sum
        # bit-identical Grams and decisions on every rank
        allg = [None] * world
        dist.all_gather_object(allg, (attempts, shifts, [gg.tobytes() for gg in grams]))
        assert all(a == allg[0] for a in allg), "ranks disagree"
        qs = [None] * world
        dist.all_gather_object(qs, q)
        if rank == 0:
            out.put((np.vstack(qs), r, attempts, shifts, grams[0]))
    finally:
        dist.destroy_process_group()


def _run(x, world=2):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = out.get(timeout=240)   # read before joining: a large put blocks until consumed
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    return res


def test_row_range_partitions_rows():
    for m in (1, 7, 16, 1001):
        for world in (1, 2, 3, 8):
            spans = [row_range(m, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        row_range(10, 2, 2)


@pytest.mark.parametrize("cond", [2.0, 12.0])
def test_sharded_rs_chol_qr_matches_single_process(cond):
    from oracle import cholqr_oracle as co
    from oracle import matgen_oracle as mg

    x = mg.generate(3000, 24, cond, seed=3)
    q, r, attempts, shifts, g0 = _run(x)
    ref = co.rs_chol_qr(x)
    # the first Gram is the same matrix up to summation order
    np.testing.assert_allclose(g0, co.gram(x), rtol=1e-12, atol=1e-12 * np.max(np.abs(g0)))
    np.testing.assert_array_equal(g0, g0.T)
    assert attempts == ref.shift_attempts
    np.testing.assert_allclose(shifts, ref.shifts_applied, rtol=1e-6)
    if cond <= 4:
        assert np.max(np.abs(r - ref.r)) <= 1e-10 * np.max(np.abs(ref.r))
    assert co.loo_fro(q) <= 10 * max(co.loo_fro(ref.q), 1e-14)
    assert co.rrr_fro(x, q, r) <= 10 * max(co.rrr_fro(x, ref.q, ref.r), 1e-15)


def _reduce_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)
        g = rng.standard_normal((33, 33)) * 10.0 ** rng.integers(-8, 8, size=(33, 33))
        g = (g + g.T) / 2.0
        bt = rng.standard_normal((5, 33))
        flat = torch.from_numpy(np.concatenate([bt.ravel(), g.ravel()]))
        reduce_ranks_(flat)
        allv = [None] * world
        dist.all_gather_object(allv, flat.numpy().tobytes())
        assert all(v == allv[0] for v in allv)
        if rank == 0:
            out.put(flat.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_reduce_ranks_is_in_rank_order_and_bit_symmetric(world):
    """The packed [Bt | G] partials summed over 2 and 3 ranks: every rank holds
    the same bits, equal to ((p0 + p1) + p2) in rank order, and the G part is
    bit-symmetric (a ring allreduce at world >= 3 may not be)."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = out.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    parts = []
    for r in range(world):
        rng = np.random.default_rng(100 + r)
        g = rng.standard_normal((33, 33)) * 10.0 ** rng.integers(-8, 8, size=(33, 33))
        g = (g + g.T) / 2.0
        bt = rng.standard_normal((5, 33))
        parts.append(np.concatenate([bt.ravel(), g.ravel()]))
    want = parts[0].copy()
    for p_ in parts[1:]:
        want = want + p_
    np.testing.assert_array_equal(got, want)
    gsum = got[5 * 33:].reshape(33, 33)
    np.testing.assert_array_equal(gsum, gsum.T)
