"""The band-cluster k x k stage (96 < k <= 256: one CTA per 32-row band in a
thread-block cluster, DSMEM hand-over, cluster-distributed power iteration,
speculative RECOMPUTE merged by the finish kernel) against the single-CTA
path on the same Gramians (cqr_debug_factor_cluster).  Both implement
kernels.py:61-194 / algorithms.py:295-317, 358-397; they differ only in
rounding order.  GPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("code", "retries", "n_shifts", "pivot_index", "est_calls", "est_flag", "escalations", "singular_index")


def _gram(k, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "spd":
        a = rng.standard_normal((4 * k, k))
        return a.T @ a
    if kind == "zerocol":
        a = rng.standard_normal((4 * k, k))
        a[:, k // 2] = 0.0
        return a.T @ a
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.logspace(0, -12, k)            # kappa 1e12: the plain attempt holds or breaks at a clear pivot
    if kind == "indef":
        lam[-1] = -1e-3                      # a clearly negative direction: structural breakdown
    g = (q * lam) @ q.T
    return 0.5 * (g + g.T)


def _run(k, policy, g, cluster, fixed_shift=0.0):
    """cluster: 1 -> mode 2 (the band-cluster path from k > 64, every policy); 0 -> single CTA."""
    import torch

    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._device import ctx
    from paper_2507_07788_b200._engine import Engine

    cx = ctx()
    cx.lib.cqr_debug_factor_cluster(2 if cluster else 0)
    try:
        eng = Engine(k, cq.AlgoConfig())
        eng.G.copy_(torch.from_numpy(g).to(cx.device))
        pol = {"plain": _lib.POLICY_PLAIN, "recompute": _lib.POLICY_RECOMPUTE,
               "shift_once": _lib.POLICY_SHIFT_ONCE, "fixed": _lib.POLICY_FIXED_SHIFT,
               "estimate": _lib.POLICY_ESTIMATE}[policy]
        st = eng.factor(pol, 10 ** 6, k, fixed_shift=fixed_shift)
        torch.cuda.synchronize()
        rk = eng.Rk.cpu().numpy()[:k, :k].T.copy()        # Rk is column-major: row c of the tensor = column c
        racc = eng.Racc.cpu().numpy()[:k, :k].T.copy()
        return st, rk, racc
    finally:
        cx.lib.cqr_debug_factor_cluster(1)


@pytest.mark.parametrize("k", [100, 128, 129, 160, 200, 255, 256])
@pytest.mark.parametrize("policy", ["plain", "recompute", "shift_once"])
def test_cluster_matches_single_cta_on_spd(k, policy):
    g = _gram(k, "spd", seed=k)
    a = _run(k, policy, g, 1)
    b = _run(k, policy, g, 0)
    for f in FIELDS:
        assert getattr(a[0], f) == getattr(b[0], f), f
    assert a[0].code == 0
    np.testing.assert_allclose(a[1], b[1], rtol=0, atol=1e-12 * np.abs(b[1]).max())
    np.testing.assert_array_equal(np.tril(a[1], -1), 0.0)
    sigma = a[0].shifts[-1] if a[0].shifts else 0.0     # shift_once factors G + sigma I
    np.testing.assert_allclose(a[1].T @ a[1], g + sigma * np.eye(k), rtol=0, atol=1e-12 * np.abs(g).max())
    np.testing.assert_allclose(a[2], b[2], rtol=0, atol=1e-12 * np.abs(b[2]).max())
    if policy == "shift_once":
        np.testing.assert_allclose(a[0].shifts, b[0].shifts, rtol=1e-12)
        if k > 128:   # the same per-row and reduction order as the single CTA's X-in-L2 estimate: the same bits
            assert a[0].norm_est == b[0].norm_est
        else:         # the single CTA runs its warp-only iteration on X in shared memory (another order)
            assert abs(a[0].norm_est / b[0].norm_est - 1) < 1e-12


@pytest.mark.parametrize("k", [136, 256])
def test_cluster_recompute_breakdown_takes_the_shifted_branch(k):
    """Plain attempt breaks down at a structural pivot: the speculative group's
    result (estimate + shifted attempt) is merged by the finish kernel, with the
    plain attempt's pivot recorded -- as in the single-CTA path."""
    g = _gram(k, "indef", seed=3)
    a = _run(k, "recompute", g, 1)
    b = _run(k, "recompute", g, 0)
    for f in ("code", "retries", "n_shifts", "pivot_index", "est_calls", "escalations"):
        assert getattr(a[0], f) == getattr(b[0], f), f
    assert a[0].retries >= 1 and a[0].pivot_index >= 0
    np.testing.assert_allclose(a[0].shifts, b[0].shifts, rtol=1e-9)
    assert a[0].plain_margin < 0 and b[0].plain_margin < 0
    if a[0].code == 0:
        np.testing.assert_array_equal(np.tril(a[1], -1), 0.0)
        np.testing.assert_allclose(a[1], b[1], rtol=0, atol=1e-9 * np.abs(b[1]).max())


@pytest.mark.parametrize("k", [144, 256])
def test_cluster_plain_breakdown_reports_the_first_pivot(k):
    g = _gram(k, "zerocol", seed=5)
    a = _run(k, "plain", g, 1)
    b = _run(k, "plain", g, 0)
    assert a[0].code == b[0].code == 3            # CQR_BREAKDOWN
    assert a[0].pivot_index == b[0].pivot_index == k // 2


@pytest.mark.parametrize("k", [160, 256])
def test_cluster_estimate_policy_same_bits(k):
    g = _gram(k, "spd", seed=7)
    a = _run(k, "estimate", g, 1)
    b = _run(k, "estimate", g, 0)
    assert a[0].code == b[0].code
    assert a[0].norm_est == b[0].norm_est
    assert a[0].est_flag == b[0].est_flag


def test_cluster_deterministic():
    g = _gram(256, "indef", seed=9)
    a = _run(256, "recompute", g, 1)
    b = _run(256, "recompute", g, 1)
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    assert a[0].shifts == b[0].shifts
