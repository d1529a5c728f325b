"""Update-pass schedules against each other (GPU only): for bases up to 64
columns the pass runs two alternating 4-warp projection teams
(cqr_debug_update_narrow_teams(1), the default) or one 8-warp group (0).
Both compute every element with the same operations in the same order, so
Q', Bt' and G must agree bit for bit -- for the iteration and initial modes,
ragged row counts and every basis width up to 64 (including q < 64, where the
cross-Gram warps past q skip their chains)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# cqr_debug_update_lag: 0 = never, 1 = always, 2 = the measured rule (the
# library's defaults, restored after every case)
DEFAULT_MODE = 2
DEFAULT_SR16_FROM = 145


def _pass(m, q, p, initial, teams, seed, mode=None, sr16_from=None, direct=None):
    import torch

    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._device import ctx
    from paper_2507_07788_b200._engine import Engine

    cx = ctx()
    cx.lib.cqr_debug_update_narrow_teams(teams)
    if mode is not None:
        cx.lib.cqr_debug_update_lag(mode)
    if sr16_from is not None:
        assert cx.lib.cqr_debug_update_sr16_from(sr16_from) == 0
    if direct is not None:
        cx.lib.cqr_debug_update_direct(direct)
    try:
        rng = np.random.default_rng(seed)
        qin = cq.CudaVectorArray.from_numpy(np.linalg.qr(rng.standard_normal((m, q)))[0])
        blk = cq.CudaVectorArray.from_numpy(rng.standard_normal((m, p)))
        eng = Engine(p, cq.AlgoConfig(), q=q)
        g = rng.standard_normal((p, p))
        eng.G.copy_(torch.from_numpy(g @ g.T + p * np.eye(p)).to(cx.device))
        eng.Bt.copy_(torch.from_numpy(1e-2 * rng.standard_normal((p, q))).to(cx.device))
        assert eng.factor(_lib.POLICY_PLAIN, m, p).code == _lib.FACTORED
        eng.update_pass(qin, blk, initial=initial)
        torch.cuda.synchronize()
        return blk.to_numpy(), eng.Bt.cpu().numpy().copy(), eng.G.cpu().numpy().copy()
    finally:
        cx.lib.cqr_debug_update_narrow_teams(1)
        cx.lib.cqr_debug_update_lag(DEFAULT_MODE)
        cx.lib.cqr_debug_update_sr16_from(DEFAULT_SR16_FROM)
        cx.lib.cqr_debug_update_direct(1)


@pytest.mark.parametrize("q", [1, 7, 16, 33, 48, 64])
@pytest.mark.parametrize("initial", [False, True])
def test_narrow_teams_match_single_group_bitwise(q, initial):
    m, p = 50_011, 16          # ragged: not a multiple of the 64-row sub-panel
    a = _pass(m, q, p, initial, 1, seed=q)
    b = _pass(m, q, p, initial, 0, seed=q)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("p", [1, 5, 16])
def test_narrow_teams_narrow_blocks(p):
    a = _pass(20_000, 40, p, False, 1, seed=p)
    b = _pass(20_000, 40, p, False, 0, seed=p)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("q", [145, 160, 192, 200, 256, 300, 333, 448, 496, 512])
@pytest.mark.parametrize("mode", [1, 2])
def test_wide_schedules_match_plain_bitwise(q, mode):
    """One projection group (bases wider than 144 columns): the cross-Gram lag
    only moves work in time."""
    m, p = 30_011, 16          # ragged; ~13 sub-panels per CTA at 16 rows
    a = _pass(m, q, p, False, 1, seed=q, mode=0)
    b = _pass(m, q, p, False, 1, seed=q, mode=mode)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("m", [16, 48, 2400, 148 * 16 * 2 + 16])
def test_lag_short_sweeps(m):
    """0, 1 or 2 sub-panels per CTA (no next sub-panel to wait for)."""
    a = _pass(m, 256, 16, False, 1, seed=m, mode=0)
    b = _pass(m, 256, 16, False, 1, seed=m, mode=1)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("q", [145, 160, 176, 192])
@pytest.mark.parametrize("initial", [False, True])
def test_sub_panel_height_switch(q, initial):
    """16-row against 32-row sub-panels (cqr_debug_update_sr16_from): Q' bitwise
    (per-row arithmetic), Bt' and G to rounding (the row sums are grouped by
    sub-panel)."""
    m, p = 40_000, 16
    a = _pass(m, q, p, initial, 1, seed=q, sr16_from=193)
    b = _pass(m, q, p, initial, 1, seed=q, sr16_from=145)
    np.testing.assert_array_equal(a[0], b[0])
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_allclose(x, y, rtol=0, atol=1e-12 * max(1.0, float(np.abs(x).max())))



@pytest.mark.parametrize("q", [1, 16, 40, 64, 100, 144, 160, 256, 333, 496])
@pytest.mark.parametrize("m", [64 * 500, 64 * 500 + 16])
def test_initial_pass_direct_matches_copy_bitwise(q, m):
    """Initial pass (Bt = Q_in^T A, G = A^T A): the cross-Gram warps reading the
    staged block in place (cqr_debug_update_direct(1), full sub-panels only) against
    the copy through the Q' ring; with ragged rows both runs take the copy path."""
    a = _pass(m, q, 16, True, 1, seed=q, direct=0)
    b = _pass(m, q, 16, True, 1, seed=q, direct=1)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
