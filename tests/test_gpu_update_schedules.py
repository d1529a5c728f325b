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


def _pass(m, q, p, initial, teams, seed):
    import torch

    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._device import ctx
    from paper_2507_07788_b200._engine import Engine

    cx = ctx()
    cx.lib.cqr_debug_update_narrow_teams(teams)
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
