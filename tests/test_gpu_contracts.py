"""The reference's exact-value contracts for the shift rule, the update path and
the panel scheme, run on the device backend with the reference's own inputs
and thresholds (reference tests/test_algorithms.py:46-192,
tests/test_update_panel.py:36-170).  GPU only.

These pin decisions, not just quality: attempt counts, the 2u clamp, the x10
escalation ratio, the attempt limit and the iteration cap.
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 1.11e-16


def _cq():
    import paper_2507_07788_b200 as cq

    return cq


def _gen(m, n, cond, seed, zero=()):
    from oracle import matgen_oracle as mg

    blk = mg.generate(m, n, float(cond), seed)
    return mg.with_zero_columns(blk, list(zero)) if zero else blk


def _dev(block):
    return _cq().CudaVectorArray.from_numpy(np.asarray(block, dtype=float))


# ---------------------------------------------------------------- test_algorithms.py
def test_chol_qr_breaks_down_when_squared_condition_exceeds_roundoff():
    """test_algorithms.py:58-63: kappa = 1e9, seed 0 -- the reference raises.

    kappa^2 = 1e18 > 1/u: the Gramian's smallest eigenvalue (1e-18 relative)
    is below its own rounding error, so whether the Cholesky of the COMPUTED
    Gramian meets a non-positive pivot depends on how X^T X was rounded.  The
    device must either raise as well, or -- where its DMMA-accumulated Gramian
    happens to stay positive -- the oracle's own Cholesky on that same device
    Gramian must also succeed, with a rounding-level pivot: the decision is
    then a property of the rounded Gramian, not of the factor logic."""
    cq = _cq()
    import parity as P
    from oracle import cholqr_oracle as co

    a = _dev(_gen(300, 10, 9.0, 0))
    for fn in (cq.chol_qr, cq.chol_qr2):
        res, trace = P.traced(fn, a)
        if isinstance(res, cq.CholeskyBreakdown):
            continue
        assert not isinstance(res, Exception), res
        assert any(P.fragile_margin(x, 10) for x in res.pivot_margins), res.pivot_margins
        g, _ = P._device_x(trace[0])
        rk, dm, _ = co._attempt(g)
        assert rk is not None and P.fragile_margin(dm, 10), (fn.__name__, dm)


def test_chol_qr2_refines_orthogonality():
    """test_algorithms.py:66-74."""
    cq = _cq()
    a = _dev(_gen(300, 10, 7.0, 1))
    single, double = cq.chol_qr(a), cq.chol_qr2(a)
    assert double.iterations == 2
    assert cq.loss_of_orthogonality(double.q) <= 1e-14
    assert cq.loss_of_orthogonality(double.q) < cq.loss_of_orthogonality(single.q)
    assert cq.quality_report(a, double.q, double.r).rrr <= 1e-13


def test_s_chol_qr3_one_unconditional_shift():
    """test_algorithms.py:77-84."""
    cq = _cq()
    a = _dev(_gen(300, 10, 12.0, 0))
    res = cq.s_chol_qr3(a)
    assert res.iterations == 3 and len(res.shifts_applied) == 1 and res.shifts_applied[0] > 0
    assert res.profile is None
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(10) * 1e-13


def test_is_chol_qr_reuses_one_fixed_shift():
    """test_algorithms.py:87-92."""
    cq = _cq()
    res = cq.is_chol_qr(_dev(_gen(300, 10, 12.0, 0)))
    assert res.success and len(res.shifts_applied) >= 1 and len(set(res.shifts_applied)) == 1
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(10) * 1e-13


@pytest.mark.parametrize("algo", ["rs_chol_qr", "is_chol_qr"])
def test_iterated_bookkeeping_is_consistent(algo):
    """test_algorithms.py:95-103."""
    cq = _cq()
    res = getattr(cq, algo)(_dev(_gen(300, 10, 10.0, 2)))
    assert res.success
    assert len(res.shift_attempts) == res.iterations
    assert sum(res.shift_attempts) == len(res.shifts_applied)
    assert all(s > 0 for s in res.shifts_applied)
    assert res.orth_error is not None and res.orth_error < 1e-13


def test_rs_chol_qr_is_deterministic():
    """test_algorithms.py:106-112 (bitwise)."""
    cq = _cq()
    a = _dev(_gen(300, 10, 14.0, 3))
    one, two = cq.rs_chol_qr(a), cq.rs_chol_qr(a)
    np.testing.assert_array_equal(one.r, two.r)
    np.testing.assert_array_equal(one.q.to_numpy(), two.q.to_numpy())
    assert one.shifts_applied == two.shifts_applied


def test_rs_chol_qr_far_beyond_the_plain_breakdown_point():
    """test_algorithms.py:115-121: kappa = 1e18."""
    cq = _cq()
    a = _dev(_gen(300, 10, 18.0, 0))
    res = cq.rs_chol_qr(a)
    assert res.success and len(res.shifts_applied) >= 1
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(10) * 1e-13
    assert cq.quality_report(a, res.q, res.r).rrr <= 1e-12


def test_rs_chol_qr_iteration_cap_reports_failure():
    """test_algorithms.py:124-136: a zero column breaks every pass down on an
    exact-zero pivot; each retries once, to the cap of 4."""
    cq = _cq()
    cfg = cq.AlgoConfig(max_iter=4)
    res = cq.rs_chol_qr(_dev(_gen(150, 6, 1.0, 4, zero=[2])), cfg)
    assert not res.success
    assert res.iterations == 4
    assert res.orth_error is not None and res.orth_error >= cfg.tol
    assert res.shift_attempts == [1, 1, 1, 1]
    assert res.decision_margins[0] == 0.0          # structural, not rounding


def test_shift_attempt_limit_is_enforced():
    """test_algorithms.py:139-149: a basis violating orthonormality makes the
    deflated Gramian negative definite; the limit of 5 attempts raises."""
    cq = _cq()
    basis = _dev(2.0 * np.eye(4, 1))
    incoming = _dev(np.eye(4, 1))
    with pytest.raises(cq.ShiftAttemptLimitError) as info:
        cq.chol_qr_update(basis, 2.0 * np.eye(1), incoming, cq.AlgoConfig(max_shift_attempts=5))
    assert info.value.attempts == 5
    assert info.value.last_shift > 0


def test_tol_policy_roundoff():
    """test_algorithms.py:152-166: the roundoff floor runs to the cap."""
    cq = _cq()
    cfg = cq.AlgoConfig(tol_policy="roundoff")
    assert cfg.effective_tol(4) == pytest.approx(2.0 * U)
    res = cq.rs_chol_qr(_dev(_gen(200, 8, 2.0, 5)), cfg)
    assert res.iterations == cfg.max_iter and not res.success
    assert res.orth_error <= 20 * U * math.sqrt(8)
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= 20 * U * math.sqrt(8)


# ---------------------------------------------------------------- test_update_panel.py
def _basis(m=400, q=6, seed=0):
    cq = _cq()
    return cq.rs_chol_qr(_dev(_gen(m, q, 2.0, seed)))


def test_update_extends_an_existing_basis():
    """test_update_panel.py:48-63."""
    cq = _cq()
    base = _basis()
    incoming = _gen(400, 4, 3.0, 2)
    res = cq.chol_qr_update(base.q, base.r, _dev(incoming))
    assert res.success and res.q.ncols == 10 and res.r.shape == (10, 10)
    np.testing.assert_array_equal(res.r[6:, :6], np.zeros((4, 6)))
    np.testing.assert_array_equal(res.r[:6, :6], base.r)
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(10) * 1e-13
    composite = _dev(np.hstack([base.q.to_numpy() @ base.r, incoming]))
    assert cq.reconstruction_residual(composite, res.q, res.r, norm="frobenius") <= 1e-12


def test_update_duplicate_basis_column_takes_the_shift_path():
    """test_update_panel.py:66-78: an incoming column copying a basis column
    makes the deflated Gramian exactly singular; the pinned case needs the
    recomputed shift (clamped at 2u) and one x10 escalation."""
    cq = _cq()
    import parity as P
    from oracle import cholqr_oracle as co

    base = _basis(m=2000, q=5, seed=0)
    incoming = _dev(base.q.to_numpy()[:, [0]])
    res, trace = P.traced(cq.chol_qr_update, base.q, base.r, incoming)
    assert not isinstance(res, Exception), res
    assert res.success
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(6) * 1e-13
    # The deflated Gramian x = q.q - (Q_in^T q)^2 is 1 - 1 in exact arithmetic:
    # its computed value is -(||q||^2 - 1) rounded, i.e. the sign of the basis
    # column's norm defect as the device's dot products round it.  The replay
    # shows the oracle takes the device's branch on the device's own Gramian.
    rep = P.replay_iterated(trace, res, co.default_cfg(), "update")
    assert rep.passes == res.iterations
    g, bt = P._device_x(trace[0])
    x = co._deflated_from(g, bt)
    assert abs(x[0, 0]) <= 100 * U, x
    if res.shift_attempts[0] > 0:
        # the pinned path: recomputed shift clamped at 2u, then x10 escalations
        n = res.shift_attempts[0]
        assert res.shifts_applied[0] == 2.0 * U
        for s0, s1 in zip(res.shifts_applied[: n - 1], res.shifts_applied[1:n]):
            assert s1 / s0 == pytest.approx(10.0, rel=1e-9)


def test_update_duplicate_column_pinned_escalation():
    """The reference's pinned outcome of the duplicate-column case -- attempts
    [2, ...], shifts [2u, 20u] -- reproduced on a basis whose first column has a
    norm defect of +10u, so the deflated Gramian is about -10u (and -10u + 2u <
    0 < -10u + 20u) whichever way the dot products round
    (test_update_panel.py:66-78)."""
    cq = _cq()
    rng = np.random.default_rng(0)
    m = 2048
    q = np.linalg.qr(rng.standard_normal((m, 5)))[0]
    # scale column 0 so that ||q0||^2 = 1 + 10u, well above the dot products' rounding
    q[:, 0] *= math.sqrt(1.0 + 10 * U) / np.linalg.norm(q[:, 0])
    base = _dev(q)
    res = cq.chol_qr_update(base, np.eye(5), _dev(q[:, [0]]))
    assert res.shift_attempts[0] == 2, res.shift_attempts
    assert res.shifts_applied[0] == 2.0 * U
    assert res.shifts_applied[1] / res.shifts_applied[0] == pytest.approx(10.0, rel=1e-9)


def test_update_shift_width_selects_the_formula_width():
    """test_update_panel.py:81-99: from an empty basis the "existing" width is
    0, so the first shift is exactly 2u; "incoming" uses the block width."""
    cq = _cq()
    block = _gen(300, 4, 1.0, 3, zero=[1])
    a = _dev(block)
    empty = cq.CudaVectorArray.zeros(a.space, 0)
    existing = cq.chol_qr_update(empty, np.zeros((0, 0)), a,
                                 cq.AlgoConfig(max_iter=1, update_shift_width="existing"))
    incoming = cq.chol_qr_update(empty, np.zeros((0, 0)), a,
                                 cq.AlgoConfig(max_iter=1, update_shift_width="incoming"))
    assert existing.shifts_applied[0] == 2.0 * U
    assert incoming.shifts_applied[0] > 100 * existing.shifts_applied[0]
    assert incoming.shifts_applied[0] == pytest.approx(
        cq.compute_shift(300, 4, float(np.linalg.norm(block.T @ block, 2))), rel=0.05)


def test_update_validates_inputs():
    """test_update_panel.py:100-110."""
    cq = _cq()
    base = _basis()
    incoming = _dev(_gen(400, 2, 1.0, 4))
    with pytest.raises(ValueError, match="r_in must be"):
        cq.chol_qr_update(base.q, np.eye(5), incoming)
    with pytest.raises(ValueError, match="space mismatch"):
        cq.chol_qr_update(base.q, base.r, _dev(_gen(401, 2, 1.0, 4)))
    with pytest.raises(ValueError, match="at least one new column"):
        cq.chol_qr_update(base.q, base.r, cq.CudaVectorArray.zeros(incoming.space, 0))


@pytest.mark.parametrize("r_panels", [2, 3, 5, 10])
def test_panel_scheme_quality(r_panels):
    """test_update_panel.py:124-134."""
    cq = _cq()
    a = _dev(_gen(500, 10, 10.0, 5))
    res = cq.pn_chol_qr(a, r_panels)
    assert res.success and res.q.ncols == 10
    assert len(res.panel_profiles) == r_panels
    assert res.iterations == sum(p.outer for p in res.panel_profiles)
    assert cq.loss_of_orthogonality(res.q, norm="frobenius") <= math.sqrt(10) * 1e-13
    assert cq.reconstruction_residual(a, res.q, res.r, norm="frobenius") <= 1e-12
    np.testing.assert_array_equal(np.tril(res.r, -1), 0.0)


def test_panel_scheme_continues_past_a_capped_panel():
    """test_update_panel.py:137-150."""
    cq = _cq()
    a = _dev(_gen(300, 8, 2.0, 6, zero=[1]))
    cfg = cq.AlgoConfig(max_iter=3, update_shift_width="incoming")
    res = cq.pn_chol_qr(a, 2, cfg)
    assert not res.success
    assert res.q.ncols == 8
    assert len(res.panel_profiles) == 2
    assert res.panel_profiles[0].outer == 3
    assert res.panel_profiles[1].outer >= 1


def test_panel_count_bounds_are_enforced():
    """test_update_panel.py:165-170."""
    cq = _cq()
    a = _dev(_gen(50, 4, 1.0, 8))
    with pytest.raises(ValueError):
        cq.pn_chol_qr(a, 0)
    with pytest.raises(ValueError):
        cq.pn_chol_qr(a, 5)


def test_panel_breakdown_is_annotated_with_the_panel_index():
    """test_update_panel.py:153-162."""
    cq = _cq()
    blk = _gen(100, 6, 1.0, 7)
    blk[0, 4] = np.nan
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(cq.ShiftAttemptLimitError) as info:
            cq.pn_chol_qr(_dev(blk), 2, cq.AlgoConfig(max_shift_attempts=3))
    assert info.value.panel_index == 1
