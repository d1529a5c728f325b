"""The reference's own unit / acceptance checks, run on the device backend
(reference tests/test_metrics.py, tests/test_acceptance.py criterion 7,
tests/test_algorithms.py bookkeeping and Householder checks,
tests/test_varray.py backend rules).  GPU only."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cq():
    import paper_2507_07788_b200 as cq

    return cq


def _dev(block):
    return _cq().CudaVectorArray.from_numpy(np.asarray(block, dtype=float))


# ---------------------------------------------------------------- metrics (test_metrics.py)
def test_loss_of_orthogonality_hand_oracle():
    cq = _cq()
    e1 = np.zeros((4, 1))
    e1[0, 0] = 1.0
    q = _dev(np.hstack([e1, e1]))   # I - Q^T Q = [[0, -1], [-1, 0]]
    assert cq.loss_of_orthogonality(q) == pytest.approx(1.0, abs=1e-15)
    assert cq.loss_of_orthogonality(q, norm="frobenius") == pytest.approx(np.sqrt(2.0), rel=1e-15)
    assert cq.loss_of_orthogonality(_dev(np.eye(5, 3))) == 0.0


def test_exact_factorization_scores_zero():
    cq = _cq()
    qb = np.eye(6, 2)
    r = np.array([[2.0, 1.0], [0.0, 3.0]])
    a, q = _dev(qb @ r), _dev(qb)
    assert cq.reconstruction_residual(a, q, r) == 0.0
    assert cq.cholesky_residual(a, r) == pytest.approx(0.0, abs=1e-15)


def test_metrics_agree_with_dense_norms():
    cq = _cq()
    block, _ = cq.generate_host(cq.MatrixSpec(80, 6, 3.0, seed=0))
    qb, r = np.linalg.qr(block)
    a, q = _dev(block), _dev(qb)
    assert cq.loss_of_orthogonality(q) == pytest.approx(np.linalg.norm(np.eye(6) - qb.T @ qb, 2),
                                                        rel=1e-6, abs=1e-15)
    assert cq.reconstruction_residual(a, q, r) == pytest.approx(
        np.linalg.norm(block - qb @ r, 2) / np.linalg.norm(block, 2), rel=1e-2, abs=1e-14)
    assert cq.cholesky_residual(a, r) == pytest.approx(
        np.linalg.norm(block.T @ block - r.T @ r, 2) / np.linalg.norm(block, 2) ** 2, rel=1e-2, abs=1e-16)
    rep = cq.quality_report(a, q, r)
    assert (rep.loo, rep.rrr, rep.rcr) == (cq.loss_of_orthogonality(q), cq.reconstruction_residual(a, q, r),
                                           cq.cholesky_residual(a, r))
    with pytest.raises(ValueError):
        cq.loss_of_orthogonality(q, norm="nuclear")


def test_metrics_are_pure():
    cq = _cq()
    block, _ = cq.generate_host(cq.MatrixSpec(60, 4, 2.0, seed=3))
    qb, r = np.linalg.qr(block)
    a, q = _dev(block), _dev(qb)
    ra = r.copy()
    cq.quality_report(a, q, r)
    np.testing.assert_array_equal(a.to_numpy(), block)
    np.testing.assert_array_equal(q.to_numpy(), qb)
    np.testing.assert_array_equal(r, ra)


# ---------------------------------------------------------------- acceptance criterion 7
def test_degenerate_single_column():
    cq = _cq()
    a, _ = cq.generate(cq.MatrixSpec(50, 1, 0.0, seed=0))
    res = cq.rs_chol_qr(a)
    assert res.success and res.q.ncols == 1
    assert cq.loss_of_orthogonality(res.q) <= 1e-13
    assert cq.reconstruction_residual(a, res.q, res.r) <= 1e-12


def test_degenerate_zero_column_runs_to_cap():
    cq = _cq()
    block, _ = cq.generate_host(cq.MatrixSpec(80, 6, 2.0, seed=1))
    block[:, 3] = 0.0
    res = cq.rs_chol_qr(_dev(block))
    assert not res.success
    assert res.shifts_applied
    assert res.iterations == cq.AlgoConfig().max_iter


def test_degenerate_scaled_orthogonal():
    cq = _cq()
    q0 = np.linalg.qr(np.random.default_rng(7).normal(size=(200, 12)))[0]
    res = cq.rs_chol_qr(_dev(2.0 * q0))
    assert res.iterations == 1 and not res.shifts_applied
    strict = cq.rs_chol_qr(_dev(q0))
    assert strict.iterations <= 1 and not strict.shifts_applied


# ---------------------------------------------------------------- test_algorithms.py
@pytest.mark.parametrize("cond", [0.0, 6.0, 12.0, 16.0])
def test_shift_bookkeeping(cond):
    """sum(shift_attempts) == len(shifts_applied) (test_algorithms.py:96-104)."""
    cq = _cq()
    a, _ = cq.generate(cq.MatrixSpec(300, 10, cond, seed=4))
    res = cq.rs_chol_qr(a)
    assert sum(res.shift_attempts) == len(res.shifts_applied)
    assert len(res.shift_attempts) == res.iterations


def test_r_matches_householder():
    """R vs Householder QR with the sign fixed, 1e-9 (test_algorithms.py:258-263)."""
    cq = _cq()
    block, _ = cq.generate_host(cq.MatrixSpec(500, 20, 4.0, seed=5))
    res = cq.rs_chol_qr(_dev(block))
    r_h = np.linalg.qr(block)[1]
    r_h = r_h * np.sign(np.diag(r_h))[:, None]
    assert np.max(np.abs(res.r - r_h)) <= 1e-9 * np.max(np.abs(r_h))


def test_cholqr_breaks_down_on_ill_conditioned():
    """Plain CholeskyQR / CholeskyQR2 at kappa = 1e9 break down in the reference
    (test_algorithms.py:58-63).  kappa^2 = 1e18 >> 1/u puts the deciding pivot
    at the rounding level, so per the parity rule a device
    run may also succeed -- but only with a margin inside the non-robust band."""
    cq = _cq()
    import parity as P

    for seed in (1, 2):   # seed 0 is the reference's own case, strict in test_gpu_contracts.py
        a, _ = cq.generate(cq.MatrixSpec(300, 10, 9.0, seed=seed))
        for fn in (cq.chol_qr, cq.chol_qr2):
            try:
                res = fn(a)
            except cq.CholeskyBreakdown as exc:
                assert exc.pivot_index >= 0
                continue
            assert not P.robust_margin(min(res.pivot_margins), 10), (fn.__name__, seed, res.pivot_margins)


def test_s_chol_qr3_applies_exactly_one_shift():
    cq = _cq()
    a, _ = cq.generate(cq.MatrixSpec(300, 10, 12.0, seed=1))
    res = cq.s_chol_qr3(a)
    assert len(res.shifts_applied) == 1 and res.iterations == 3


# ---------------------------------------------------------------- test_varray.py backend rules
def test_backend_mixing_and_ownership():
    cq = _cq()
    rng = np.random.default_rng(9)
    blk = rng.standard_normal((33, 4))
    a = _dev(blk)
    with pytest.raises((TypeError, AttributeError)):   # as varray.py:86-94 (space checked first)
        a.append(np.zeros((33, 1)))          # not a device array
    with pytest.raises(ValueError):
        a.append(_dev(np.zeros((34, 1))))    # space mismatch
    b = a.copy()
    b.axpy(1.0, a)                           # in place on the copy only
    np.testing.assert_array_equal(a.to_numpy(), blk)
    np.testing.assert_array_equal(b.to_numpy(), 2.0 * blk)
    c = a.copy([2, 0])
    np.testing.assert_array_equal(c.to_numpy(), blk[:, [2, 0]])
    g = a.gramian()
    assert isinstance(g, np.ndarray) and g.shape == (4, 4)
    np.testing.assert_array_equal(g, g.T)
