"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (`oracle/cholqr_oracle.py`) is a NumPy restatement of the
reference's algorithms; `tests/golden/make_golden.py` ran the UNMODIFIED
reference on the same inputs.  On the same NumPy/OpenBLAS stack the oracle
must reproduce the reference's decisions exactly and its factors to rounding
(in practice bitwise).  CPU only.
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import pytest

from oracle import cholqr_oracle as co
from oracle import matgen_oracle as mg

from conftest import Golden, oracle_cfg

G = Golden()
SINGLE = [c for c in G.meta["cases"]
          if c["algo"] in ("rs_chol_qr", "is_chol_qr", "s_chol_qr3", "chol_qr", "chol_qr2")]
UPDATE = [c for c in G.meta["cases"] if c["algo"] == "chol_qr_update"]


def _run_single(case, a):
    algo = case["algo"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if algo == "rs_chol_qr":
            return co.rs_chol_qr(a, oracle_cfg(case))
        if algo == "is_chol_qr":
            return co.is_chol_qr(a, oracle_cfg(case))
        if algo == "s_chol_qr3":
            return co.s_chol_qr3(a)
        if algo == "chol_qr":
            return co.chol_qr(a)
        return co.chol_qr2(a)


@pytest.mark.parametrize("case", SINGLE, ids=[c["name"] for c in SINGLE])
def test_oracle_single_input_matches_reference(case):
    a = G.input(case)
    if "exception" in case:
        with pytest.raises(co.OracleBreakdown) as info:
            _run_single(case, a)
        assert info.value.pivot_index == case["pivot_index"]
        return
    res = _run_single(case, a)
    assert res.iterations == case["iterations"]
    assert res.shift_attempts == case["attempts"]
    assert res.success == case["success"]
    np.testing.assert_allclose(res.shifts_applied, case["shifts"], rtol=1e-12, atol=0)
    r_ref = G.r(case)
    scale = max(np.max(np.abs(r_ref)), 1e-300)
    assert np.max(np.abs(res.r - r_ref)) <= 1e-12 * scale
    if case.get("orth_error") is not None:
        assert res.orth_error == pytest.approx(case["orth_error"], rel=1e-6, abs=1e-17)
    if "loo" in case:
        assert co.loo_fro(res.q) == pytest.approx(case["loo"], rel=1e-6, abs=1e-18)


@pytest.mark.parametrize("case", UPDATE, ids=[c["name"] for c in UPDATE])
def test_oracle_update_matches_reference(case):
    a_new = G.arrays[case["name"] + "__in"]
    q_in = G.arrays[case["name"] + "__qin"]
    r_in = G.arrays[case["name"] + "__rin"]
    cfg = oracle_cfg(case)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if "exception" in case:
            with pytest.raises(co.OracleShiftLimit) as info:
                co.chol_qr_update(q_in, r_in, a_new, cfg)
            assert info.value.attempts == case["attempts"]
            if case["last_shift"] is None or (isinstance(case["last_shift"], float) and math.isnan(case["last_shift"])):
                assert math.isnan(info.value.last_shift)
            else:
                assert info.value.last_shift == pytest.approx(case["last_shift"], rel=1e-12)
            return
        res = co.chol_qr_update(q_in, r_in, a_new, cfg)
    assert res.iterations == case["iterations"]
    assert res.shift_attempts == case["attempts"]
    assert res.success == case["success"]
    np.testing.assert_allclose(res.shifts_applied, case["shifts"], rtol=1e-12)
    r_ref = G.r(case)
    scale = max(np.max(np.abs(r_ref)), 1e-300)
    assert np.max(np.abs(res.r - r_ref)) <= 1e-12 * scale
    k = q_in.shape[1]
    np.testing.assert_array_equal(res.r[k:, :k], 0.0)
    np.testing.assert_array_equal(res.r[:k, :k], r_in)


def test_matgen_matches_reference():
    for name, (m, n, x, s) in {"matgen_300_10_c6_s0": (300, 10, 6.0, 0),
                               "matgen_50_1_c0_s0": (50, 1, 0.0, 0)}.items():
        np.testing.assert_array_equal(mg.generate(m, n, x, s), G.arrays[name])


def test_kernel_known_answers():
    k = G.meta["kernels"]
    np.testing.assert_array_equal(co.cholesky_upper(np.array([[4.0, 2.0], [2.0, 5.0]])), k["chol_4252"])
    with pytest.raises(co.OracleBreakdown) as info:
        co.cholesky_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert [info.value.pivot_index, info.value.pivot_value] == k["chol_1221"]
    assert co.shift_value(300, 10, 1.0) == k["shift_300_10_1"]
    assert co.shift_value(300, 10, 0.0) == k["shift_clamp"]
    spd = G.arrays["kern_spd8"]
    np.testing.assert_array_equal(co.cholesky_upper(spd), G.arrays["kern_spd8_chol"])
    np.testing.assert_array_equal(co.tri_inverse(co.cholesky_upper(spd)), G.arrays["kern_spd8_inv"])
    assert co.spectral_estimate(spd)[0] == k["spd8_est"]


def test_oracle_nan_pivot_is_breakdown():
    x = np.eye(2)
    x[1, 1] = np.nan
    with pytest.raises(co.OracleBreakdown):
        co.cholesky_upper(x)


def test_decision_rule_compares_every_golden_decision():
    """The decision rule of tests/parity.py, applied to the oracle against the
    reference's own records, compares every decision of every iterated golden
    case: all 42 shifted iterations (shift attempts exact, shifts 1e-6) and the
    stop decisions.  The GPU tests apply the same rule to the device path."""
    import parity as P

    shifted = total = 0
    for case in SINGLE:
        if case["algo"] not in ("rs_chol_qr", "is_chol_qr") or "exception" in case:
            continue
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = _run_single(case, G.input(case))
        k = G.input(case).shape[1]
        tol = co.effective_tol(oracle_cfg(case), k)
        cmp = P.compare_iterated(res, P.Record(case), k, tol)
        assert cmp.full, (case["name"], cmp)
        assert cmp.decisions == case["iterations"]
        shifted += cmp.shifted
        total += sum(1 for a in case["attempts"] if a > 0)
    assert shifted == total == 42


def test_decision_rule_rejects_robust_differences():
    """A robust branch difference, a shift off by 1e-5, a different attempt
    count and a NaN pivot all fail the rule; a rounding-level margin passes."""
    import types

    import parity as P

    def run(att, shifts, dms, its=None, ok=True):
        its = len(att) if its is None else its
        return types.SimpleNamespace(iterations=its, shift_attempts=att, shifts_applied=shifts, success=ok,
                                     err_history=[1.0] * its + [1e-16], decision_margins=dms)

    ref = run([1, 0], [1e-10], [-1e-3, 0.5])
    assert P.compare_iterated(run([1, 0], [1e-10 * (1 + 1e-9)], [-1e-3, 0.5]), ref, 8, 1e-13).full
    with pytest.raises(AssertionError):
        P.compare_iterated(run([0, 0], [], [1e-3, 0.5]), ref, 8, 1e-13)
    with pytest.raises(AssertionError):
        P.compare_iterated(run([1, 0], [1.00001e-10], [-1e-3, 0.5]), ref, 8, 1e-13)
    with pytest.raises(AssertionError):      # an escalation that is not the x10 ladder
        P.compare_iterated(run([2, 0], [1e-10, 3e-10], [-1e-3, 0.5]), ref, 8, 1e-13)
    with pytest.raises(AssertionError):      # a ladder from a different first shift
        P.compare_iterated(run([2, 0], [2e-10, 2e-9], [-1e-3, 0.5]), ref, 8, 1e-13)
    ladder = P.compare_iterated(run([2, 0], [1e-10, 1e-9], [-1e-3, 0.5]), ref, 8, 1e-13)
    assert not ladder.full and "escalations" in ladder.reason
    nan = run([1, 0], [1e-10], [float("nan"), 0.5])
    with pytest.raises(AssertionError):
        P.compare_iterated(run([0, 0], [], [float("nan"), 0.5]), nan, 8, 1e-13)
    fragile = run([1, 0], [1e-10], [-1e-16, 0.5])
    cmp = P.compare_iterated(run([0, 0], [], [1e-16, 0.5]), fragile, 8, 1e-13)
    assert not cmp.full and cmp.decisions == 0


PANEL = [c for c in G.meta["cases"] if c["algo"] == "pn_chol_qr"]


@pytest.mark.parametrize("case", PANEL, ids=[c["name"] for c in PANEL])
def test_oracle_panel_scheme_matches_reference(case):
    """Alg. 3 (algorithms.py:470-505) against the unmodified reference: per-panel
    profiles, attempts, shifts, R, and the panel index of an exception."""
    a = G.input(case)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if "exception" in case:
            with pytest.raises(co.OracleShiftLimit) as info:
                co.pn_chol_qr(a, case["r_panels"], oracle_cfg(case))
            assert info.value.panel_index == case["panel_index"]
            assert info.value.attempts == case["attempts"]
            return
        res = co.pn_chol_qr(a, case["r_panels"], oracle_cfg(case))
    assert res.iterations == case["iterations"]
    assert res.shift_attempts == case["attempts"]
    assert res.success == case["success"]
    assert [None if p is None else [p[0], list(p[1])] for p in res.panel_profiles] == case["panel_profiles"]
    np.testing.assert_allclose(res.shifts_applied, case["shifts"], rtol=1e-12)
    r_ref = G.r(case)
    assert np.max(np.abs(res.r - r_ref)) <= 1e-12 * max(np.max(np.abs(r_ref)), 1e-300)
    if "loo" in case:
        assert co.loo_fro(res.q) == pytest.approx(case["loo"], rel=1e-6, abs=1e-18)


def test_oracle_panel_bounds():
    with pytest.raises(ValueError):
        co.pn_chol_qr(np.ones((50, 4)), 0)
    with pytest.raises(ValueError):
        co.pn_chol_qr(np.ones((50, 4)), 5)
