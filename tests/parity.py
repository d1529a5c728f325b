"""Decision-parity rule shared by the parity tests.

The iterated schemes (rs_chol_qr, is_chol_qr, chol_qr_update; reference
algorithms.py:247-458) take two kinds of decision per outer iteration i:

* stop or not: ||X_i - I||_F < tol (converged), or the iteration cap;
* the branch of the pass: the plain factorization held (0 shifted attempts)
  or broke down, and then how many shifted attempts it took and with which
  shifts (algorithms.py:295-317, 369-397).

Both runs' decisions are compared pass by pass.  Where the two runs took the
SAME branch the decision is compared in full: shift_attempts exactly and the
shifts applied within 1e-6 relative (the first shift of a pass comes from the
norm estimate of the Gramian, which is well conditioned; escalations are x10
of it).  The comparison stops only where the two runs took DIFFERENT branches,
and that is allowed only when the deciding quantity sat at the rounding level
in at least one run:

* a breakdown decision: the signed relative pivot of the pass's first attempt
  (min Schur diagonal / max diag X) has |margin| <= 100 k u.  A NaN pivot
  (non-finite data) is never rounding-determined.  An exact-zero pivot is
  rounding-level too unless X's diagonal entry at that pivot is itself zero (a
  zero column): s = x_jj - r_j.r_j is a difference of two numbers near x_jj,
  so a pivot below ulp(x_jj) comes out as exactly 0.0 in an implementation
  that rounds the dot product first and as a tiny non-zero value in one that
  fuses it (measured: the golden rs_300x10_c16_s1 pass 1 has s = 0.0 at
  pivot 9 with x_99 = 0.69 in the reference, +1.1e-18 relative on the device).
  The replay below, which sees X, tells the two apart;
* a convergence decision: ||X - I||_F within [tol/100, 100 tol] in either run
  (after a pass it is itself ~kappa^2 u rounding noise of the previous Q).

Two refinements, both measured on the golden panel cases:

* the shifts of an update pass are compared within max(1e-6, 100 u r), r =
  max diag G / max |diag X| of the deflated Gramian X = G - Bt^T Bt (from the
  oracle): the deflation cancels r-fold, so X -- and the norm estimate and
  shift taken from it -- carries a relative rounding error of ~u r in any
  implementation (pn_2000x64_c12_s0_r4, panel 4: r ~ 1e10, the two shifts
  differ by 3.7e-6);
* the number of x10 escalations after a failed shifted attempt may differ:
  an escalation only happens when the shift sits below the Gramian's own
  rounding-level negative eigenvalue (the 2u clamp of an empty basis), and
  how many decades that noise spans is itself rounding (pn_500x10_c10_s5_r1:
  19 escalations on the device, 21 in the reference).  The first shift must
  still agree and every later one must be the x10 ladder above it.

A third, from the extended randomised sweep: for an update pass the breakdown
band is 100 (k + q) u, q the basis width -- every entry of the deflated
Gramian G - Bt^T Bt carries the rounding of a q-term dot product on top of the
factorization's own k-term ones, and the device's factor kernel and the
oracle order those sums differently (sweep case 5264, 323 x 64, kappa 1e14,
32-column basis: on the SAME G and Bt the oracle's plain attempt breaks down
at a relative pivot of -5.8e-13 = 164 k u where the device's holds).

Any other difference fails the test.  The compare functions return a record
with how many decisions were compared, so each test can assert its count.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

U = 1.11e-16


def fragile_margin(margin, k):
    """True when a breakdown decision with this signed relative pivot is
    rounding-determined: finite and within 100 k u of zero."""
    if margin is None:
        return False
    margin = float(margin)
    if math.isnan(margin):
        return False
    return abs(margin) <= 100 * k * U


def robust_margin(margin, k):
    """The complement of fragile_margin (kept for the single-shot tests)."""
    return not fragile_margin(margin, k)


def fragile_conv(tol, *errs):
    """True when a converged-or-not decision may be rounding-determined: one
    of the runs' ||X - I||_F lies within two decades of tol."""
    return any(e is not None and not math.isnan(e) and tol / 100 <= e <= 100 * tol for e in errs)


@dataclass
class Compared:
    decisions: int          # pass-branch decisions compared (and equal)
    shifted: int            # of which both runs broke down (shifts compared)
    stops: int              # stop decisions compared (and equal)
    full: bool              # every decision of both runs was compared
    reason: str = ""        # why the comparison ended early (rounding-level divergence)


def _at(seq, i):
    seq = list(seq or [])
    return seq[i] if i < len(seq) else None


def compare_iterated(mine, ref, k, tol):
    """Compare the two runs' decisions pass by pass (module docstring).
    Raises AssertionError on a robust difference; returns a Compared."""
    shifts_m = list(mine.shifts_applied)
    shifts_r = list(ref.shifts_applied)
    pm = pr = 0
    dec = shifted = stops = 0
    i = 0
    while True:
        stop_m = i >= mine.iterations
        stop_r = i >= ref.iterations
        err_m = _at(getattr(mine, "err_history", None), i)
        err_r = _at(getattr(ref, "err_history", None), i)
        if stop_m or stop_r:
            if stop_m and stop_r:
                if mine.success != ref.success:
                    # one converged on its last allowed pass, the other was capped
                    assert fragile_conv(tol, err_m, err_r), (i, mine.success, ref.success, err_m, err_r)
                    return Compared(dec, shifted, stops, False, f"cap vs converged at pass {i}")
                return Compared(dec, shifted, stops + 1, True)
            assert fragile_conv(tol, err_m, err_r), (
                f"stop decision differs at pass {i}: mine {mine.iterations} passes, ref {ref.iterations}",
                err_m, err_r)
            return Compared(dec, shifted, stops, False, f"stop at pass {i} (err {err_m} / {err_r})")
        stops += 1
        a_m = mine.shift_attempts[i]
        a_r = ref.shift_attempts[i]
        if (a_m > 0) != (a_r > 0):
            dm_m = _at(mine.decision_margins, i)
            dm_r = _at(ref.decision_margins, i)
            assert fragile_margin(dm_m, k) or fragile_margin(dm_r, k), (
                f"breakdown decision differs at pass {i}", mine.shift_attempts, ref.shift_attempts, dm_m, dm_r)
            return Compared(dec, shifted, stops, False, f"branch at pass {i} (margins {dm_m} / {dm_r})")
        ratio = _at(getattr(ref, "deflation_ratios", None), i) or 1.0
        rtol = max(1e-6, 100 * U * ratio)
        if a_m != a_r:
            # both broke down; the escalation count differs: allowed only as a
            # rounding-level ladder (module docstring)
            assert max(a_m, a_r) >= 2, (f"shift attempts differ at pass {i}", mine.shift_attempts,
                                        ref.shift_attempts)
            np.testing.assert_allclose(shifts_m[pm], shifts_r[pr], rtol=rtol, err_msg=f"first shift of pass {i}")
            for sh, a in ((shifts_m[pm:pm + a_m], a_m), (shifts_r[pr:pr + a_r], a_r)):
                for s0, s1 in zip(sh[:-1], sh[1:]):
                    assert s1 == pytest_approx_ratio(s0, s1), (f"pass {i}: not a x10 ladder", sh)
            return Compared(dec, shifted, stops, False, f"escalations at pass {i} ({a_m} / {a_r})")
        if a_m:
            np.testing.assert_allclose(shifts_m[pm:pm + a_m], shifts_r[pr:pr + a_r], rtol=rtol,
                                       err_msg=f"shifts of pass {i}")
            shifted += 1
        pm += a_m
        pr += a_r
        dec += 1
        i += 1


def pytest_approx_ratio(s0, s1, esc=10.0):
    """s1 when s1 / s0 is the escalation factor to 1e-12, else None."""
    return s1 if abs(s1 / s0 - esc) <= 1e-12 * esc else None


def compare_single(res_m, exc_m, res_r, exc_r, k, m=None):
    """Fixed schedules (chol_qr, chol_qr2, s_chol_qr3): the decision is
    breakdown or not.  Both raising (or both not) is a match; otherwise the
    deciding pivot must be rounding-level in the run that knows it.  Returns
    True when the two runs agree.  With the row count `m` the band counts the
    Gramian's own rounding as well: each entry is an m-term dot product summed
    in a different order by each implementation (~sqrt(m) u), so the band is
    100 (k + sqrt(m)) u (sweep case 13343, chol_qr2 on 1200 x 3 at kappa 1e10:
    relative pivots -2.7e-13 on the device, +1.5e-13 in the oracle)."""
    if m is not None:
        k = k + math.sqrt(m)
    if (exc_m is None) == (exc_r is None):
        if exc_m is not None:
            assert exc_m.pivot_index >= 0 and exc_r.pivot_index >= 0
        return True
    if exc_m is not None:
        margins = [getattr(exc_m, "margin", None)] + list(getattr(res_r, "pivot_margins", []) or [])
    else:
        margins = [getattr(exc_r, "margin", None)] + list(getattr(res_m, "pivot_margins", []) or [])
    assert any(fragile_margin(x, k) for x in margins), ("breakdown differs", exc_m, exc_r, margins)
    return False


def within10(mine, ref, k, tol=None):
    """mine <= 10 x ref (floored at 10 u sqrt(k)); after a rounding-determined
    convergence decision both runs stopped on ||X - I||_F < tol, so tol also
    bounds the comparison then."""
    floor = 10 * U * math.sqrt(k)
    if tol is not None:
        floor = max(floor, tol)
    return mine <= 10 * max(ref, floor)


class Record:
    """A golden-vector record (tests/golden/golden.json, written by the
    unmodified reference) in the shape compare_iterated reads.  The reference's
    QRResult carries no margins or per-pass errors, so a divergence from it is
    accepted only where the other run's own margin was rounding-level."""

    def __init__(self, case):
        self.iterations = case["iterations"]
        self.shift_attempts = list(case["attempts"])
        self.shifts_applied = list(case["shifts"])
        self.success = case["success"]
        self.err_history = [None] * self.iterations + [case.get("orth_error")]
        self.decision_margins = []


# ----------------------------------------------------------------------------
# Decision-stage replay: the oracle's k x k stage on the device's own Gramians
# ----------------------------------------------------------------------------
#
# The trajectory comparison above stops at the first rounding-level divergence,
# because from there on the two runs factor different Gramians.  The replay
# removes that coupling: the device records the exact k x k inputs of every
# factor call (DeviceContext.trace), and the oracle's decision stage
# (algorithms.py:295-317, 341-349, 369-397; kernels.py:61-194) runs on those
# same bits.  Every pass is then compared independently: ||X - I||_F, the stop
# decision, the branch, the attempt count and the shifts.  The only remaining
# source of difference is the arithmetic order inside the Cholesky and the
# power iteration, so a branch may differ only where the oracle's own pivot on
# the same X is rounding-level.


@dataclass
class Replayed:
    passes: int = 0        # passes whose decisions were replayed
    shifted: int = 0       # of which shifted (attempts and shifts compared)
    fragile: int = 0       # branch differences at a rounding-level pivot (allowed)


def _sym_from_lower(g):
    g = np.asarray(g, dtype=float)
    low = np.tril(g)
    return low + np.tril(g, -1).T


def _device_x(entry):
    """The k x k matrix the device factor call read: G (column-major, lower
    triangle) and, for updates, Bt (q x p)."""
    g = entry["G"].cpu().numpy().T      # column-major device buffer -> row-major
    bt = entry["Bt"].cpu().numpy().T if entry["Bt"] is not None else None   # (p, q) torch -> q x p
    return _sym_from_lower(g), bt


def replay_iterated(trace, mine, cfg, kind="rs"):
    """Replay rs_chol_qr / chol_qr_update decisions on the device's Gramians.
    `trace` holds the entries of this run's factor calls in order; `cfg` is the
    oracle config dict.  Returns a Replayed; AssertionError on a robust
    difference."""
    import warnings

    from oracle import cholqr_oracle as co

    out = Replayed()
    pm = 0
    shifts_m = list(mine.shifts_applied)
    for i in range(mine.iterations + 1):
        if i >= len(trace):
            break
        e = trace[i]
        g, bt = _device_x(e)
        k = g.shape[0]
        # width of the rounding noise in the factored matrix: its own k, plus, for a
        # deflated Gramian G - Bt^T Bt, the q-term dot products of the deflation (the
        # device's factor kernel and the oracle order them differently)
        kn = k
        if kind == "update" and bt is not None and bt.size:
            x = co._deflated_from(g, bt)
            top = float(np.max(np.diag(g))) if g.size else None
            kn = k + bt.shape[0]
        else:
            x = g
            top = None
        tol = e["tol"]
        err = co.identity_distance(x)
        err_m = mine.err_history[i] if i < len(mine.err_history) else None
        if err_m is not None:
            assert abs(err_m - err) <= 1e-10 * err + 1e-300, (i, err_m, err)
        stop_o = err < tol or i == cfg["max_iter"]     # converged, or the cap (algorithms.py:341-343)
        stop_m = i >= mine.iterations
        if stop_o != stop_m:
            assert abs(err - tol) <= 1e-10 * tol, (f"stop decision at pass {i}", err, tol, mine.iterations)
            out.fragile += 1
            break
        if stop_m:
            assert mine.success == (err < tol), (i, mine.success, err, tol)
            break
        m, width = e["m_global"], e["width"]
        a_m = mine.shift_attempts[i]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if kind == "update":
                _, dm, exc = co._attempt(co._with_shift(x, 0.0), top)
                shifts_o = []
                try:
                    _, a_o, _ = co._update_attempts(x, m, width, cfg, shifts_o)
                except co.OracleShiftLimit:
                    a_o = None
            else:
                rk, dm, exc = co._attempt(x)
                shifts_o = []
                if rk is not None:
                    a_o = 0
                else:
                    try:
                        _, a_o, _ = co._recomputed_shift_attempts(x, m, width, cfg, shifts_o)
                    except co.OracleShiftLimit:
                        a_o = None
        out.passes += 1
        structural = exc is not None and x[exc.pivot_index, exc.pivot_index] == 0.0   # a zero column
        if a_o is None or (a_o > 0) != (a_m > 0) or a_o != a_m:
            if (a_o is not None and (a_o > 0) != (a_m > 0)) and fragile_margin(dm, kn) and not structural:
                out.fragile += 1
                pm += a_m
                continue
            raise AssertionError((f"pass {i}: device attempts {a_m}, oracle on the device Gramian {a_o}", dm,
                                  shifts_m[pm:pm + a_m], shifts_o))
        if a_m:
            np.testing.assert_allclose(shifts_m[pm:pm + a_m], shifts_o, rtol=1e-6, err_msg=f"shifts of pass {i}")
            out.shifted += 1
        pm += a_m
    return out


def traced(fn, *args, **kw):
    """Run a device algorithm with the factor-input trace on; returns
    (result or exception, trace)."""
    from paper_2507_07788_b200._device import ctx

    cx = ctx()
    cx.trace = []
    try:
        try:
            res = fn(*args, **kw)
        except Exception as exc:   # noqa: BLE001 -- returned to the caller
            res = exc
    finally:
        tr, cx.trace = cx.trace, None
    return res, tr


def split_panels(res, tols):
    """Per-panel views of a pn_chol_qr result (algorithms.py:470-505), in the
    shape compare_iterated reads: panel i took outer_i passes (its profile),
    its slice of shift_attempts / shifts / decision margins, and outer_i + 1
    ||X - I||_F values; it converged when the last one is below tols[i]."""
    import types

    out = []
    pa = ps = pe = pd = 0
    for prof, tol in zip(res.panel_profiles, tols):
        outer = prof[0] if isinstance(prof, tuple) else prof.outer
        att = list(res.shift_attempts[pa:pa + outer])
        nsh = sum(att)
        errs = list(res.err_history[pe:pe + outer + 1])
        out.append(types.SimpleNamespace(
            iterations=outer, shift_attempts=att, shifts_applied=list(res.shifts_applied[ps:ps + nsh]),
            success=bool(errs and errs[-1] < tol), err_history=errs,
            decision_margins=list(res.decision_margins[pd:pd + outer]),
            deflation_ratios=list(getattr(res, "deflation_ratios", [])[pd:pd + outer])))
        pa += outer
        ps += nsh
        pe += outer + 1
        pd += outer
    return out
