"""CPU oracle for the shifted Cholesky QR hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package's algorithms
(`/root/reference/pkg/src/cholqr`, arXiv 2507.07788).  It exists to check the
CUDA path, never to run it: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product package (`paper_2507_07788_b200`) must not import anything from here.

Parity pin: the oracle is checked against golden vectors produced by the
reference itself (`tests/golden/make_golden.py` imports the reference from
`/root/reference/pkg/src` in the build container and stores its outputs in
`tests/golden/*.npz`); `tests/test_oracle_golden.py` asserts the match.

Data layout follows the reference's dense backend: an m x k float64 block in
Fortran (column-major) order (`varray.py:107`), every tall product producing a
fresh Fortran-ordered block (`varray.py:157-163`).  The tall-side arithmetic is
NumPy/OpenBLAS, the triangular inverse is LAPACK ``dtrtri`` -- the same
third-party arithmetic the reference calls (`kernels.py:97`).  The Cholesky
loop, power iteration, shift rule and all control flow are restated here.
"""

from __future__ import annotations

import math
import warnings

import numpy as np
from scipy.linalg import lapack

#: unit roundoff used by the reference (`kernels.py:22`)
U = 1.11e-16


class OracleBreakdown(Exception):
    """Non-positive (or NaN) Schur diagonal; mirrors `kernels.py:25-39`."""

    def __init__(self, pivot_index, pivot_value):
        super().__init__(f"breakdown at pivot {pivot_index}: {pivot_value:.6e}")
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value


class OracleShiftLimit(Exception):
    """Shifted retries exhausted; mirrors `algorithms.py:47-56`."""

    def __init__(self, attempts, last_shift):
        super().__init__(f"shift limit after {attempts} attempts ({last_shift:.3e})")
        self.attempts = attempts
        self.last_shift = last_shift


# ----------------------------------------------------------------------------
# tall side (varray.py:150-171)
# ----------------------------------------------------------------------------

def gram(x, y=None):
    """Self Gramian symmetrized as (G+G^T)/2 (`varray.py:150-153`) or the
    cross Gramian x^T y (`varray.py:154-155`)."""
    if y is None:
        g = x.T @ x
        return (g + g.T) / 2.0
    return x.T @ y


def lincomb(x, c):
    """x @ c stored as a fresh Fortran-order block (`varray.py:157-163`)."""
    return np.asfortranarray(x @ np.asarray(c, dtype=float))


# ----------------------------------------------------------------------------
# k x k kernels (kernels.py:61-194)
# ----------------------------------------------------------------------------

def cholesky_upper(x):
    """Row-by-row (up-looking) upper Cholesky (`kernels.py:61-82`): the
    breakdown test is ``not s > 0`` so zero and NaN pivots both fail."""
    x = np.asarray(x, dtype=float)
    n = x.shape[0]
    r = np.zeros_like(x)
    for j in range(n):
        col = r[:j, j]
        s = x[j, j] - col @ col
        if not s > 0.0:
            exc = OracleBreakdown(j, float(s))
            top = float(np.max(np.diag(x)))
            exc.margin = float(s) / top if top > 0 else float("nan")
            raise exc
        d = math.sqrt(s)
        r[j, j] = d
        if j + 1 < n:
            r[j, j + 1:] = (x[j, j + 1:] - col @ r[:j, j + 1:]) / d
    return r


def tri_inverse(r):
    """Upper-triangular inverse through LAPACK dtrtri (`kernels.py:85-100`)."""
    n = r.shape[0]
    if n == 0:
        return r.copy()
    zero = np.flatnonzero(np.diag(r) == 0.0)
    if zero.size:
        raise ZeroDivisionError(int(zero[0]))
    inv, info = lapack.dtrtri(r, lower=0, unitdiag=0)
    if info != 0:
        raise ZeroDivisionError(int(info - 1))
    return np.triu(inv)


def tri_mult(a, b):
    """triu(a @ b) (`kernels.py:103-114`)."""
    return np.triu(a @ b)


def identity_distance(x):
    """||x - I||_F (`algorithms.py:197-198`, `kernels.py:117-123`)."""
    return float(np.linalg.norm(x - np.eye(x.shape[0])))


def spectral_estimate(x, tol=1e-2, max_iter=100):
    """Power iteration from the normalized all-ones vector with the Rayleigh
    settling rule; Frobenius fallback with a warning (`kernels.py:126-178`).
    Returns (estimate, flag) with flag 0 = converged, 1 = stalled,
    2 = not converged."""
    n = x.shape[0]
    if n == 0:
        return 0.0, 0
    fro = float(np.linalg.norm(x))
    if fro == 0.0:
        return 0.0, 0
    if np.linalg.norm(x - x.T) > 1e-8 * fro:
        raise ValueError("spectral estimate needs a symmetric matrix")
    v = np.full(n, 1.0 / math.sqrt(n))
    prev = None
    for _ in range(max_iter):
        w = x @ v
        nw = float(np.linalg.norm(w))
        if nw == 0.0:
            warnings.warn("power iteration stalled on a nullspace vector; "
                          "falling back to the Frobenius upper bound", stacklevel=2)
            return fro, 1
        lam = float(v @ w)
        v = w / nw
        if prev is not None and abs(lam - prev) <= tol * abs(lam):
            return abs(lam), 0
        prev = lam
    warnings.warn("power iteration did not converge; falling back to the "
                  "Frobenius upper bound", stacklevel=2)
    return fro, 2


def shift_value(m, n, norm_x, u=U):
    """max(11 (m n + n (n+1)) u ||X||, 2u) with Python `max` semantics (a NaN
    norm yields a NaN shift) (`kernels.py:181-194`)."""
    return max(11.0 * (m * n + n * (n + 1)) * u * norm_x, 2.0 * u)


def _with_shift(x, sigma):
    out = x.copy()
    out[np.diag_indices_from(out)] += sigma
    return out


# ----------------------------------------------------------------------------
# drivers (algorithms.py:201-458)
# ----------------------------------------------------------------------------

class Result:
    """Plain record of one oracle run (the fields of `QRResult`,
    `algorithms.py:99-126`)."""

    def __init__(self, q, r, iterations, shifts=(), attempts=(), success=True,
                 orth_error=None, margins=()):
        self.q = q
        self.r = r
        self.iterations = iterations
        self.shifts_applied = list(shifts)
        self.shift_attempts = list(attempts)
        self.success = success
        self.orth_error = orth_error
        # relative min pivot min(diag(R)^2)/max(diag(X)) of each accepted
        # factorization: tells how rounding-determined a decision was
        self.pivot_margins = list(margins)
        # ||X - I||_F measured at the top of each outer iteration (iterated
        # schemes): tells how rounding-determined the convergence test was
        self.err_history = []
        # signed relative pivot of each pass's first factorization attempt
        # (min Schur diagonal / max diag(X); negative when it broke down)
        self.decision_margins = []


def _attempt(x, top=None):
    """One factorization attempt: (r, signed margin) or (None, margin); the
    margin is the smallest Schur pivot over `top` (default max diag(x))."""
    if top is None:
        top = float(np.max(np.diag(x))) if x.size else 1.0
    try:
        r = cholesky_upper(x)
    except OracleBreakdown as exc:
        return None, exc.pivot_value / top, exc
    return r, _margin(x, r), None


def _margin(x, r):
    d = np.diag(r)
    top = float(np.max(np.diag(x))) if x.size else 1.0
    return float(np.min(d * d) / top) if top > 0 else float("nan")


def chol_qr(a):
    """One plain pass (`algorithms.py:201-212`)."""
    a = np.asfortranarray(a, dtype=float)
    x = gram(a)
    r = cholesky_upper(x)
    return Result(lincomb(a, tri_inverse(r)), r, 1, margins=[_margin(x, r)])


def chol_qr2(a):
    """Two plain passes, factors multiplied (`algorithms.py:215-220`)."""
    one = chol_qr(a)
    two = chol_qr(one.q)
    return Result(two.q, tri_mult(two.r, one.r), 2,
                  margins=one.pivot_margins + two.pivot_margins)


def s_chol_qr3(a, u=U):
    """Unconditionally shifted pass, then two plain passes
    (`algorithms.py:223-244`)."""
    a = np.asfortranarray(a, dtype=float)
    m, n = a.shape
    x = gram(a)
    est, _ = spectral_estimate(x)
    sigma = shift_value(m, n, est, u)
    xs = _with_shift(x, sigma)
    r = cholesky_upper(xs)
    margins = [_margin(xs, r)]
    q = lincomb(a, tri_inverse(r))
    for _ in range(2):
        x = gram(q)
        rk = cholesky_upper(x)
        margins.append(_margin(x, rk))
        q = lincomb(q, tri_inverse(rk))
        r = tri_mult(rk, r)
    return Result(q, r, 3, shifts=[sigma], margins=margins)


def _recomputed_shift_attempts(x, m, width, cfg, shifts):
    """Shifted retries after a plain breakdown, shift re-derived from the
    current Gramian then escalated (`algorithms.py:295-317`)."""
    est, _ = spectral_estimate(x)
    sigma = shift_value(m, width, est, cfg["u"])
    tries = 0
    while True:
        tries += 1
        if tries > cfg["max_shift_attempts"]:
            raise OracleShiftLimit(tries - 1, sigma)
        shifts.append(sigma)
        xs = _with_shift(x, sigma)
        try:
            return cholesky_upper(xs), tries, xs
        except OracleBreakdown:
            sigma = max(cfg["shift_escalation"] * sigma, 2.0 * cfg["u"])


def default_cfg(**kw):
    """AlgoConfig defaults (`algorithms.py:71-77`)."""
    cfg = dict(tol=1e-13, max_iter=10, shift_escalation=10.0,
               max_shift_attempts=60, u=U, tol_policy="fixed",
               update_shift_width="existing")
    cfg.update(kw)
    return cfg


def effective_tol(cfg, width):
    """`AlgoConfig.effective_tol` (`algorithms.py:93-96`)."""
    if cfg["tol_policy"] == "roundoff":
        return cfg["u"] * math.sqrt(max(width, 1))
    return cfg["tol"]


def rs_chol_qr(a, cfg=None):
    """The paper's shift-recomputing iteration, Alg. 1 (`algorithms.py:320-355`)."""
    cfg = cfg or default_cfg()
    a = np.asfortranarray(a, dtype=float)
    m, n = a.shape
    tol = effective_tol(cfg, n)
    q = a.copy(order="F")
    r = np.eye(n)
    x = gram(q)
    shifts, attempts, margins = [], [], []
    its = 0
    err = identity_distance(x)
    hist = [err]
    dms = []
    while not err < tol:
        if its == cfg["max_iter"]:
            out = Result(q, r, its, shifts, attempts, False, err, margins)
            out.err_history = hist
            out.decision_margins = dms
            return out
        rk, dm, _ = _attempt(x)
        dms.append(dm)
        if rk is not None:
            attempts.append(0)
            xs = x
        else:
            rk, tries, xs = _recomputed_shift_attempts(x, m, n, cfg, shifts)
            attempts.append(tries)
        margins.append(_margin(xs, rk))
        q = lincomb(q, tri_inverse(rk))
        r = tri_mult(rk, r)
        x = gram(q)
        its += 1
        err = identity_distance(x)
        hist.append(err)
    out = Result(q, r, its, shifts, attempts, True, err, margins)
    out.err_history = hist
    out.decision_margins = dms
    return out


def is_chol_qr(a, cfg=None):
    """Iterated passes with one fixed shift taken from the initial Gramian's
    norm estimate at the first breakdown; no escalation
    (`algorithms.py:247-292`)."""
    cfg = cfg or default_cfg()
    a = np.asfortranarray(a, dtype=float)
    m, n = a.shape
    tol = effective_tol(cfg, n)
    q = a.copy(order="F")
    r = np.eye(n)
    x = gram(q)
    first = x
    sigma0 = None
    shifts, attempts, margins, dms = [], [], [], []
    its = 0
    err = identity_distance(x)
    hist = [err]
    while not err < tol:
        if its == cfg["max_iter"]:
            out = Result(q, r, its, shifts, attempts, False, err, margins)
            out.err_history, out.decision_margins = hist, dms
            return out
        rk, dm, _ = _attempt(x)
        dms.append(dm)
        if rk is not None:
            attempts.append(0)
            xs = x
        else:
            if sigma0 is None:
                est, _ = spectral_estimate(first)
                sigma0 = shift_value(m, n, est, cfg["u"])
            xs = _with_shift(x, sigma0)
            rk = cholesky_upper(xs)
            shifts.append(sigma0)
            attempts.append(1)
        margins.append(_margin(xs, rk))
        q = lincomb(q, tri_inverse(rk))
        r = tri_mult(rk, r)
        x = gram(q)
        its += 1
        err = identity_distance(x)
        hist.append(err)
    out = Result(q, r, its, shifts, attempts, True, err, margins)
    out.err_history, out.decision_margins = hist, dms
    return out


def _deflated(q, bt):
    """Deflated, symmetrized Gramian (`algorithms.py:358-366`)."""
    return _deflated_from(gram(q), bt)


def _deflated_from(g, bt):
    """The same from an already formed Gramian g = q^T q (used to replay the
    decision stage on another implementation's Gramians)."""
    x = g - bt.T @ bt
    return (x + x.T) / 2.0


def _update_attempts(x, m, width, cfg, shifts):
    """sigma = 0, then the width-scaled shift, then escalations
    (`algorithms.py:369-397`)."""
    sigma = 0.0
    tries = 0
    while True:
        xs = _with_shift(x, sigma)
        try:
            return cholesky_upper(xs), tries, xs
        except OracleBreakdown:
            tries += 1
            if tries > cfg["max_shift_attempts"]:
                raise OracleShiftLimit(tries - 1, sigma) from None
            if sigma == 0.0:
                est, _ = spectral_estimate(x)
                sigma = shift_value(m, width, est, cfg["u"])
            else:
                sigma = cfg["shift_escalation"] * sigma
            sigma = max(sigma, 2.0 * cfg["u"])
            shifts.append(sigma)


def chol_qr_update(q_in, r_in, a_new, cfg=None):
    """Block-append update, Alg. 2 (`algorithms.py:400-458`).  q_in is m x k
    (k may be 0), a_new m x p; returns the augmented basis and factor."""
    cfg = cfg or default_cfg()
    q_in = np.asfortranarray(q_in, dtype=float)
    a_new = np.asfortranarray(a_new, dtype=float)
    m, k = q_in.shape
    p = a_new.shape[1]
    r_in = np.asarray(r_in, dtype=float).reshape(k, k)
    tol = effective_tol(cfg, p)
    width = k if cfg["update_shift_width"] == "existing" else p
    q = a_new.copy(order="F")
    b = np.zeros((k, p))
    r = np.eye(p)
    bt = gram(q_in, q)
    x = _deflated(q, bt)
    shifts, attempts, margins = [], [], []
    its = 0
    ok = True
    err = identity_distance(x)
    hist = [err]
    dms = []
    ratios = []
    while not err < tol:
        if its == cfg["max_iter"]:
            ok = False
            break
        top = float(np.max(np.diag(x) + np.sum(bt * bt, axis=0))) if bt.size else None
        dms.append(_attempt(_with_shift(x, 0.0), top)[1])
        # how much of the Gramian the deflation cancelled: X's rounding error
        # relative to X is ~u times this (test infrastructure: it scales the
        # tolerance of the shift comparison, tests/parity.py)
        dx = float(np.max(np.abs(np.diag(x)))) if x.size else 0.0
        ratios.append(top / dx if (top is not None and dx > 0) else 1.0)
        rk, tries, xs = _update_attempts(x, m, width, cfg, shifts)
        attempts.append(tries)
        margins.append(_margin(xs, rk))
        q = np.asfortranarray(q - lincomb(q_in, bt))
        q = lincomb(q, tri_inverse(rk))
        b = b + bt @ r
        r = tri_mult(rk, r)
        bt = gram(q_in, q)
        x = _deflated(q, bt)
        its += 1
        err = identity_distance(x)
        hist.append(err)
    q_out = np.asfortranarray(np.concatenate([q_in, q], axis=1))
    r_out = np.block([[r_in, b], [np.zeros((p, k)), r]])
    out = Result(q_out, r_out, its, shifts, attempts, ok, err, margins)
    out.err_history = hist
    out.decision_margins = dms
    out.deflation_ratios = ratios
    return out


# ----------------------------------------------------------------------------
# quality measures (metrics.py:42-71), Frobenius variants
# ----------------------------------------------------------------------------

def loo_fro(q):
    """||I - Q^T Q||_F (`metrics.py:42-50`)."""
    return float(np.linalg.norm(np.eye(q.shape[1]) - gram(q)))


def rrr_fro(a, q, r):
    """sqrt(trace(D^T D)) / sqrt(trace(A^T A)), D = A - Q R (`metrics.py:53-71`)."""
    d = np.asfortranarray(a - q @ r)
    num = math.sqrt(max(float(np.trace(gram(d))), 0.0))
    den = math.sqrt(max(float(np.trace(gram(a))), 0.0))
    return num / den


def panel_widths(n, r_panels):
    """n columns in r contiguous panels, the first n mod r one wider
    (`algorithms.py:461-467`)."""
    if not 1 <= r_panels <= n:
        raise ValueError(f"need 1 <= r_panels <= {n}, got {r_panels}")
    base, extra = divmod(n, r_panels)
    return [base + 1] * extra + [base] * (r_panels - extra)


def pn_chol_qr(a, r_panels, cfg=None):
    """Panel scheme, Alg. 3: chol_qr_update folded over contiguous column
    panels from an empty basis; a capped panel marks the result unsuccessful
    but later panels still run; an exception is annotated with its panel
    index (`algorithms.py:470-505`)."""
    cfg = cfg or default_cfg()
    a = np.asfortranarray(a, dtype=float)
    m = a.shape[0]
    q = np.zeros((m, 0), order="F")
    r = np.zeros((0, 0))
    shifts, attempts, profiles, margins, dms, hist, ratios = [], [], [], [], [], [], []
    its = 0
    ok = True
    err = None
    start = 0
    for index, width in enumerate(panel_widths(a.shape[1], r_panels)):
        panel = a[:, start:start + width]
        start += width
        try:
            res = chol_qr_update(q, r, panel, cfg)
        except OracleShiftLimit as exc:
            exc.panel_index = index
            raise
        q, r = res.q, res.r
        its += res.iterations
        shifts.extend(res.shifts_applied)
        attempts.extend(res.shift_attempts)
        profiles.append((res.iterations, tuple(res.shift_attempts))
                        if len(res.shift_attempts) == res.iterations else None)
        margins.extend(res.pivot_margins)
        dms.extend(res.decision_margins)
        hist.extend(res.err_history)
        ratios.extend(res.deflation_ratios)
        err = res.orth_error
        ok = ok and res.success
    out = Result(q, r, its, shifts, attempts, ok, err, margins)
    out.panel_profiles = profiles
    out.decision_margins = dms
    out.err_history = hist
    out.deflation_ratios = ratios
    return out
