"""Decision-parity rule shared by the GPU parity tests.

A decision -- breakdown or not of a pass's first factorization attempt, and
converged-or-not of the ||X - I||_F < tol test -- is *robust* when it is far
from rounding noise: |signed pivot margin| > 100 k u, and ||X - I||_F outside
[tol/100, 100 tol] (see robust_conv).  Robust decisions must be identical to the oracle's; from
the first rounding-determined decision on, the runs may take different
branches and only the final quality (LOO_F, RRR_F within 10x) is compared.
"""

from __future__ import annotations

import math

import numpy as np

U = 1.11e-16


def robust_margin(margin, k):
    return margin is not None and not math.isnan(margin) and abs(margin) > 100 * k * U


def robust_conv(err, tol, mine=None):
    """The converged-or-not test ||X - I||_F < tol is robust when err is far
    from tol.  After a pass, err is itself rounding noise (~kappa^2 u of the
    previous Q), and two correct implementations were seen 10x apart on it
    (1200x3 at kappa 1e2: 1.0e-12 in the oracle, below 1e-13 here), so the band
    is two decades either side of tol, on the oracle's and (when given) our
    own value."""
    for e in (err, mine):
        if e is not None and tol / 100 <= e <= 100 * tol:
            return False
    return True


def compare_iterated(mine, ref, k, tol):
    """Compare per-iteration decisions while they are robust.  Returns the
    number of iterations whose decisions were compared (and matched)."""
    n = min(len(mine.shift_attempts), len(ref.shift_attempts))
    mine_err = list(getattr(mine, "err_history", []) or [])

    def my_err(i):
        return mine_err[i] if i < len(mine_err) else None

    pm = pr = 0
    for i in range(n):
        if not robust_conv(ref.err_history[i], tol, my_err(i)):
            return i
        if not (robust_margin(ref.decision_margins[i], k) and robust_margin(mine.decision_margins[i], k)):
            return i
        assert mine.shift_attempts[i] == ref.shift_attempts[i], (i, mine.shift_attempts, ref.shift_attempts)
        a = mine.shift_attempts[i]
        np.testing.assert_allclose(mine.shifts_applied[pm:pm + a], ref.shifts_applied[pr:pr + a], rtol=1e-6)
        pm += a
        pr += a
    if len(ref.err_history) > n and robust_conv(ref.err_history[n], tol, my_err(n)):
        assert mine.iterations == ref.iterations, (mine.iterations, ref.iterations, ref.err_history)
    return n


def within10(mine, ref, k, tol=None):
    """mine <= 10 x ref (floored at 10 u sqrt(k)); after a rounding-determined
    convergence decision both runs stopped on ||X - I||_F < tol, so tol also
    bounds the comparison then."""
    floor = 10 * U * math.sqrt(k)
    if tol is not None:
        floor = max(floor, tol)
    return mine <= 10 * max(ref, floor)
