"""The reference's k x k kernel API (reference kernels.py:61-194), backed by
the device factor kernel (K4) where there is arithmetic to do.

`cholesky(x)` and `spectral_norm_estimate(x)` run the same single-CTA kernel
the drivers use each pass, so the reference's kernel-level known-answer
tests exercise the device code directly.  `compute_shift` is the scalar
formula (host arithmetic, same expression and Python `max` semantics).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import flops as _flops
from ._engine import Engine
from .algorithms import UNIT_ROUNDOFF, AlgoConfig, _raise_for
from .errors import CholeskyBreakdown, TriangularSingularError  # noqa: F401 (re-export)


def compute_shift(m, n, norm_x, u=UNIT_ROUNDOFF):
    """max(11 (m n + n (n+1)) u ||X||, 2u) (reference kernels.py:181-194)."""
    if m < 0 or n < 0:
        raise ValueError("dimensions must be nonnegative")
    if norm_x < 0:
        raise ValueError("norm_x must be >= 0")
    if not 0.0 < u < 1e-7:
        raise ValueError("unit roundoff out of range")
    return max(11.0 * (m * n + n * (n + 1)) * u * norm_x, 2.0 * u)


def _square(x, who):
    x = np.asarray(x, dtype=float)
    if x.ndim != 2 or x.shape[0] != x.shape[1]:
        raise ValueError(f"{who} needs a square matrix, got shape {x.shape}")
    return x


def _engine_for(x):
    k = x.shape[0]
    eng = Engine(k, AlgoConfig())
    # the kernel reads the lower triangle of the column-major G; the transpose
    # of x in that layout makes it read x's upper triangle, as the reference's
    # row-oriented loop does (kernels.py:74-81)
    eng.G.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return eng


def cholesky(x, ledger=None):
    """Upper Cholesky factor; CholeskyBreakdown at the first Schur diagonal
    that is not > 0 (reference kernels.py:61-82), computed on the device."""
    x = _square(x, "cholesky")
    n = x.shape[0]
    if ledger is not None:
        ledger.add("potrf", _flops.cholesky_flops(n))
    if n == 0:
        return np.zeros((0, 0))
    eng = _engine_for(x)
    st = eng.factor(_lib.POLICY_PLAIN, 1, n)
    _raise_for(st)
    return eng.Rk[:, :n].cpu().numpy().T.copy()


def spectral_norm_estimate(x, ledger=None):
    """Power-iteration estimate of the largest |eigenvalue| with the Frobenius
    fallback (reference kernels.py:126-178), computed on the device."""
    x = _square(x, "spectral_norm_estimate")
    n = x.shape[0]
    if ledger is not None:
        ledger.add("eig_est", _flops.eig_estimate_flops(n))
    if n == 0:
        return 0.0
    # input validation of the reference (kernels.py:145-153); the device
    # kernel itself only ever sees symmetric matrices
    fro = float(np.linalg.norm(x))
    if fro == 0.0:
        return 0.0
    asym = float(np.linalg.norm(x - x.T))
    if asym > 1e-8 * fro:
        raise ValueError(
            f"spectral_norm_estimate needs a symmetric matrix (asymmetry {asym:.3e} vs norm {fro:.3e})")
    eng = _engine_for(x)
    st = eng.factor(_lib.POLICY_SHIFT_ONCE, 1, n)
    if st.code == _lib.ASYMMETRIC:
        raise ValueError("spectral_norm_estimate needs a symmetric matrix")
    from .algorithms import _emit_estimate_warning

    _emit_estimate_warning(st)
    return float(st.norm_est)
