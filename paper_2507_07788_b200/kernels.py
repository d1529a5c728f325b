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
from ._device import ctx
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


def _upper(r, who):
    r = _square(r, who)
    if r.shape[0] and np.any(np.tril(r, -1) != 0.0):
        raise ValueError(f"{who} needs an upper-triangular matrix")
    return r


def _to_dev(x):
    # column-major on the device: torch (n, n) row-major of x^T
    return torch.from_numpy(np.ascontiguousarray(x.T)).to(ctx().device)


def _from_dev(t):
    return t.cpu().numpy().T.copy()


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


def spectral_norm_estimate(x, ledger=None, tol=1e-2, max_iter=100):
    """Power-iteration estimate of the largest |eigenvalue| with the Frobenius
    fallback (reference kernels.py:126-178), computed on the device; `tol` and
    `max_iter` are the settling tolerance and the iteration cap."""
    x = _square(x, "spectral_norm_estimate")
    if max_iter < 1:
        # the reference's loop body never runs: straight to the fallback warning
        max_iter = 0
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
    st = eng.factor(_lib.POLICY_ESTIMATE, 1, n, est_tol=float(tol), est_max_iter=int(max_iter))
    if st.code == _lib.ASYMMETRIC:
        raise ValueError("spectral_norm_estimate needs a symmetric matrix")
    from .algorithms import _emit_estimate_warning

    _emit_estimate_warning(st)
    return float(st.norm_est)


def tri_inverse(r, ledger=None):
    """Inverse of an upper-triangular matrix, upper triangular with exact zeros
    below the diagonal (reference kernels.py:85-100), on the device.  A zero
    diagonal raises TriangularSingularError with its index."""
    r = _upper(r, "tri_inverse")
    n = r.shape[0]
    if ledger is not None:
        ledger.add("trtri", _flops.tri_inverse_flops(n))
    if n == 0:
        return r.copy()
    zero = np.flatnonzero(np.diag(r) == 0.0)
    if zero.size:
        raise TriangularSingularError(int(zero[0]))
    cx = ctx()
    rd = _to_dev(r)
    out = torch.empty_like(rd)
    _lib.check(cx.lib.cqr_tri_inverse(rd.data_ptr(), n, n, out.data_ptr(), n, cx.stream), "tri_inverse")
    cx.launches += 1
    return _from_dev(out)


def tri_multiply(a, b, ledger=None):
    """triu(a @ b) of two upper-triangular matrices (reference kernels.py:103-114),
    on the device."""
    a = _upper(a, "tri_multiply")
    b = _upper(b, "tri_multiply")
    if a.shape != b.shape:
        raise ValueError(f"size mismatch: {a.shape} vs {b.shape}")
    n = a.shape[0]
    if ledger is not None:
        ledger.add("trmm", _flops.trmm_flops(n))
    if n == 0:
        return np.zeros((0, 0))
    cx = ctx()
    ad, bd = _to_dev(a), _to_dev(b)
    out = torch.empty_like(ad)
    _lib.check(cx.lib.cqr_tri_multiply(ad.data_ptr(), n, bd.data_ptr(), n, n, out.data_ptr(), n, cx.stream),
               "tri_multiply")
    cx.launches += 1
    return _from_dev(out)


def frobenius(x, ledger=None):
    """Frobenius norm (reference kernels.py:117-123), one fixed-order device
    reduction.  Ledger charges assume a square matrix (2n^2 + n)."""
    x = np.asarray(x, dtype=float)
    if ledger is not None:
        _square(x, "frobenius (with ledger)")
        ledger.add("fro_norm", _flops.frobenius_flops(x.shape[0]))
    x2 = x.reshape(x.shape[0], -1) if x.ndim == 2 else x.reshape(-1, 1)
    rows, cols = x2.shape
    cx = ctx()
    out = torch.empty(1, dtype=torch.float64, device=cx.device)
    xd = _to_dev(x2) if x2.size else out
    _lib.check(cx.lib.cqr_frobenius(xd.data_ptr(), max(rows, 1), rows, cols, out.data_ptr(), cx.stream),
               "frobenius")
    cx.launches += 1
    return float(out.item())
