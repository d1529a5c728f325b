"""Shifted Cholesky QR drivers on the B200 backend, reference API.

Same names, signatures, results and exceptions as the reference's
`cholqr.algorithms` (reference algorithms.py:201-505):

  chol_qr(a, cfg, ledger)            algorithms.py:201-212
  chol_qr2(a, cfg, ledger)           algorithms.py:215-220   (configs 2, 5)
  s_chol_qr3(a, cfg, ledger)         algorithms.py:223-244   (config 1)
  rs_chol_qr(a, cfg, ledger)         algorithms.py:320-355   (config 3, Alg. 1)
  chol_qr_update(q_in, r_in, a_new)  algorithms.py:400-458   (config 4, Alg. 2)
  pn_chol_qr(a, r_panels)            algorithms.py:461-505   (Alg. 3)

The host keeps only the loop control: each pass is a fused tall kernel on
the device (TRMM by R^-1 + next Gram, one HBM stream), one NCCL allreduce of
the k x k Gram when rows are sharded, and one k x k kernel that measures
||X - I||_F, factors with breakdown detection and the shift rule, and
inverts; its status record (one small D2H copy) drives the loop.  Flop
ledgers are charged exactly as the reference charges them.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import flops as _flops
from ._engine import Engine, cross_gram_device
from .errors import CholeskyBreakdown, ShiftAttemptLimitError, TriangularSingularError
from .flops import IterationProfile
from .varray import CudaVectorArray

#: Unit roundoff of 64-bit floats as the reference defines it (kernels.py:22).
UNIT_ROUNDOFF = 1.11e-16


@dataclass(frozen=True)
class AlgoConfig:
    """Shared knobs (reference algorithms.py:59-96)."""

    tol: float = 1e-13
    max_iter: int = 10
    shift_escalation: float = 10.0
    max_shift_attempts: int = 60
    unit_roundoff: float = UNIT_ROUNDOFF
    tol_policy: str = "fixed"
    update_shift_width: str = "existing"

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError("tol must be > 0")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if not self.shift_escalation > 1:
            raise ValueError("shift_escalation must be > 1")
        if self.max_shift_attempts < 1:
            raise ValueError("max_shift_attempts must be >= 1")
        if self.tol_policy not in ("fixed", "roundoff"):
            raise ValueError("tol_policy must be 'fixed' or 'roundoff'")
        if self.update_shift_width not in ("existing", "incoming"):
            raise ValueError("update_shift_width must be 'existing' or 'incoming'")

    def effective_tol(self, width):
        if self.tol_policy == "roundoff":
            return self.unit_roundoff * math.sqrt(max(width, 1))
        return self.tol


@dataclass
class QRResult:
    """Factors plus run diagnostics (reference algorithms.py:99-156).

    `pivot_margins` / `decision_margins` are additions: min diag(R_k)^2 /
    max diag(X + sigma I) of every accepted factorization, and the signed
    relative Schur pivot of each pass's first attempt (negative: it broke
    down), i.e. how far each decision was from the rounding boundary
    (SURVEY.md §8(c))."""

    q: "CudaVectorArray"
    r: np.ndarray
    iterations: int
    shifts_applied: list = field(default_factory=list)
    shift_attempts: list = field(default_factory=list)
    success: bool = True
    orth_error: float | None = None
    dropped: list = field(default_factory=list)
    panel_profiles: list | None = None
    pivot_margins: list = field(default_factory=list)
    decision_margins: list = field(default_factory=list)
    err_history: list = field(default_factory=list)   # ||X - I||_F measured by every pass

    @property
    def profile(self):
        if len(self.shift_attempts) != self.iterations:
            return None
        return IterationProfile(self.iterations, tuple(self.shift_attempts))

    def r_with_drops(self):
        if not self.dropped:
            return self.r
        k, kept = self.r.shape
        n = kept + len(self.dropped)
        out = np.zeros((k, n))
        dropped = set(self.dropped)
        cols = [j for j in range(n) if j not in dropped]
        out[:, cols] = self.r
        return out


# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------

def _device_array(a):
    if isinstance(a, CudaVectorArray):
        return a
    if hasattr(a, "_iter_columns") or hasattr(a, "to_numpy"):
        return CudaVectorArray.from_array(a)
    raise TypeError(f"expected a VectorArray, got {type(a).__name__}")


def _charge(ledger, cat, n):
    if ledger is not None:
        ledger.add(cat, n)


def _emit_estimate_warning(st):
    # spectral_norm_estimate's UserWarnings (reference kernels.py:162-177)
    if st.est_flag == 1:
        warnings.warn("power iteration stalled on a nullspace vector; "
                      "falling back to the Frobenius upper bound", stacklevel=3)
    elif st.est_flag == 2:
        warnings.warn("power iteration did not converge; falling back to the "
                      "Frobenius upper bound", stacklevel=3)


def _raise_for(st):
    if st.code == _lib.BREAKDOWN:
        exc = CholeskyBreakdown(int(st.pivot_index), float(st.pivot_value))
        exc.margin = float(st.plain_margin)   # pivot / max diag: how decisive the breakdown was
        raise exc
    if st.code == _lib.SHIFT_LIMIT:
        raise ShiftAttemptLimitError(int(st.retries), float(st.last_shift))
    if st.code == _lib.TRI_SINGULAR:
        raise TriangularSingularError(int(st.singular_index))
    if st.code == _lib.ASYMMETRIC:
        raise ValueError("spectral_norm_estimate needs a symmetric matrix")


def _charge_plain_attempt(ledger, n):
    _charge(ledger, "potrf", _flops.cholesky_flops(n))


def _charge_recompute(ledger, n, st):
    """cholesky + (_retry_with_recomputed_shift) charges (algorithms.py:295-317,
    kernels.py:71-72,141-142)."""
    _charge_plain_attempt(ledger, n)
    if st.est_calls:
        _charge(ledger, "eig_est", _flops.eig_estimate_flops(n))
    tried = st.n_shifts
    _charge(ledger, "potrf", tried * (_flops.cholesky_flops(n) + n))
    _charge(ledger, "eig_est", st.escalations)


def _charge_update(ledger, p, st):
    """_update_factor_attempts charges (algorithms.py:369-397)."""
    attempts = st.n_shifts + 1
    if st.code == _lib.SHIFT_LIMIT:
        attempts = st.retries + 1
    _charge(ledger, "potrf", attempts * (_flops.cholesky_flops(p) + p))
    if st.est_calls:
        _charge(ledger, "eig_est", st.est_calls * _flops.eig_estimate_flops(p))
    _charge(ledger, "eig_est", st.escalations)


# ----------------------------------------------------------------------------
# one-shot passes
# ----------------------------------------------------------------------------

def chol_qr(a, cfg=None, ledger=None):
    """One plain pass: Q = A R^-1 with R from the Gramian; breakdown propagates.

    Fixed schedule: the kernels are enqueued back to back and the factor status
    is read once at the end; charges and raises replay the reference's order
    (algorithms.py:201-212), so a breakdown raises with the same ledger state."""
    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    if a.ncols < 1:
        raise ValueError("need at least one column")
    m, n = a.space.dim, a.ncols
    eng, q, (st,) = _run_fixed(a, cfg, [_lib.POLICY_PLAIN])
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    _charge_plain_attempt(ledger, n)
    _raise_for(st)
    _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    return QRResult(q=q, r=eng.r_host(), iterations=1, pivot_margins=[st.min_pivot_rel],
                    decision_margins=[st.plain_margin])


def _fresh_like(a, n):
    return CudaVectorArray(a.space, a._alloc(a.space, n, zero=False), n)


def chol_qr2(a, cfg=None, ledger=None):
    """Two plain passes, factors multiplied (algorithms.py:215-220).

    Device schedule: Gram(A) | factor | Q1 = A R1^-1 + Gram(Q1) | factor |
    Q = Q1 R2^-1 in place, enqueued without a host sync; both statuses are read
    at the end and the reference's charge / raise sequence is replayed."""
    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    if a.ncols < 1:
        raise ValueError("need at least one column")
    m, n = a.space.dim, a.ncols
    eng, q, (st1, st2) = _run_fixed(a, cfg, [_lib.POLICY_PLAIN, _lib.POLICY_PLAIN])
    margins = []
    for i, st in enumerate((st1, st2)):
        if i == 1:
            _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))      # lincomb of pass 1
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))          # Gram of this pass
        _charge_plain_attempt(ledger, n)
        _raise_for(st)
        margins.append(st.min_pivot_rel)
        _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    _charge(ledger, "trmm", _flops.trmm_flops(n))
    return QRResult(q=q, r=eng.r_host(), iterations=2, pivot_margins=margins)


def _apply_last(eng, q):
    """q <- q R^-1 without a following Gram (in place when the kernels allow)."""
    if eng.in_place_ok():
        eng.apply(q, q, with_gram=False)
    else:
        tmp = _fresh_like(q, q.ncols)
        eng.apply(q, tmp, with_gram=False)
        q._buf = tmp._buf


def _apply_gram_into(eng, src, fresh_ok):
    """dst = src R^-1 with the Gram of dst; in place where the fused kernel
    allows it, else into a new buffer.  Returns dst."""
    if not fresh_ok and eng.in_place_gram_ok():
        eng.apply(src, src, with_gram=True)
        return src
    dst = _fresh_like(src, src.ncols)
    eng.apply(src, dst, with_gram=True)
    return dst


def _run_fixed(a, cfg, policies):
    """Enqueue a fixed schedule -- Gram(A), then per pass the k x k stage
    (policies[i]) and Q_i = Q_{i-1} R_i^-1 with the next pass's Gram (plain
    TRMM on the last) -- and read the statuses once at the end.  Returns
    (engine, Q, statuses).  On one rank the whole schedule is one libcqr call
    (cqr_fixed_schedule, replayed as a CUDA graph); otherwise, or with a
    timer / decision trace attached, the same launches go one by one."""
    m, n = a.space.dim, a.ncols
    eng = Engine(n, cfg, defer_reset=True)
    npass = len(policies)
    if eng.fixed_ok():
        q = _fresh_like(a, n)
        dsts = [q]
        spare = None
        for i in range(1, npass):
            last = i == npass - 1
            if eng.in_place_ok() if last else eng.in_place_gram_ok():
                dsts.append(dsts[-1])
                continue
            if spare is None:
                spare = _fresh_like(a, n)
            dsts.append(spare if dsts[-1] is q else q)   # ping-pong: never the pass's own source
        hs = eng.run_fixed(policies, m, n, a, dsts)
        return eng, dsts[-1], eng.collect(hs)
    eng.reset_racc()
    eng.gram(a)
    hs = []
    q = a
    for i, pol in enumerate(policies):
        hs.append(eng.factor_async(pol, m, n))
        if i < npass - 1:
            q = _apply_gram_into(eng, q, fresh_ok=(i == 0))   # the first pass never writes A
        elif i == 0:
            dst = _fresh_like(a, n)
            eng.apply(a, dst, with_gram=False)
            q = dst
        else:
            _apply_last(eng, q)
    eng.r_prefetch()
    return eng, q, eng.collect(hs)


def s_chol_qr3(a, cfg=None, ledger=None):
    """Shifted first pass (sigma from the first Gram's norm estimate), then two
    plain passes; a breakdown in any pass propagates (algorithms.py:223-244).

    Fixed schedule: all three passes are enqueued without a host sync, the three
    statuses are read once, then the reference's warnings, charges and raises
    are replayed in order."""
    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    if a.ncols < 1:
        raise ValueError("need at least one column")
    m, n = a.space.dim, a.ncols
    eng, q, sts = _run_fixed(a, cfg, [_lib.POLICY_SHIFT_ONCE, _lib.POLICY_PLAIN, _lib.POLICY_PLAIN])

    st = sts[0]
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    _emit_estimate_warning(st)
    _charge(ledger, "eig_est", _flops.eig_estimate_flops(n))
    _charge(ledger, "potrf", n)
    _charge_plain_attempt(ledger, n)
    _raise_for(st)
    sigma = st.shifts[0]
    margins = [st.min_pivot_rel]
    _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    for st in sts[1:]:
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))      # Gram of this pass
        _charge_plain_attempt(ledger, n)
        _raise_for(st)
        margins.append(st.min_pivot_rel)
        _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
        _charge(ledger, "trmm", _flops.trmm_flops(n))
    return QRResult(q=q, r=eng.r_host(), iterations=3, shifts_applied=[sigma], pivot_margins=margins)


# ----------------------------------------------------------------------------
# iterated scheme (Alg. 1)
# ----------------------------------------------------------------------------

def rs_chol_qr(a, cfg=None, ledger=None):
    """Iterated passes with the shift recomputed at every breakdown
    (algorithms.py:320-355): plain attempt first; on breakdown the shift is
    re-derived from the current Gramian's norm estimate and escalated until
    the shifted factorization succeeds.  Stops when ||Q^T Q - I||_F < tol;
    the iteration cap returns success=False with the last distance.

    Host loop one pass ahead of the device: pass i+1 (factor, then TRMM +
    Gram) is enqueued before pass i's status is read; its launches are gated
    on the device by pass i's (resp. its own) factor status, so after the
    convergence / cap / error pass they do nothing.  The status is then read
    while the GPU already runs the next pass, and the reference's charges,
    warnings and raises are replayed in its order."""
    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    if a.ncols < 1:
        raise ValueError("need at least one column")
    m, n = a.space.dim, a.ncols
    tol = cfg.effective_tol(n)
    eng = Engine(n, cfg)
    eng.gram(a)
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    handles, outs = [], []

    def enqueue(p):
        prev = handles[p - 1] if p else None
        h = eng.factor_async(_lib.POLICY_RECOMPUTE, m, n, tol=tol, check_tol=True, stop=(p == cfg.max_iter),
                             gate=eng.gate(prev) if p else None, gate_slot=prev)
        src = a if p == 0 else outs[p - 1]
        # the reference's q = a.copy(), taken lazily: pass 0 writes a fresh array,
        # later passes work in place where the kernels allow it
        dst = src if (p > 0 and eng.in_place_gram_ok()) else _fresh_like(src, n)
        if p < cfg.max_iter:
            eng.apply(src, dst, with_gram=True, gate=eng.gate(h), gate_slot=h)
        handles.append(h)
        outs.append(dst)

    enqueue(0)
    shifts, attempts, margins, dms, errs = [], [], [], [], []
    its = 0
    while True:
        if its + 1 <= cfg.max_iter:
            enqueue(its + 1)
        (st,) = eng.collect([handles[its]])
        errs.append(st.err)
        if its >= 2:
            outs[its - 2] = None   # no longer a source or a result
        _charge(ledger, "fro_norm", _flops.frobenius_flops(n))
        if st.code == _lib.CONVERGED:
            break
        if st.code == _lib.CAPPED:
            return QRResult(outs[its - 1] if its else a.copy(), eng.r_host(), its, shifts, attempts,
                            success=False, orth_error=st.err, pivot_margins=margins, decision_margins=dms, err_history=errs)
        _emit_estimate_warning(st)
        _charge_recompute(ledger, n, st)
        _raise_for(st)
        dms.append(st.plain_margin)
        attempts.append(st.retries)
        shifts.extend(st.shifts)
        margins.append(st.min_pivot_rel)
        _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
        _charge(ledger, "trmm", _flops.trmm_flops(n))
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
        its += 1
    return QRResult(outs[its - 1] if its else a.copy(), eng.r_host(), its, shifts, attempts,
                    success=True, orth_error=st.err, pivot_margins=margins, decision_margins=dms, err_history=errs)


def is_chol_qr(a, cfg=None, ledger=None):
    """Iterated passes with one fixed shift (algorithms.py:247-292): at the
    first breakdown the shift is derived from the INITIAL Gramian's norm
    estimate and reused unchanged; a breakdown of the shifted factorization
    propagates (no escalation)."""
    import torch

    from .kernels import compute_shift

    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    if a.ncols < 1:
        raise ValueError("need at least one column")
    m, n = a.space.dim, a.ncols
    tol = cfg.effective_tol(n)
    eng = Engine(n, cfg)
    eng.gram(a)
    first = torch.empty_like(eng.G)
    first.copy_(eng.G)
    _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
    q = None
    sigma0 = None
    shifts, attempts, margins, dms, errs = [], [], [], [], []
    its = 0
    while True:
        st = eng.factor(_lib.POLICY_PLAIN, m, n, tol=tol, check_tol=True, stop=(its == cfg.max_iter))
        errs.append(st.err)
        _charge(ledger, "fro_norm", _flops.frobenius_flops(n))
        if st.code == _lib.CONVERGED:
            break
        if st.code == _lib.CAPPED:
            return QRResult(q if q is not None else a.copy(), eng.r_host(), its, shifts, attempts,
                            success=False, orth_error=st.err, pivot_margins=margins, decision_margins=dms, err_history=errs)
        _charge_plain_attempt(ledger, n)
        dms.append(st.plain_margin)
        err = st.err
        if st.code == _lib.BREAKDOWN:
            if sigma0 is None:
                cur = torch.empty_like(eng.G)
                cur.copy_(eng.G)
                eng.G.copy_(first)
                est = eng.factor(_lib.POLICY_ESTIMATE, m, n)
                eng.G.copy_(cur)
                _emit_estimate_warning(est)
                _raise_for(est)
                _charge(ledger, "eig_est", _flops.eig_estimate_flops(n))
                sigma0 = compute_shift(m, n, est.norm_est, cfg.unit_roundoff)
            _charge(ledger, "potrf", n)
            _charge_plain_attempt(ledger, n)
            st = eng.factor(_lib.POLICY_FIXED_SHIFT, m, n, fixed_shift=sigma0)
            _raise_for(st)
            shifts.append(sigma0)
            attempts.append(1)
        else:
            _raise_for(st)
            attempts.append(0)
        margins.append(st.min_pivot_rel)
        _charge(ledger, "trtri", _flops.tri_inverse_flops(n))
        q = _apply_gram_into(eng, a if q is None else q, fresh_ok=q is None)
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
        _charge(ledger, "trmm", _flops.trmm_flops(n))
        _charge(ledger, "gemm", _flops.gemm_flops(m, n, n))
        its += 1
        del err
    return QRResult(q if q is not None else a.copy(), eng.r_host(), its, shifts, attempts,
                    success=True, orth_error=st.err, pivot_margins=margins, decision_margins=dms, err_history=errs)


# ----------------------------------------------------------------------------
# block-append update (Alg. 2) and the panel fold (Alg. 3)
# ----------------------------------------------------------------------------

def chol_qr_update(q_in, r_in, a_new, cfg=None, ledger=None):
    """Extend an orthonormal basis by a new block (algorithms.py:400-458).

    Returns the augmented basis [q_in, Q] and the factor [[r_in, B], [0, R]]
    (lower-left block exactly zero, r_in embedded bitwise).  The new block is
    deflated against the basis and refactored until its deflated Gramian is
    within tolerance of the identity."""
    cfg = cfg or AlgoConfig()
    q_in = _device_array(q_in)
    a_new = _device_array(a_new)
    if a_new.ncols < 1:
        raise ValueError("need at least one new column")
    if q_in.space != a_new.space:
        raise ValueError("space mismatch between basis and new block")
    k, p = q_in.ncols, a_new.ncols
    r_in = np.asarray(r_in, dtype=float)
    if r_in.shape != (k, k):
        raise ValueError(f"r_in must be {k} x {k}, got {r_in.shape}")
    m = a_new.space.dim
    tol = cfg.effective_tol(p)
    width = k if cfg.update_shift_width == "existing" else p
    eng = Engine(p, cfg, q=k)
    fused = k > 0 and eng.cx.lib.cqr_update_supported(k, p) == 1

    def deflated_gram(qq):
        # bt = Q_in^T Q (device, q x p), G = Q^T Q; deflation happens in the factor kernel
        if fused:
            eng.update_pass(q_in, qq, initial=True)
        else:
            if k:
                cross_gram_device(q_in, qq, out=eng.Bt)
            eng.gram(qq)
        _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
        _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
        _charge(ledger, "gemm", _flops.gemm_flops(p, k, p) + p * p)

    q = None
    deflated_gram(a_new)
    shifts, attempts, margins, dms, errs = [], [], [], [], []
    its = 0
    success = True
    if fused:
        return _update_pipelined(eng, q_in, r_in, a_new, m, k, p, width, tol, cfg, ledger)
    while True:
        st = eng.factor(_lib.POLICY_UPDATE, m, width, tol=tol, check_tol=True, stop=(its == cfg.max_iter),
                        update_b=True)
        errs.append(st.err)
        _charge(ledger, "fro_norm", _flops.frobenius_flops(p))
        if st.code == _lib.CONVERGED:
            break
        if st.code == _lib.CAPPED:
            success = False
            break
        _emit_estimate_warning(st)
        _charge_update(ledger, p, st)
        _raise_for(st)
        dms.append(st.plain_margin)
        attempts.append(st.retries)
        shifts.extend(st.shifts)
        margins.append(st.min_pivot_rel)
        src = a_new if q is None else q
        if k == 0:
            # empty basis: identical device path to rs_chol_qr (bitwise contract,
            # reference tests/test_update_panel.py:36-45)
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", m * p)
            _charge(ledger, "trtri", _flops.tri_inverse_flops(p))
            q = _apply_gram_into(eng, src, fresh_ok=q is None)
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(k, p, p) + k * p)
            _charge(ledger, "trmm", _flops.trmm_flops(p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(p, k, p) + p * p)
        elif fused:
            # one sweep: Q <- (Q - Q_in Bt) R^-1, Bt <- Q_in^T Q, G <- Q^T Q; the
            # first one reads the caller's block and writes a fresh Q (no copy)
            if q is None:
                q = _fresh_like(a_new, p)
                eng.update_pass(q_in, a_new, initial=False, out=q)
            else:
                eng.update_pass(q_in, q, initial=False)
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", m * p)
            _charge(ledger, "trtri", _flops.tri_inverse_flops(p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(k, p, p) + k * p)
            _charge(ledger, "trmm", _flops.trmm_flops(p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(p, k, p) + p * p)
        else:
            # Q <- Q - Q_in Bt in one pass (the reference's lincomb + axpy), into a
            # fresh array: the caller's block is never written
            q = _lincomb_device(q_in, eng.Bt, k, p, minus_from=src)
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", m * p)
            _charge(ledger, "trtri", _flops.tri_inverse_flops(p))
            # Q <- Q R^-1 with G = Q^T Q from the same kernel where the block has
            # at most 64 columns (in place: q is this call's own array)
            q = _apply_gram_into(eng, q, fresh_ok=False)
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(k, p, p) + k * p)
            _charge(ledger, "trmm", _flops.trmm_flops(p))
            cross_gram_device(q_in, q, out=eng.Bt)
            _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
            _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
            _charge(ledger, "gemm", _flops.gemm_flops(p, k, p) + p * p)
        its += 1
    if q is None:
        q = a_new.copy()
    q_out = q_in.extended(q)
    b = eng.b_host() if k else np.zeros((0, p))
    r_out = np.block([[r_in, b], [np.zeros((p, k)), eng.r_host()]])
    return QRResult(q_out, r_out, its, shifts, attempts, success=success, orth_error=st.err,
                    pivot_margins=margins, decision_margins=dms, err_history=errs)


def _update_pipelined(eng, q_in, r_in, a_new, m, k, p, width, tol, cfg, ledger):
    """The iteration of chol_qr_update with the fused update pass, one pass
    ahead of the host (as rs_chol_qr): pass i+1 (factor, update pass) is
    enqueued before pass i's status is read, gated on the device by the
    statuses, and the reference's charges / raises are replayed in order."""
    handles, outs = [], []
    # Q' goes straight into the basis' free capacity when it has some (the
    # final [q_in, Q] then needs no copy); else into a fresh array
    tail = q_in._tail_block(p) if q_in._tail_free(p) else None

    def enqueue(i):
        prev = handles[i - 1] if i else None
        h = eng.factor_async(_lib.POLICY_UPDATE, m, width, tol=tol, check_tol=True, stop=(i == cfg.max_iter),
                             update_b=True, gate=eng.gate(prev) if i else None, gate_slot=prev)
        dst = outs[i - 1] if i else None
        if i < cfg.max_iter:
            if i == 0:
                # the first sweep reads the caller's block and writes Q' elsewhere (no copy)
                dst = tail if tail is not None else _fresh_like(a_new, p)
                eng.update_pass(q_in, a_new, initial=False, out=dst, gate=eng.gate(h), gate_slot=h)
            else:
                eng.update_pass(q_in, dst, initial=False, gate=eng.gate(h), gate_slot=h)
        handles.append(h)
        outs.append(dst)

    enqueue(0)
    shifts, attempts, margins, dms, errs = [], [], [], [], []
    its = 0
    success = True
    while True:
        if its + 1 <= cfg.max_iter:
            enqueue(its + 1)
        eng.br_prefetch()   # B and R as of the last enqueued pass (later passes are gated no-ops)
        (st,) = eng.collect([handles[its]])
        errs.append(st.err)
        _charge(ledger, "fro_norm", _flops.frobenius_flops(p))
        if st.code == _lib.CONVERGED:
            break
        if st.code == _lib.CAPPED:
            success = False
            break
        _emit_estimate_warning(st)
        _charge_update(ledger, p, st)
        _raise_for(st)
        dms.append(st.plain_margin)
        attempts.append(st.retries)
        shifts.extend(st.shifts)
        margins.append(st.min_pivot_rel)
        _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
        _charge(ledger, "gemm", m * p)
        _charge(ledger, "trtri", _flops.tri_inverse_flops(p))
        _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
        _charge(ledger, "gemm", _flops.gemm_flops(k, p, p) + k * p)
        _charge(ledger, "trmm", _flops.trmm_flops(p))
        _charge(ledger, "gemm", _flops.gemm_flops(m, k, p))
        _charge(ledger, "gemm", _flops.gemm_flops(m, p, p))
        _charge(ledger, "gemm", _flops.gemm_flops(p, k, p) + p * p)
        its += 1
    if its == 0:
        q_out = q_in.extended(a_new)          # the block itself (copied into the basis)
    elif tail is not None:
        q_out = q_in._claim_tail(p)           # already written in place
    else:
        q_out = q_in.extended(outs[its - 1])
    b_host, r_host = eng.br_host()
    r_out = np.block([[r_in, b_host], [np.zeros((p, k)), r_host]])
    return QRResult(q_out, r_out, its, shifts, attempts, success=success, orth_error=st.err,
                    pivot_margins=margins, decision_margins=dms, err_history=errs)


def _lincomb_device(arr, coeff_dev, k, p, minus_from=None):
    """arr (m x k) @ C with C = Bt already on the device as column-major k x p
    (torch (p, k)), packed into coefficient tiles for libcqr.  With
    `minus_from` (m x p) the result is minus_from - arr @ C in one pass
    (cqr_lincomb_sub: the projection and its axpy, algorithms.py:442-444, with
    the same roundings), written to a fresh array."""
    from ._device import ctx
    from .varray import coeff_tiles

    cx = ctx()
    c = coeff_tiles(coeff_dev, k, p, k)
    out = _fresh_like(arr, p)
    if minus_from is None:
        _lib.check(cx.lib.cqr_lincomb(arr.ptr(), arr.ld, arr.m_local, k, c.data_ptr(), p, 0, out.ptr(), out.ld,
                                      cx.stream), "projection")
    else:
        _lib.check(cx.lib.cqr_lincomb_sub(arr.ptr(), arr.ld, arr.m_local, k, c.data_ptr(), p, minus_from.ptr(),
                                          minus_from.ld, out.ptr(), out.ld, cx.stream), "projection")
    cx.launches += 1
    return out


def panel_widths(n, r_panels):
    """n columns in r contiguous panels, the first n mod r one column wider
    (algorithms.py:461-467)."""
    if not 1 <= r_panels <= n:
        raise ValueError(f"need 1 <= r_panels <= {n}, got {r_panels}")
    base, extra = divmod(n, r_panels)
    return [base + 1] * extra + [base] * (r_panels - extra)


def pn_chol_qr(a, r_panels, cfg=None, ledger=None):
    """Panel scheme: fold chol_qr_update over contiguous column panels
    (algorithms.py:470-505)."""
    cfg = cfg or AlgoConfig()
    a = _device_array(a)
    widths = panel_widths(a.ncols, r_panels)
    q = CudaVectorArray.zeros(a.space, 0, capacity=a.ncols)
    r = np.zeros((0, 0))
    shifts, attempts, profiles, margins, dms, errs = [], [], [], [], [], []
    its = 0
    success = True
    err = None
    start = 0
    for index, width in enumerate(widths):
        panel = a.copy(range(start, start + width))
        start += width
        try:
            res = chol_qr_update(q, r, panel, cfg, ledger)
        except (CholeskyBreakdown, ShiftAttemptLimitError) as exc:
            exc.panel_index = index
            raise
        q, r = res.q, res.r
        its += res.iterations
        shifts.extend(res.shifts_applied)
        attempts.extend(res.shift_attempts)
        profiles.append(res.profile)
        margins.extend(res.pivot_margins)
        dms.extend(res.decision_margins)
        errs.extend(res.err_history)
        err = res.orth_error
        success = success and res.success
    return QRResult(q, r, its, shifts, attempts, success=success, orth_error=err,
                    panel_profiles=profiles, pivot_margins=margins, decision_margins=dms, err_history=errs)
