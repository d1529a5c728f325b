"""ctypes binding of libcqr.so (the C ABI declared in include/cqr.h).

The product path has no CPU fallback: if the shared library is missing or a
CUDA device is absent, importing the device layer raises.  Symbols are bound
lazily so that `load()` can be exercised on a CPU-only machine (tests check
that every symbol declared in include/cqr.h is exported).
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CQR_LIB (diagnostics only): a variant library built by build.build(defines=..., out=...)
LIB_PATH = os.environ.get("CQR_LIB") or os.path.join(HERE, "libcqr.so")

CQR_OK = 0
CQR_EINVAL = -1
CQR_ECUDA = -2

FACTORED, CONVERGED, CAPPED, BREAKDOWN, SHIFT_LIMIT, TRI_SINGULAR, ASYMMETRIC, ESTIMATED, SKIPPED = range(9)
POLICY_PLAIN, POLICY_SHIFT_ONCE, POLICY_RECOMPUTE, POLICY_UPDATE, POLICY_FIXED_SHIFT, POLICY_ESTIMATE = range(6)

c_double_p = ctypes.c_void_p  # device pointers are passed as integers


class FactorConfig(ctypes.Structure):
    """cqr_factor_config (include/cqr.h)."""

    _fields_ = [
        ("policy", ctypes.c_int32),
        ("shift_width", ctypes.c_int32),
        ("m_global", ctypes.c_int64),
        ("unit_roundoff", ctypes.c_double),
        ("shift_escalation", ctypes.c_double),
        ("max_shift_attempts", ctypes.c_int32),
        ("check_tol", ctypes.c_int32),
        ("tol", ctypes.c_double),
        ("stop", ctypes.c_int32),
        ("accumulate", ctypes.c_int32),
        ("update_b", ctypes.c_int32),
        ("est_max_iter", ctypes.c_int32),
        ("est_tol", ctypes.c_double),
        ("fixed_shift", ctypes.c_double),
        ("gate", ctypes.c_void_p),
        ("status_mirror", ctypes.c_void_p),
        ("shifts_mirror", ctypes.c_void_p),
    ]


class FactorStatus(ctypes.Structure):
    """cqr_factor_status (include/cqr.h)."""

    _fields_ = [
        ("code", ctypes.c_int32),
        ("retries", ctypes.c_int32),
        ("n_shifts", ctypes.c_int32),
        ("pivot_index", ctypes.c_int32),
        ("pivot_value", ctypes.c_double),
        ("err", ctypes.c_double),
        ("norm_est", ctypes.c_double),
        ("last_shift", ctypes.c_double),
        ("min_pivot_rel", ctypes.c_double),
        ("est_calls", ctypes.c_int32),
        ("est_flag", ctypes.c_int32),
        ("escalations", ctypes.c_int32),
        ("singular_index", ctypes.c_int32),
        ("plain_margin", ctypes.c_double),
        ("diag_max", ctypes.c_double),
    ]


class FixedPlan(ctypes.Structure):
    """cqr_fixed_plan (include/cqr.h)."""

    _fields_ = [
        ("passes", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("m", ctypes.c_int64),
        ("X", ctypes.c_void_p),
        ("ldx", ctypes.c_int64),
        ("dst", ctypes.c_void_p * 3),
        ("lddst", ctypes.c_int64 * 3),
        ("G", ctypes.c_void_p),
        ("Rk", ctypes.c_void_p),
        ("Rinv", ctypes.c_void_p),
        ("Racc", ctypes.c_void_p),
        ("Racc0", ctypes.c_void_p),
        ("R_host", ctypes.c_void_p),
        ("ldr", ctypes.c_int32),
        ("use_graph", ctypes.c_int32),
        ("fcfg", ctypes.POINTER(FactorConfig) * 3),
        ("status", ctypes.c_void_p * 3),
        ("fws", ctypes.c_void_p),
        ("fws_bytes", ctypes.c_size_t),
        ("ws", ctypes.c_void_p),
        ("ws_bytes", ctypes.c_size_t),
    ]


# name -> (restype, argtypes); mirrors include/cqr.h one to one
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_SZ = ctypes.c_size_t
SIGNATURES = {
    "cqr_abi_version": (_I, []),
    "cqr_last_error": (ctypes.c_char_p, []),
    "cqr_gram_workspace_bytes": (_SZ, [_I64, _I, _I, _I]),
    "cqr_gram": (_I, [_P, _I64, _I64, _I, _P, _I, _P, _SZ, _P]),
    "cqr_set_gram_pairs": (None, [_I]),
    "cqr_cross_gram": (_I, [_P, _I64, _I, _P, _I64, _I, _I64, _P, _I, _P, _SZ, _P]),
    "cqr_lincomb": (_I, [_P, _I64, _I64, _I, _P, _I, _I, _P, _I64, _P]),
    "cqr_lincomb_sub": (_I, [_P, _I64, _I64, _I, _P, _I, _P, _I64, _P, _I64, _P]),
    "cqr_axpy": (_I, [_P, _I64, ctypes.c_double, _P, _I64, _I64, _I, _P]),
    "cqr_pack_tall": (_I, [_P, _I64, _I64, _I, _P, _I64, _P]),
    "cqr_unpack_tall": (_I, [_P, _I64, _I64, _I, _P, _I64, _P]),
    "cqr_gather_cols": (_I, [_P, _I64, _P, _I, _P, _I64, _I, _I, _I64, _P]),
    "cqr_coeff_doubles": (_SZ, [_I, _I]),
    "cqr_pack_coeffs": (_I, [_P, _I, _I, _I, _P, _P]),
    "cqr_apply_gram_workspace_bytes": (_SZ, [_I64, _I]),
    "cqr_set_fused": (None, [_I]),
    "cqr_apply_gram_launches": (_I, [_I]),
    "cqr_apply_gram_inplace_ok": (_I, [_I]),
    "cqr_apply_gram": (_I, [_P, _I64, _I64, _I, _P, _P, _I64, _P, _I, _P, _SZ, _P]),
    "cqr_apply_gram_gated": (_I, [_P, _I64, _I64, _I, _P, _P, _I64, _P, _I, _P, _SZ, _P, _P]),
    "cqr_update_supported": (_I, [_I, _I]),
    "cqr_update_workspace_bytes": (_SZ, [_I64, _I, _I]),
    "cqr_update_pass": (_I, [_P, _I64, _I, _P, _I64, _I, _I64, _P, _I, _P, _I, _P, _P, _I, _P, _SZ, _P]),
    "cqr_update_pass_to": (_I, [_P, _I64, _I, _P, _I64, _P, _I64, _I, _I64, _P, _I, _P, _I, _P, _P, _I, _P, _SZ, _P]),
    "cqr_update_pass_gated": (_I, [_P, _I64, _I, _P, _I64, _P, _I64, _I, _I64, _P, _I, _P, _I, _P, _P, _I, _P, _SZ,
                                   _P, _P]),
    "cqr_factor_workspace_bytes": (_SZ, [_I]),
    "cqr_debug_factor_profile": (_I, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "cqr_debug_update_tma": (None, [_I]),
    "cqr_debug_factor_banded": (_I, [_I]),
    "cqr_debug_update_narrow_teams": (_I, [_I]),
    "cqr_debug_update_lag": (_I, [_I]),
    "cqr_debug_update_direct": (_I, [_I]),
    "cqr_debug_update_sr16_from": (_I, [_I]),
    "cqr_debug_factor_cluster": (_I, [_I]),
    "cqr_debug_factor_cluster_profile": (_I, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "cqr_debug_factor_step_profile": (_I, [_I, ctypes.c_void_p]),
    "cqr_tri_inverse": (_I, [_P, _I, _I, _P, _I, _P]),
    "cqr_tri_multiply": (_I, [_P, _I, _P, _I, _I, _P, _I, _P]),
    "cqr_frobenius": (_I, [_P, _I, _I, _I, _P, _P]),
    "cqr_sum_ranks": (_I, [_P, _I, _I64, _P, _P]),
    "cqr_store_to_host": (_I, [_P, _I64, _P, _P]),
    "cqr_resid_gram_supported": (_I, [_I]),
    "cqr_resid_gram_workspace_bytes": (_SZ, [_I64, _I]),
    "cqr_resid_gram": (_I, [_P, _I64, _P, _I64, _I64, _I, _P, _P, _I, _P, _P, _SZ, _P]),
    "cqr_fixed_schedule": (_I, [ctypes.POINTER(FixedPlan), _P]),
    "cqr_fixed_graphs": (_I, []),
    "cqr_factor": (_I, [ctypes.POINTER(FactorConfig), _I, _P, _I, _P, _I, _I, _P, _P, _I, _P, _P, _I, _P, _P,
                        _P, _SZ, _P]),
}

_lib = None


def load():
    """Load libcqr.so (raises OSError when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(
                f"{LIB_PATH} not found: build it with `python -m paper_2507_07788_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class CqrError(RuntimeError):
    """A libcqr call failed (bad arguments or a CUDA error)."""


def check(rc, what=""):
    if rc != CQR_OK:
        msg = load().cqr_last_error().decode(errors="replace")
        raise CqrError(f"{what}: libcqr returned {rc}: {msg}")
