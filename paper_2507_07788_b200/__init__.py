"""B200-native shifted Cholesky QR (arXiv 2507.07788 hot path).

Drop-in for the reference package's data-parallel path (`cholqr`): the same
algorithm API (`chol_qr2`, `s_chol_qr3`, `rs_chol_qr`, `chol_qr_update`,
`pn_chol_qr`, `AlgoConfig`, `QRResult`, the exception types and the flop
ledger), running on fp64 sm_100a kernels (libcqr.so, C ABI in
include/cqr.h) over device-resident `CudaVectorArray`s.  There is no CPU
fallback: without the built library or a CUDA device the calls raise.
"""

from .algorithms import (
    UNIT_ROUNDOFF,
    AlgoConfig,
    QRResult,
    chol_qr,
    chol_qr2,
    chol_qr_update,
    is_chol_qr,
    panel_widths,
    pn_chol_qr,
    rs_chol_qr,
    s_chol_qr3,
)
from .errors import CholeskyBreakdown, ShiftAttemptLimitError, TriangularSingularError
from .matgen import MatrixSpec, effective_seed, generate, generate_host, random_orthogonal, singular_values
from .mmio import load_matrix_market, save_matrix_market, to_dense_block
from .flops import (
    CATEGORIES,
    FlopLedger,
    IterationProfile,
    LedgerComparison,
    cholesky_flops,
    eig_estimate_flops,
    frobenius_flops,
    gemm_flops,
    ledger_report,
    panel_counts,
    panel_flop_ratio,
    panel_flop_ratio_limit,
    predict_rscholqr,
    rscholqr_counts,
    tri_inverse_flops,
    trmm_flops,
    update_counts,
)
from .varray import CudaVectorArray, VectorSpace

BACKENDS = {"cuda": CudaVectorArray}


def backend_class(name):
    try:
        return BACKENDS[name]
    except KeyError:
        raise ValueError(f"unknown backend {name!r}; expected one of {sorted(BACKENDS)}") from None


def __getattr__(name):
    # k x k API and metrics are imported lazily (they pull in torch device code)
    if name in ("cholesky", "spectral_norm_estimate", "compute_shift", "tri_inverse", "tri_multiply", "frobenius"):
        from . import kernels

        return getattr(kernels, name)
    if name in ("loss_of_orthogonality", "reconstruction_residual", "cholesky_residual", "quality_report",
                "QualityReport"):
        from . import metrics

        return getattr(metrics, name)
    raise AttributeError(name)


__version__ = "0.1.0"
