/*
 * cqr.h -- C ABI of the B200-native shifted Cholesky QR hot path (libcqr.so).
 *
 * The reference (arXiv 2507.07788 `cholqr` package, Python/NumPy) reaches the
 * tall-side arithmetic through the VectorArray interface
 * (/root/reference/pkg/src/cholqr/varray.py:47-100) and the k x k stage through
 * kernels.py:61-194.  Each entry point below replaces one of those calls; the
 * citation is given per function.  INTEGRATION.md shows the ctypes binding the
 * reference would add (and the one paper_2507_07788_b200/_lib.py uses).
 *
 * Conventions
 *  - All matrices are fp64.  TALL arrays (m rows, k columns, column capacity
 *    ldk >= k) use the row-quad interleaved ("QI") layout:
 *        element (r, c)  at  X[(r/4)*4*ldk + 4*c + r%4]
 *    i.e. blocks of 4 consecutive rows, each block holding its k columns as
 *    contiguous 4-row runs.  A panel of 32 rows is one contiguous 32*ldk run,
 *    so a single bulk (TMA) copy stages it, and the DMMA fragment loads from
 *    the staged copy are bank-conflict free without padding.  Storage covers
 *    m_pad = round_up(m, 16) rows; rows [m, m_pad) must be zero (kernels
 *    process m_pad rows and keep the padding zero).  Base pointers are 16-byte
 *    aligned.  cqr_pack_tall / cqr_unpack_tall convert from / to column-major.
 *  - SMALL outputs (Gram G, Rk, Racc, B) are column-major with a leading
 *    dimension.  Coefficient operands of a tall product (C of lincomb, R^-1)
 *    use the tiled layout written by cqr_pack_coeffs and by cqr_factor:
 *        32 x 64 tiles, tile (kt, nt) at (nt*ceil(k/32) + kt) * 2304,
 *        element (i, j) at +(j%64)*36 + i%32, zero padded
 *    (cqr_coeff_doubles(k, n) doubles).
 *  - All pointers except `cfg` are DEVICE pointers; `stream` is a cudaStream_t
 *    (NULL = legacy default stream).  Every call is asynchronous on `stream`;
 *    results are valid once the stream reaches that point.
 *  - Return value: 0 = launched, CQR_EINVAL = bad arguments, CQR_ECUDA = CUDA
 *    error; cqr_last_error() describes the last failure of the calling thread.
 *  - Not thread-safe per workspace buffer.  Gram outputs are LOCAL partial sums
 *    over the rows passed in; under row sharding the caller sums them across
 *    ranks (NCCL allreduce) before cqr_factor, which reads the lower triangle.
 */
#ifndef CQR_H
#define CQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CQR_ABI_VERSION 10

#define CQR_OK 0
#define CQR_EINVAL (-1)
#define CQR_ECUDA (-2)

/* cqr_factor_status.code */
#define CQR_FACTORED 0     /* Rk, Rinv written; Racc (and B) updated                  */
#define CQR_CONVERGED 1    /* ||X - I||_F < tol on entry: nothing factored            */
#define CQR_CAPPED 2       /* cfg.stop set: only ||X - I||_F measured                 */
#define CQR_BREAKDOWN 3    /* CholeskyBreakdown (kernels.py:25-39, :76-77)            */
#define CQR_SHIFT_LIMIT 4  /* ShiftAttemptLimitError (algorithms.py:47-56,309-310,384) */
#define CQR_TRI_SINGULAR 5 /* TriangularSingularError (kernels.py:42-47,94-99)        */
#define CQR_ASYMMETRIC 6   /* ValueError of spectral_norm_estimate (kernels.py:148-153) */
#define CQR_ESTIMATED 7    /* CQR_POLICY_ESTIMATE: norm_est / est_flag written only     */
#define CQR_SKIPPED 8      /* gated off: cfg.gate pointed at a status that is not FACTORED */

/* cqr_factor_config.policy: which reference factorization rule runs */
#define CQR_POLICY_PLAIN 0      /* cholesky(x)                       algorithms.py:209-210 */
#define CQR_POLICY_SHIFT_ONCE 1 /* cholesky(x + sigma I), sigma from the norm estimate
                                                                     algorithms.py:233-237 */
#define CQR_POLICY_RECOMPUTE 2  /* plain, then recomputed + escalated shifts
                                                                     algorithms.py:344-349, 295-317 */
#define CQR_POLICY_UPDATE 3     /* deflated x = G - Bt^T Bt; sigma = 0, recomputed, escalated
                                                                     algorithms.py:358-397 */
#define CQR_POLICY_FIXED_SHIFT 4 /* cholesky(x + fixed_shift I), breakdown propagates
                                                                     algorithms.py:284 (is_chol_qr) */
#define CQR_POLICY_ESTIMATE 5   /* spectral_norm_estimate(x) only    algorithms.py:279-283 */

typedef struct cqr_factor_config {
  int32_t policy;
  int32_t shift_width;        /* width entering compute_shift (n, or q/p for updates) */
  int64_t m_global;           /* GLOBAL row count (compute_shift, kernels.py:181-194) */
  double unit_roundoff;       /* AlgoConfig.unit_roundoff (1.11e-16)                 */
  double shift_escalation;    /* AlgoConfig.shift_escalation (10)                    */
  int32_t max_shift_attempts; /* AlgoConfig.max_shift_attempts (60)                  */
  int32_t check_tol;          /* 1: report CONVERGED when ||X - I||_F < tol         */
  double tol;                 /* AlgoConfig.effective_tol(width)                     */
  int32_t stop;               /* 1: iteration cap reached, measure only              */
  int32_t accumulate;         /* 1: Racc <- triu(Rk Racc)  (kernels.py:103-114)      */
  int32_t update_b;           /* 1: B <- B + Bt Racc_old   (algorithms.py:445)       */
  int32_t est_max_iter;       /* power-iteration cap (100, kernels.py:126)           */
  double est_tol;             /* power-iteration settling tolerance (1e-2)           */
  double fixed_shift;         /* CQR_POLICY_FIXED_SHIFT: the shift                   */
  const int32_t* gate;        /* NULL, or the code field of an earlier pass's status in
                                 device memory: unless it is CQR_FACTORED the launch only
                                 writes code = CQR_SKIPPED (lets a host loop run ahead) */
  struct cqr_factor_status* status_mirror; /* NULL, or pinned host memory: the kernel also writes the
                                 status there (and the pass's shifts to shifts_mirror), so
                                 the host reads it after the launch without a D2H copy  */
  double* shifts_mirror;      /* pinned host memory, >= max_shift_attempts doubles (with
                                 status_mirror)                                         */
} cqr_factor_config;

typedef struct cqr_factor_status {
  int32_t code;          /* CQR_FACTORED ... CQR_ASYMMETRIC                            */
  int32_t retries;       /* shifted retries this pass (QRResult.shift_attempts entry)  */
  int32_t n_shifts;      /* shifts appended to `shifts` this pass                      */
  int32_t pivot_index;   /* last breakdown: pivot index                                */
  double pivot_value;    /* last breakdown: Schur diagonal (<= 0 or NaN)              */
  double err;            /* ||X - I||_F on entry (X deflated for updates)             */
  double norm_est;       /* spectral norm estimate used for the shift (if any)        */
  double last_shift;     /* ShiftAttemptLimitError.last_shift                          */
  double min_pivot_rel;  /* min diag(Rk)^2 / max diag(X + sigma I): decision margin    */
  int32_t est_calls;     /* spectral estimates run (ledger eig_est)                    */
  int32_t est_flag;      /* 0 converged, 1 stalled, 2 not converged (UserWarning)      */
  int32_t escalations;   /* escalation steps charged one flop each (ledger eig_est)    */
  int32_t singular_index;/* TriangularSingularError.index                             */
  double plain_margin;   /* signed min Schur pivot / max diag(X) of the pass's first
                            attempt (< 0: it broke down): how far the breakdown
                            decision was from rounding noise                        */
  double diag_max;       /* max diag(X)                                              */
} cqr_factor_status;

int cqr_abi_version(void);
const char* cqr_last_error(void);

/* Gram G = X^T X over the local rows, written full and bit-symmetric (lower
 * triangle computed, mirrored) into G (k x k, ldg >= k).  Replaces
 * DenseVectorArray.gramian() (varray.py:150-153, _charged_gramian
 * algorithms.py:159-165). */
size_t cqr_gram_workspace_bytes(int64_t m, int ka, int kb, int self);
int cqr_gram(const double* X, int64_t ldx, int64_t m, int k, double* G, int ldg, void* ws, size_t ws_bytes,
             void* stream);

/* Select the self-Gram schedule: 1 (default) = register-resident row sweep for
 * k = 64, m >= 2^21 and block-row pairs over full-row panels for k <= 256; 2 = block-row
 * pairs for every k <= 256; 0 = 64x64 tile items. */
void cqr_set_gram_pairs(int mode);

/* Cross Gram G = A^T B (ka x kb).  Replaces gramian(other) (varray.py:154-155). */
int cqr_cross_gram(const double* A, int64_t lda, int ka, const double* B, int64_t ldb, int kb, int64_t m, double* G,
                   int ldg, void* ws, size_t ws_bytes, void* stream);

/* Y = X C (m x n), C in coefficient tiles (k x n).  upper=1 declares C upper
 * triangular (TRMM by R^-1; zero blocks are skipped).  Y may alias X only
 * when n <= 64.  Replaces DenseVectorArray.lincomb (varray.py:157-163,
 * algorithms.py:168-174). */
int cqr_lincomb(const double* X, int64_t ldx, int64_t m, int k, const double* C, int n, int upper, double* Y,
                int64_t ldy, void* stream);

/* Y = Yin - X C (m x n; general C in coefficient tiles, k x n): the projection of
 * the update iteration and its subtraction in one pass, `proj = q_in.lincomb(bt);
 * q.axpy(-1.0, proj)` (algorithms.py:442-444; varray.py:157-171), with the same two
 * roundings per element.  Y may alias Yin (not X). */
int cqr_lincomb_sub(const double* X, int64_t ldx, int64_t m, int k, const double* C, int n, const double* Yin,
                    int64_t ldyin, double* Y, int64_t ldy, void* stream);

/* Y += alpha X, in place.  Replaces DenseVectorArray.axpy (varray.py:165-171). */
int cqr_axpy(double* Y, int64_t ldy, double alpha, const double* X, int64_t ldx, int64_t m, int n, void* stream);

/* Layout conversions and column moves (the copy / append / from_numpy /
 * _iter_columns plumbing of varray.py:139-148,291-319). */
int cqr_pack_tall(const double* src, int64_t lds, int64_t m, int k, double* dst, int64_t ldk, void* stream);
int cqr_unpack_tall(const double* src, int64_t ldk, int64_t m, int k, double* dst, int64_t ldd, void* stream);
/* dst(:, dcol0 + j) = src(:, idx ? idx[j] : j0 + j), j < n (idx: device int array) */
int cqr_gather_cols(const double* src, int64_t lds, const int* idx, int j0, double* dst, int64_t ldd, int dcol0,
                    int n, int64_t m, void* stream);
size_t cqr_coeff_doubles(int k, int n);
int cqr_pack_coeffs(const double* src, int ld, int k, int n, double* dst, void* stream);

/* Fused pass: Q = X Rinv (Rinv upper triangular) and G = Q^T Q in one stream
 * over X (Q may alias X).  Replaces the lincomb + gramian pair of one
 * iteration (algorithms.py:350,352 / :238,:240 / :211 + :209). */
size_t cqr_apply_gram_workspace_bytes(int64_t m, int k);
/* Fused TRMM + Gram selection: 2 (default) = the single-kernel pass for
 * k <= 64 only; 1 = also the two-group kernel for 97 <= k <= 128 (slower on
 * B200 than TRMM then Gram there: those passes are FP64-pipe bound); 0 = never
 * fused (TRMM then Gram, for comparisons). */
void cqr_set_fused(int mode);
/* Number of kernel launches one cqr_apply_gram call issues for width k. */
int cqr_apply_gram_launches(int k);
/* 1 when cqr_apply_gram may run in place (Q == X) for width k. */
int cqr_apply_gram_inplace_ok(int k);
int cqr_apply_gram(const double* X, int64_t ldx, int64_t m, int k, const double* Rinv_tiles, double* Q,
                   int64_t ldq, double* G, int ldg, void* ws, size_t ws_bytes, void* stream);
/* Same, as a no-op on the device unless *gate == CQR_FACTORED (gate: the code
 * field of the factor status this pass applies; NULL = always run).  With the
 * gated factor (cqr_factor_config.gate) a host loop can enqueue pass i+1
 * before reading pass i's status. */
int cqr_apply_gram_gated(const double* X, int64_t ldx, int64_t m, int k, const double* Rinv, double* Q,
                         int64_t ldq, double* G, int ldg, void* ws, size_t ws_bytes, const int32_t* gate,
                         void* stream);

/* Fused block-update pass (Alg. 2, p <= 16, 1 <= q <= 512), one sweep over
 * the rows with Q_in read from HBM once:
 *   initial = 1:  Bt_next = Q_in^T Q, G = Q^T Q            (algorithms.py:430-431)
 *   initial = 0:  Q <- (Q - Q_in Bt) R^-1 in place, then
 *                 Bt_next = Q_in^T Q, G = Q^T Q             (algorithms.py:442-450)
 * Bt (q x p, ldbt) and Bt_next (q x p, ld q) may alias; R^-1 in coefficient
 * tiles (p x p); G lower triangle mirrored (ldg). */
int cqr_update_supported(int q, int p);
size_t cqr_update_workspace_bytes(int64_t m, int q, int p);
int cqr_update_pass(const double* Qin, int64_t ldqin, int q, double* Q, int64_t ldq, int p, int64_t m,
                    const double* Bt, int ldbt, const double* Rinv_tiles, int initial, double* Bt_next, double* G,
                    int ldg, void* ws, size_t ws_bytes, void* stream);
/* Same pass reading the block from Q and writing Q' to Qout (iteration mode;
 * Qout must not overlap Q), so the first iteration needs no copy of the
 * caller's block (the reference copies it, algorithms.py:427). */
int cqr_update_pass_to(const double* Qin, int64_t ldqin, int q, const double* Q, int64_t ldq, double* Qout,
                       int64_t ldqout, int p, int64_t m, const double* Bt, int ldbt, const double* Rinv_tiles,
                       int initial, double* Bt_next, double* G, int ldg, void* ws, size_t ws_bytes, void* stream);
/* cqr_update_pass_to gated like cqr_apply_gram_gated. */
int cqr_update_pass_gated(const double* Qin, int64_t ldqin, int q, const double* Q, int64_t ldq, double* Qout,
                          int64_t ldqout, int p, int64_t m, const double* Bt, int ldbt, const double* Rinv_tiles,
                          int initial, double* Bt_next, double* G, int ldg, void* ws, size_t ws_bytes,
                          const int32_t* gate, void* stream);

/* The k x k stage of one pass, one launch: forms X (G, or the deflated
 * G - Bt^T Bt for updates), measures ||X - I||_F, runs the policy's
 * factorization attempts with breakdown detection, power-iteration norm
 * estimate and shift rule (kernels.py:61-194, algorithms.py:187-198,295-317,
 * 369-397), inverts the factor (kernels.py:85-100) and accumulates
 * Racc <- triu(Rk Racc) and B <- B + Bt Racc (two launches: a single-CTA
 * factorization and a one-warp-per-column finish).  Rk, Racc: column-major,
 * ldr >= round_up(k, 32), zero-padded; Rinv: coefficient tiles
 * (cqr_coeff_doubles(k, k), zero-initialised once).  `shifts` receives the shift values tried
 * (capacity max_shift_attempts + 1).  `status` is device memory. */
size_t cqr_factor_workspace_bytes(int k);
/* Diagnostics: globaltimer stamps (ns) of the phases of the last cqr_factor
 * launch (HOST array of 16; synchronous). */
int cqr_debug_factor_profile(unsigned long long* out16);
/* Diagnostics: 1 (default) = the update pass stages narrow sub-panels with one
 * TMA tensor copy each; 0 = per-row-quad bulk copies only (comparisons). */
void cqr_debug_update_tma(int on);
/* Diagnostics: 1 (default) = update passes with bases up to 64 columns run two
 * alternating 4-warp projection teams; 0 = one 8-warp projection group. */
int cqr_debug_update_narrow_teams(int on);
/* Diagnostics: in iteration-mode update passes with one projection group the
 * cross-Gram warps may start sub-panel j only once the projection DMMAs of
 * j + 1 are issued (their DMMAs then fill the projection group's serial tail).
 * 0 = never, 1 = always, 2 (default) = where measured to pay (16-row sub-panels
 * with a 4- or 5-stage ring).  Results are bitwise the same. */
int cqr_debug_update_lag(int mode);
/* Diagnostics: 1 (default) = in the initial pass of an append (full 16-column
 * block, rows a multiple of the sub-panel height) the cross-Gram warps read the
 * staged block in place; 0 = the projection warps copy it into the Q' ring first
 * (the path of ragged / narrower blocks).  Bitwise the same results. */
int cqr_debug_update_direct(int on);
/* Diagnostics: bases of at least q columns (145 <= q <= 193) stage 16-row
 * sub-panels in the update pass, narrower ones 32-row (64-row up to 64 columns). */
int cqr_debug_update_sr16_from(int q);
/* Diagnostics: 1 (default) = the blocked Cholesky in bands of 32 pivots with a
 * rank-32 update between bands; 0 = one lookahead chain over all block steps. */
int cqr_debug_factor_banded(int on);
/* 1 (default): 128 < k <= 256 (96 < k for the estimating policies) factors on
   a thread-block cluster of ceil(k/32) CTAs, one 32-row band each; 2: from
   64 < k (but the update policy with a basis); 0: the single-CTA path (A/B). */
int cqr_debug_factor_cluster(int on);
/* Diagnostics: globaltimer stamps (ns) of the band-cluster path's last attempt,
 * [band][event] (HOST array of 64; synchronous). */
int cqr_debug_factor_cluster_profile(unsigned long long* out64);
/* Diagnostics: out32 == NULL selects the CTA (blockIdx, -1 = off) whose first
 * four blocked-Cholesky steps record clock64 stamps; else copies the [4][8]
 * stamps to the HOST array out32 (synchronous). */
int cqr_debug_factor_step_profile(int cta, long long* out32);
int cqr_factor(const cqr_factor_config* cfg, int k, const double* G, int ldg, const double* Bt, int ldbt, int q,
               double* Rk, double* Rinv, int ldr, double* Racc, double* B, int ldb, double* shifts,
               cqr_factor_status* status, void* ws, size_t ws_bytes, void* stream);

/* Standalone k x k kernels behind the reference's kernel API (the drivers
 * never call them: cqr_factor does the same work inside its launch).
 * Column-major, one CTA.
 *   cqr_tri_inverse:  Rinv = R^-1, R upper triangular with a nonzero diagonal
 *                     (checked by the caller), exact zeros below the diagonal
 *                     -- replaces tri_inverse (kernels.py:85-100);
 *   cqr_tri_multiply: C = triu(A B) for upper-triangular A, B
 *                     -- replaces tri_multiply (kernels.py:103-114);
 *   cqr_frobenius:    out[0] = ||X||_F, fixed-order reduction
 *                     -- replaces frobenius (kernels.py:117-123). */
int cqr_tri_inverse(const double* R, int ldr, int n, double* Rinv, int ldinv, void* stream);
int cqr_tri_multiply(const double* A, int lda, const double* B, int ldb, int n, double* C, int ldc, void* stream);
int cqr_frobenius(const double* X, int ldx, int rows, int cols, double* out, void* stream);

/* Deterministic cross-rank sum of a row-sharded partial (the Gram, or the
 * packed [Bt | G] of an update pass): parts holds the nparts per-rank
 * partials of n doubles back to back (as ncclAllGather leaves them), out[e] =
 * parts[0][e] + parts[1][e] + ... in rank order.  Every rank computes the same
 * bits whatever algorithm the collective used, and bit-symmetric partials sum
 * to a bit-symmetric matrix (the reference's run-to-run
 * determinism, tests/test_algorithms.py:107-113). */
int cqr_sum_ranks(const double* parts, int nparts, int64_t n, double* out, void* stream);

/* host_pinned[0:n] = src[0:n] (device), written by a kernel through the
 * pinned buffer's mapped alias instead of a copy-engine transfer: the small
 * results of a call (R, the status records) leave the GPU without queueing
 * behind a large cudaMemcpy another stream has in flight.  Asynchronous on
 * `stream`; the host reads after synchronizing with it. */
int cqr_store_to_host(const double* src, int64_t n, double* host_pinned, void* stream);

/* Streaming reconstruction residual (K5), k <= 64: one sweep over the rows of
 * Q and A (both QI, m rows) that forms D = A - Q R in registers -- never as a
 * tall array -- and returns DtD = D^T D (k x k, ldd; bit-symmetric) and
 * asq[0] = ||A||_F^2, both summed over CTAs in a fixed order.  R (k x k upper
 * triangular) in coefficient tiles (cqr_pack_coeffs).  Replaces
 * reconstruction_residual's a.copy() / q.lincomb(r) / axpy / diff.gramian()
 * (metrics.py:53-71), which needs two extra m x k arrays.  Local rows only:
 * under row sharding the caller sums DtD and asq over ranks. */
int cqr_resid_gram_supported(int k);
size_t cqr_resid_gram_workspace_bytes(int64_t m, int k);
int cqr_resid_gram(const double* Q, int64_t ldq, const double* A, int64_t lda, int64_t m, int k, const double* R_tiles,
                   double* DtD, int ldd, double* asq, void* ws, size_t ws_bytes, void* stream);

/* Fixed-schedule runs (chol_qr, chol_qr2, s_chol_qr3), enqueued natively.
 * The reference's fixed schedules (algorithms.py:201-244) take no host
 * decision between passes: every pass is Gram -> factor -> TRMM, and the
 * statuses are inspected only after the last one.  cqr_fixed_schedule
 * enqueues the whole run with ONE host call, in the order the per-call API
 * would (bitwise the same kernels and arguments):
 *     Racc <- Racc0;  G = X^T X;
 *     for i < passes:  cqr_factor(fcfg[i], status[i]);
 *                      dst[i] = src_i R_i^-1 (+ G = dst[i]^T dst[i] unless i is the last pass)
 *     R_host <- Racc (k * ldr doubles, mapped stores), when R_host != NULL
 * with src_0 = X and src_i = dst[i-1] (dst[i] may equal src_i where the
 * in-place rules of cqr_apply_gram / cqr_lincomb allow it).
 * use_graph != 0: the run is captured once as a CUDA graph, keyed on every
 * field of the plan and of the three factor configs, and replayed on later
 * calls with the same key (one graph launch instead of ~10 kernel launches).
 * Local rows only: no cross-rank reduction happens inside (world size 1). */
#define CQR_FIXED_MAX_PASSES 3
typedef struct cqr_fixed_plan {
  int32_t passes;            /* 1 (chol_qr), 2 (chol_qr2), 3 (s_chol_qr3)   */
  int32_t k;
  int64_t m;                 /* local rows                                  */
  const double* X;
  int64_t ldx;
  double* dst[CQR_FIXED_MAX_PASSES];
  int64_t lddst[CQR_FIXED_MAX_PASSES];
  double* G;                 /* k x k, ldg = k                              */
  double* Rk;
  double* Rinv;
  double* Racc;
  const double* Racc0;       /* reset source of Racc (k x ldr doubles)      */
  double* R_host;            /* pinned host copy of Racc, or NULL           */
  int32_t ldr;
  int32_t use_graph;
  const cqr_factor_config* fcfg[CQR_FIXED_MAX_PASSES];
  void* status[CQR_FIXED_MAX_PASSES];  /* device slot: status record, then shifts at +96 bytes */
  void* fws;
  size_t fws_bytes;
  void* ws;                  /* Gram / apply_gram workspace                 */
  size_t ws_bytes;
} cqr_fixed_plan;
int cqr_fixed_schedule(const cqr_fixed_plan* plan, void* stream);
/* number of CUDA graphs cached by cqr_fixed_schedule (this process) */
int cqr_fixed_graphs(void);

#ifdef __cplusplus
}
#endif

#endif /* CQR_H */
