// Internal (C++) interfaces between the C-ABI layer and the kernel files.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/cqr.h"

#include <string>

namespace cqr {

// record `msg` as cqr_last_error() of this thread and return `code` (cqr_abi.cu)
int set_error(int code, const std::string& msg);

int num_sms();   // of the current device (cqr_device.cu)
// opt the kernel `fn` into `bytes` of dynamic shared memory on the current
// device (cached per device and kernel)
cudaError_t smem_attr(const void* fn, size_t bytes);

// ------------------------------------------------------------- Gram (K1)
struct GramArgs {
  const double* A; int64_t lda; int ka;
  const double* B; int64_t ldb; int kb;
  int64_t rows;       // padded local row count (multiple of 16)
  int self;           // lower-triangular tiles only, mirrored output
  int ntile_i, ntile_j, ntiles, nitems;
  int nsplit;
  int64_t npanels;
  double* ws;         // [nsplit][nitems][2][64*64]
  const int* gate = nullptr;   // launch is a no-op unless *gate == CQR_FACTORED (0)
};
GramArgs gram_plan(const double* A, int64_t lda, int ka, const double* B, int64_t ldb, int kb, int64_t rows,
                   bool self);
size_t gram_workspace_bytes(const GramArgs& a);
cudaError_t gram_launch(GramArgs& a, double* G, int ldg, cudaStream_t stream);

bool gram_pairs_supported(int k);
size_t gram_pairs_ws_bytes(int64_t rows, int k);
cudaError_t gram_pairs_launch(const double* X, int64_t ldx, int k, int64_t rows, double* G, int ldg, double* ws,
                              cudaStream_t s, const int* gate = nullptr);

// ------------------------------------------------------------- row-panel GEMM (K2 building block)
struct GemmArgs {
  const double* X; int64_t ldx; int kx;   // QI m x kx (ldx = column capacity)
  const double* C;                        // kx x n coefficient tiles
  double* Y; int64_t ldy; int n;          // QI m x n
  int64_t rows;                           // padded local row count
  int upper;                              // C upper triangular: skip zero blocks
  int ntile_n;
  int64_t nrow_tiles;
  const int* gate = nullptr;   // launch is a no-op unless *gate == CQR_FACTORED (0)
  const double* Yin = nullptr; int64_t ldyin = 0;   // non-null: Y = Yin - X C (general C only; may alias Y)
};
cudaError_t gemm_launch(GemmArgs& a, cudaStream_t stream);

cudaError_t axpy_launch(double* Y, int64_t ldy, double alpha, const double* X, int64_t ldx, int64_t m, int n,
                        cudaStream_t stream);
cudaError_t pack_tall_launch(const double* src, int64_t lds, int64_t m, int k, double* dst, int64_t ldk,
                             cudaStream_t s);
cudaError_t unpack_tall_launch(const double* src, int64_t ldk, int64_t m, int k, double* dst, int64_t ldd,
                               cudaStream_t s);
cudaError_t gather_cols_launch(const double* src, int64_t lds, const int* idx, int j0, double* dst, int64_t ldd,
                               int dcol0, int n, int64_t m, cudaStream_t s);
cudaError_t pack_coeff_launch(const double* src, int ld, int k, int n, double* dst, cudaStream_t s);

// ------------------------------------------------------------- fused TRMM + Gram (K2, k <= 128)
cudaError_t apply_gram_fused_launch(const double* X, int64_t ldx, int k, const double* Rinv_tiles, double* Q,
                                    int64_t ldq, int64_t rows, double* G, int ldg, double* ws, size_t ws_bytes,
                                    cudaStream_t stream, const int* gate = nullptr);
size_t apply_gram_fused_ws_bytes(int64_t rows, int k);
bool apply_gram_fused_supported(int k);
void set_fused(int mode);
// self Gram for k = 64, register-resident row sweep (cqr_fused.cu)
bool gram_rt_supported(int k, int64_t rows);
size_t gram_rt_ws_bytes(int64_t rows, int k);
cudaError_t gram_rt_launch(const double* X, int64_t ldx, int k, int64_t rows, double* G, int ldg, double* ws,
                           cudaStream_t stream, const int* gate);

// ------------------------------------------------------------- fused update pass (K3)
void set_update_tma(int on);
int update_set_narrow_teams(int on);
int update_set_lag(int on);
int update_set_direct(int on);
int update_set_sr16_from(int q);
bool update_pass_supported(int q, int p);
size_t update_pass_ws_bytes(int64_t rows, int q);
cudaError_t update_pass_launch(const double* Qin, int64_t ldqin, int q, const double* Qb, int64_t ldqb, double* Qo,
                               int64_t ldqo, int p, int64_t rows, const double* Bt, int ldbt, const double* Rinv_tiles,
                               int initial, double* Bt_next, double* G, int ldg, double* ws, cudaStream_t s,
                               const int* gate = nullptr);

// ------------------------------------------------------------- k x k stage (K4)
struct FactorArgs {
  const double* G; int ldg;
  const double* Bt; int ldbt; int q;
  int k;
  int policy;
  int64_t m_global; int shift_width;
  double u, esc; int max_shift_attempts;
  double tol; int check_tol; int stop;
  double est_tol; int est_max_iter;
  double fixed_shift;
  int accumulate; int update_b;
  double* X;       // k*k workspace
  double* part;    // k > 128: per-tile (err^2, max diag G) partials of factor_prep_kernel
  double* W;       // packed-upper workspace (k > smem limit)
  double* Ri;      // packed-upper workspace (k > smem limit)
  double* Rk; double* Rinv; int ldr;   // Rk column-major (ldr); Rinv coefficient tiles
  double* Racc;
  double* B; int ldb;
  double* shifts;
  cqr_factor_status* st;
  const int* gate;   // nullptr, or: skip the pass unless *gate == CQR_FACTORED
  cqr_factor_status* stm; double* shm;   // host-mapped mirrors of the status and shifts (or nullptr)
  // speculative shifted branch (RECOMPUTE policy): a second CTA runs the
  // estimate + shifted attempts into private buffers while CTA 0 tries the
  // plain factorization; CTA 0 publishes its outcome in `pub` (epoch-tagged)
  int spec; unsigned epoch;
  int bt_stage;    // update policy: Bt staged in shared memory after the work area
  double* Rk1; int ldr1; double* W1; double* shifts1; double* pub;
  int ncl;         // CTAs per attempt group (band-cluster path, 128 < k <= 256), else 1
};
cudaError_t factor_launch(FactorArgs& a, cudaStream_t stream);
size_t factor_workspace_bytes(int k);
int factor_profile(unsigned long long* out);
int factor_set_banded(int on);
int factor_set_cluster(int on);
int factor_cluster_profile(unsigned long long* out64);
int factor_step_profile(int cta, long long* out32);

// ------------------------------------------------------------- standalone k x k kernels (cqr_small.cu)
cudaError_t tri_inverse_launch(const double* R, int ldr, int n, double* X, int ldx, cudaStream_t s);
cudaError_t tri_multiply_launch(const double* A, int lda, const double* B, int ldb, int n, double* C, int ldc,
                                cudaStream_t s);
cudaError_t frobenius_launch(const double* X, int ldx, int rows, int cols, double* out, cudaStream_t s);
cudaError_t sum_ranks_launch(const double* parts, int nparts, int64_t n, double* out, cudaStream_t s);
cudaError_t store_mapped_launch(const double* src, int64_t n, double* dst_dev_alias, cudaStream_t s);

// ------------------------------------------------------------- streaming quality measures (K5, cqr_metrics.cu)
bool resid_gram_supported(int k);
size_t resid_gram_ws_bytes(int64_t rows, int k);
cudaError_t resid_gram_launch(const double* Q, int64_t ldq, const double* A, int64_t lda, int k,
                              const double* R_tiles, int64_t rows, double* DtD, int ldd, double* asq, double* ws,
                              cudaStream_t s);

}  // namespace cqr
