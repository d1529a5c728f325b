// K4: the k x k stage of one pass, in one single-CTA launch.
//
// Replaces the reference's small dense kernels and the per-pass decision
// logic that sits between two tall passes:
//   _deflated_gramian            algorithms.py:358-366   (update policy)
//   frobenius / _identity_distance kernels.py:117-123, algorithms.py:197-198
//   cholesky (breakdown on `not s > 0`)          kernels.py:61-82
//   spectral_norm_estimate (power iteration)      kernels.py:126-178
//   compute_shift (Python max semantics)          kernels.py:181-194
//   _shifted                                      algorithms.py:187-194
//   _retry_with_recomputed_shift                  algorithms.py:295-317
//   _update_factor_attempts                       algorithms.py:369-397
//   tri_inverse                                   kernels.py:85-100
//   tri_multiply, b + bt @ r                      kernels.py:103-114, algorithms.py:445
// The loop control that stays on the host (iteration count, QRResult) only
// reads the status record this kernel writes.
//
// Two launches per pass.  `factor_kernel` (one CTA, 384 threads) forms X,
// measures it, runs the policy's factorization attempts and writes Rk;
// `factor_finish_kernel` (one warp per column, k/8 CTAs) does the column-
// independent rest: B += Bt Racc, Racc <- triu(Rk Racc) and the inverse by
// column back substitution (R Rinv = I), reading Rk from L2.
//
// Storage: X (the symmetric input) is kept in a k x k global workspace (L2
// resident) so shifted retries restart from it.  The Cholesky is
// right-looking (pivot check, row scaled, rank-1 trailing update, two block
// barriers per step) on a packed upper triangle in shared memory:
//   k <= 128      : the whole packed triangle (66 KB);
//   128 < k <= 256: the first 32 rows are factored as a panel in shared
//                   memory and written to Rk, the trailing (k-32) matrix
//                   S = X22 - R12^T R12 is formed with DMMA from the panel in
//                   L2 straight into shared memory (202 KB at k = 256), and
//                   the unblocked loop continues there;
//   k > 256       : packed triangle in global memory (slow generic path).
// All reductions use a fixed order: bitwise reproducible run to run.
#include <algorithm>
#include <cmath>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int FK_THREADS = 384;
constexpr int FK_NW = FK_THREADS / 32;
constexpr int FK_SMEM_K = 128;   // whole packed triangle in shared memory
constexpr int FK_BIG_K = 256;    // panel + shared trailing matrix
constexpr int FK_MAX_K = 2048;
// FactorArgs.pub (64 doubles): [0] group 0's outcome flag, [1..3] its plain
// margin / pivot; group 1's status record
constexpr int PUB_ST1 = 24;      // cqr_factor_status of the speculative group (96 bytes)

__host__ __device__ __forceinline__ int64_t pk(int i, int c) { return (int64_t)c * (c + 1) / 2 + i; }

// phase timestamps of the last factor launch (globaltimer ns), for profiling;
// slots 9..12 accumulate SM cycles of the blocked-Cholesky step phases
__device__ unsigned long long g_fprof[16];
// 1: bands of 4 block rows with a rank-32 update between bands; 0: one
// lookahead chain over every block step (cqr_debug_factor_banded)
__device__ int g_banded = 1;
// band-cluster path, group 0: globaltimer stamps per band of the last attempt
// [band][0 start, 1 band loaded, 2 last upstream band received, 3 updates
//  applied, 4 band factored, 5 published, 6 outcome agreed]
__device__ unsigned long long g_cprof[8][8];
// per-step clock64 stamps of chol_blocked in the last band of the cluster
// (diagnostics): [step][0 start, 1 warp 0 solved, 2 warp 0 updated, 3 diag
// done, 4 workers' panel done, 5 workers' update done, 6 step barrier passed]
__device__ long long g_sprof[4][8];
__device__ int g_sprof_cta = -1;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum: lane-0 warp partials, then every thread adds the
// 16 partials in the same order (identical result in every thread).
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < FK_NW; ++w) s += red[w];
  return s;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ double block_max(double v, double* red) {
  v = warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = -INFINITY;
#pragma unroll
  for (int w = 0; w < FK_NW; ++w) s = fmax(s, red[w]);
  return s;
}

// compute_shift (kernels.py:194): ((11 * N) * u) * norm, then Python max with 2u.
__device__ __forceinline__ double shift_value(int64_t m, int64_t w, double norm, double u) {
  const double N = (double)(m * w + w * (w + 1));
  const double s = __dmul_rn(__dmul_rn(__dmul_rn(11.0, N), u), norm);
  return py_max(s, 2.0 * u);
}

struct FState {
  int code, retries, n_shifts, pivot_index, est_calls, est_flag, escalations, singular_index, attempts;
  double pivot_value, err, norm_est, last_shift, min_pivot_rel, sigma, plain_margin, diag_max, min_pivot;
  double fro;   // ||X||_F (k > 128: from factor_prep_kernel's partials)
  // speculative CTA: the flag CTA 0 publishes and the value meaning "plain attempt held"
  const volatile unsigned long long* spec_flag;
  unsigned long long spec_done;
  int aborted;
  // band-cluster path (csize > 1): this CTA's rank = its 32-row band, the
  // attempt sequence number (uniform over the cluster)
  int crank, csize;
  unsigned seq;
  double* crec;   // [2][8][4] attempt records, written into every CTA of the cluster
  unsigned* crows;   // [8] block rows published by each earlier band (seq * 16 + rows; + 15: failed)
};

__device__ __forceinline__ void cmark(const FState& fs, int slot) {
  if (threadIdx.x == 0 && blockIdx.x < 8 && fs.csize > 1 && (int)blockIdx.x < fs.csize) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cprof[fs.crank][slot] = t;
  }
}

// ---------------------------------------------------------------------------
// thread-block cluster helpers (band-cluster path)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// st.shared::cluster of one double into CTA `cta`'s copy of the shared variable at `p`
__device__ __forceinline__ void dsmem_st(double* p, int cta, double v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
// generic address of `p` in CTA `cta`'s shared memory window (ld / st.shared::cluster operand)
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, int cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(cta));
  return ra;
}
__device__ __forceinline__ double dsmem_ld(uint32_t ra) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}
// release store of a u32 into CTA `cta`'s copy of the shared variable at `p`
__device__ __forceinline__ void dsmem_st_release(unsigned* p, int cta, unsigned v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(dsmem_addr(p, cta)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cluster(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// Speculative CTA only: has CTA 0's plain attempt already succeeded?  Polled at
// band boundaries (all threads must call it; it holds a barrier).
__device__ bool spec_should_stop(FState& fs) {
  if (fs.spec_flag == nullptr) return false;
  if (threadIdx.x == 0 && !fs.aborted && *fs.spec_flag == fs.spec_done) fs.aborted = 1;
  __syncthreads();
  return fs.aborted != 0;
}

// Unblocked right-looking Cholesky of the packed upper n x n matrix W (already
// loaded).  Pivot indices are reported offset by `off`; `smin` carries the
// smallest pivot seen so far.  Returns false (pivot recorded) on breakdown.
__device__ bool chol_packed(double* W, int n, int off, double* rowbuf, double& smin, FState& fs) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int j = 0; j < n; ++j) {
    const double s = W[pk(j, j)];
    if (!(s > 0.0)) {
      if (tid == 0) { fs.pivot_index = j + off; fs.pivot_value = s; }
      __syncthreads();
      return false;
    }
    smin = fmin(smin, s);
    const double d = sqrt(s);
    for (int c = j + 1 + tid; c < n; c += FK_THREADS) {
      const double v = W[pk(j, c)] / d;
      W[pk(j, c)] = v;
      rowbuf[c] = v;
    }
    __syncthreads();
    if (tid == 0) W[pk(j, j)] = d;
    for (int c = j + 1 + warp; c < n; c += FK_NW) {
      const double rc = rowbuf[c];
      double* col = W + pk(0, c);
      for (int i = j + 1 + lane; i <= c; i += 32) col[i] -= rowbuf[i] * rc;
    }
    __syncthreads();
  }
  return true;
}

// ---------------------------------------------------------------------------
// Blocked right-looking Cholesky on a block-packed upper triangle in shared
// memory: 8x8 blocks (I <= J) stored full (64 doubles, column-major inside),
// block (I, J) at ((J (J+1))/2 + I) * 64.  Each block step factors an 8-pivot
// panel (block row P) with scalar updates restricted to the panel, then
// applies the rank-8 update to every trailing block with two DMMA.8x8x4.
// Rows/columns >= n are identity padding (pivots 1, no coupling).
__device__ __forceinline__ int boff(int I, int J) { return (J * (J + 1) / 2 + I) * 64; }
__device__ __forceinline__ int belem(int i, int c) { return boff(i >> 3, c >> 3) + (c & 7) * 8 + (i & 7); }

// Column J of linear upper-triangle block index blk = J (J + 1) / 2 + I, I <= J:
// an approximate root from the MUFU reciprocal square root, then an exact
// integer fix-up (the IEEE sqrtf with its slow-path branch showed up as a hot
// spot of the block loops under ncu source sampling).
__device__ __forceinline__ int tri_col(int blk) {
  const float x = 8.0f * (float)blk + 1.0f;
  int J = (int)((x * __frsqrt_rn(x) - 1.0f) * 0.5f);
  J = max(J, 0);
  while ((J + 1) * (J + 2) / 2 <= blk) ++J;
  while (J * (J + 1) / 2 > blk) --J;
  return J;
}

// The two k-steps' A (or B) fragments of an 8x8 block for lane (g, t): rows t and
// t + 4 of block column g, at p[0] and p[4] for p = block + 8 g + t.  Loading
// the +4 element first on lanes with (g >> 1) & 1 spreads each half-warp's
// loads over all 32 banks (g and g + 2 share banks at the same offset), halving
// the shared-memory wavefronts of every fragment load; the values are then
// swapped back, so each DMMA sees exactly the operands it saw before.
__device__ __forceinline__ void frag_pair(const double* p, int g, double& lo, double& hi) {
  const bool sw = (g >> 1) & 1;
  const double x = p[sw ? 4 : 0];
  const double y = p[sw ? 0 : 4];
  lo = sw ? y : x;
  hi = sw ? x : y;
}

// The C fragment of an 8x8 block for lane (g, t): elements (g, 2t) and
// (g, 2t + 1) at p[0] and p[8] for p = block + 16 t + g.  Lanes with odd t
// take the +8 element first, so a half-warp's accesses land on 8 distinct
// 8-byte bank pairs instead of 4 (2-way instead of 4-way conflicts); the
// values are the same.
__device__ __forceinline__ void cfrag_load(const double* p, int t, double (&c)[2]) {
  const bool sw = t & 1;
  const double x = p[sw ? 8 : 0];
  const double y = p[sw ? 0 : 8];
  c[0] = sw ? y : x;
  c[1] = sw ? x : y;
}
__device__ __forceinline__ void cfrag_store(double* p, int t, const double (&c)[2]) {
  const bool sw = t & 1;
  p[sw ? 8 : 0] = sw ? c[1] : c[0];
  p[sw ? 0 : 8] = sw ? c[0] : c[1];
}

// Rotations of an 8-vector by a lane-dependent amount (three conditional
// stages, register selects only): rot_right gives x[i] = v[(i - r) & 7],
// rot_left x[i] = v[(i + r) & 7].
__device__ __forceinline__ void rot_right8(double (&v)[8], int r) {
#pragma unroll
  for (int s = 1; s < 8; s <<= 1) {
    double w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (r & s) ? v[(i - s) & 7] : v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = w[i];
  }
}
__device__ __forceinline__ void rot_left8(double (&v)[8], int r) {
#pragma unroll
  for (int s = 1; s < 8; s <<= 1) {
    double w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (r & s) ? v[(i + s) & 7] : v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = w[i];
  }
}

// block layouts: the full upper triangle, or a band of the first 4 block rows
struct LayoutUpper {
  __device__ __forceinline__ int operator()(int I, int J) const { return boff(I, J); }
};
struct LayoutBand4 {
  __device__ __forceinline__ int operator()(int I, int J) const { return (J * 4 + I) * 64; }
};

// 8x8 diagonal block factorization (block column-major in shared memory).
// Pivot j is s = Schur diagonal, breakdown on `not s > 0` (kernels.py:76);
// d = s * rsqrt(s), the row is scaled by rsqrt(s) and the reciprocal is kept
// in inv[] for the panel solve.  Returns 1 (warp-uniform) on breakdown.
// One lane does it with the 36 upper entries in registers: 8 dependent pivots
// cost ~1100 cycles this way against ~3100 with the block spread over the
// warp, where 64-bit shuffles serialise on the MIO pipe
// (profiles/r01_diag_block.jsonl).  Only lane 0's smin is used afterwards.
__device__ __forceinline__ constexpr int pk8(int i, int c) { return c * (c + 1) / 2 + i; }
__device__ int diag_block_warp(double* D, int P, int n, int off, double* inv, double& smin, FState& fs) {
  const int lane = threadIdx.x & 31;
  int bad = 0;
  if (lane == 0) {
    double a[36];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int i = 0; i <= c; ++i) a[pk8(i, c)] = D[c * 8 + i];
    // all 8 pivots run unconditionally (no early exit to serialise the
    // schedule); the first failing pivot is recorded with predicated moves and
    // everything computed after it is discarded
    int bj = -1;
    double bv = 0.0, sm = smin;
    double rr[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = 8 * P + jj;
      const double sj = a[pk8(jj, jj)];
      const bool live = j < n;
      if (live && !(sj > 0.0) && bj < 0) { bj = j; bv = sj; }
      if (live && bj < 0) sm = fmin(sm, sj);
      const double r = rsqrt(sj);
      rr[jj] = r;
      // the next pivot's chain first (scale (jj, jj+1), update (jj+1, jj+1)),
      // then the rest of the step: the same operations in the same order per
      // element, listed so that the schedule starts the dependent chain early
      if (jj + 1 < 8) {
        a[pk8(jj, jj + 1)] *= r;
        a[pk8(jj + 1, jj + 1)] -= a[pk8(jj, jj + 1)] * a[pk8(jj, jj + 1)];
      }
      a[pk8(jj, jj)] = sj * r;
#pragma unroll
      for (int c = jj + 2; c < 8; ++c) a[pk8(jj, c)] *= r;
#pragma unroll
      for (int c = jj + 1; c < 8; ++c)
#pragma unroll
        for (int i = jj + 1; i <= c; ++i)
          if (!(i == jj + 1 && c == jj + 1)) a[pk8(i, c)] -= a[pk8(jj, i)] * a[pk8(jj, c)];
    }
    if (bj >= 0) {
      fs.pivot_index = bj + off;
      fs.pivot_value = bv;
      bad = 1;
    } else {
      smin = sm;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) inv[8 * P + jj] = rr[jj];
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int i = 0; i <= c; ++i) D[c * 8 + i] = a[pk8(i, c)];
    }
  }
  bad = __shfl_sync(0xffffffffu, bad, 0);
  __syncwarp();
  return bad;
}

// Blocked right-looking Cholesky over block rows [0, nbr) of an nb x nb block
// upper triangle (rows/cols >= n are identity padding).  Per block step P:
//   (b) all threads solve the panel R_PP^T R_PJ = W_PJ column by column;
//   (c) the trailing blocks (I, J), P < I < nbr, I <= J get the rank-8 update
//       with two DMMA.8x8x4 each -- warp 0 takes block (P+1, P+1) first and
//       then factors it (lookahead), the other warps take the rest.
// Two block barriers per 8 pivots.
// the per-step hook of chol_blocked: called by every thread once block row P
// is final (after the step's barrier); the band-cluster path publishes the row
struct NoRowHook {
  __device__ __forceinline__ void operator()(int) const {}
};

template <typename Lay, typename Hook = NoRowHook>
__device__ bool chol_blocked(double* Wb, int n, int nb, int P0, int nbr, int off, double* inv, double& smin,
                             FState& fs, Lay lay, int* flag, Hook hook = Hook()) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  if (warp == 0) {
    const int f = diag_block_warp(Wb + lay(P0, P0), P0, n, off, inv, smin, fs);
    if (lane == 0) *flag = f;
  }
  __syncthreads();
  if (*flag) return false;
  // speculative CTA: thread 0 polls CTA 0's flag once per step without
  // waiting on it -- the load issued in one step is tested in the next
  unsigned long long spec_pend = 0;
  bool spec_have = false;
  constexpr int NWKR = FK_NW - 1;                    // worker warps 1.. (panel solve)
  constexpr int NWK = FK_NW - FK_NW / 4;             // of which the trailing-update warps (warp % 4 != 0)
  const bool sp = (int)blockIdx.x == g_sprof_cta && P0 == 0;
  for (int P = P0; P < nbr; ++P) {
    const long long c0 = clock64();
    if (sp && tid == 0 && P < 4) g_sprof[P][0] = c0;
    int spec_abort = 0;
    if (tid == 0 && fs.spec_flag != nullptr) {
      if (spec_have && spec_pend == fs.spec_done) { spec_abort = 1; fs.aborted = 1; }
      spec_pend = *fs.spec_flag;
      spec_have = true;
    }
    const double* D = Wb + lay(P, P);
    const double* iv = inv + 8 * P;
    const int ncb = nb - 1 - P;                      // block columns right of the diagonal
    const int nrows_b = nbr - 1 - P;                 // band rows below P
    const bool ahead = nrows_b > 0;                  // warp 0 runs the lookahead chain
    // panel row P: R_PJ = R_PP^{-T} W_PJ, one column per thread (8-long chain)
    // (col and the lane have the same parity.  The column's 8 rows are read and
    // written in an order rotated by (lane >> 1) & 7: with the column stride of
    // 8 doubles a half-warp then touches 16 distinct bank pairs per access,
    // against 2 in row order -- 16-way conflicts, the panel solve's cost)
    auto solve_col = [&](int col) {
      double* blk = Wb + lay(P, P + 1 + (col >> 3)) + (col & 7) * 8;   // column (col & 7), rows 0..7
      const int rot = (lane >> 1) & 7;
      double y[8], dl[28], ivr[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) y[q] = blk[(q + rot) & 7];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) ivr[jj] = iv[jj];
#pragma unroll
      for (int jj = 1, e = 0; jj < 8; ++jj)
#pragma unroll
        for (int l = 0; l < jj; ++l, ++e) dl[e] = D[jj * 8 + l];
      rot_right8(y, rot);   // y[jj] = row jj
      // right-looking order (per element the same subtractions, ascending l)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        y[jj] *= ivr[jj];
#pragma unroll
        for (int l2 = jj + 1; l2 < 8; ++l2) y[l2] -= dl[l2 * (l2 - 1) / 2 + jj] * y[jj];
      }
      rot_left8(y, rot);    // y[q] = row (q + rot) & 7
#pragma unroll
      for (int q = 0; q < 8; ++q) blk[(q + rot) & 7] = y[q];
    };
    int f = 0;
    if (warp == 0) {
      // ---- the critical chain of the step, alone on warp 0:
      // solve block (P, P+1) -> rank-8 update of (P+1, P+1) -> factor it
      if (ahead) {
        if (lane < 8) {
          // block (P, P+1) on 8 lanes: row order (at most 4-way conflicts for 8 lanes,
          // cheaper than the rotation selects on the critical chain)
          double* blk = Wb + lay(P, P + 1) + lane * 8;
          double v[8], dl[28], ivr[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) { v[jj] = blk[jj]; ivr[jj] = iv[jj]; }
#pragma unroll
          for (int jj = 1, e = 0; jj < 8; ++jj)
#pragma unroll
            for (int l = 0; l < jj; ++l, ++e) dl[e] = D[jj * 8 + l];
          // right-looking: row jj's value is final once y[0..jj-1] are out; each
          // element still subtracts its terms in ascending l (the same rounding
          // as the row-by-row form), but the chain is 2 dependent ops per row
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            v[jj] *= ivr[jj];
#pragma unroll
            for (int l2 = jj + 1; l2 < 8; ++l2) v[l2] -= dl[l2 * (l2 - 1) / 2 + jj] * v[jj];
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) blk[jj] = v[jj];
        }
        __syncwarp();
        // (P, P+1) is final: release it to the workers' updates of block row P+1
        asm volatile("bar.arrive 2, %0;" ::"n"(FK_THREADS) : "memory");
        if (sp && lane == 0 && P < 4) g_sprof[P][1] = clock64();
        const double* pa = Wb + lay(P, P + 1) + g * 8 + t;
        double* pc = Wb + lay(P + 1, P + 1) + 2 * t * 8 + g;
        double c2[2];
        cfrag_load(pc, t, c2);
        double p0, p1;
        frag_pair(pa, g, p0, p1);
        dmma(c2, -p0, p0);
        dmma(c2, -p1, p1);
        cfrag_store(pc, t, c2);
        __syncwarp();
        const long long cd = clock64();
        if (sp && lane == 0 && P < 4) g_sprof[P][2] = cd;
        f = diag_block_warp(Wb + lay(P + 1, P + 1), P + 1, n, off, inv, smin, fs);
        if (sp && lane == 0 && P < 4) g_sprof[P][3] = clock64();
        if (lane == 0 && blockIdx.x == 0) atomicAdd(&g_fprof[12], (unsigned long long)(clock64() - cd));
      }
      if (lane == 0) *flag = f | spec_abort;
    } else {
      // ---- workers: the rest of panel row P, then the trailing update
      // (the 9 warps outside warp 0's SM sub-partition: warps 4 and 8 would take
      // its issue slots while it runs the diagonal chain)
      const int first = ahead ? 8 : 0;               // warp 0 solves block (P, P+1)
      if (warp & 3)
        for (int col = first + 32 * (warp - 1 - (warp >> 2)) + lane; col < 8 * ncb; col += 32 * NWK) solve_col(col);
      asm volatile("bar.sync 1, %0;" ::"n"(32 * NWKR) : "memory");   // panel row P final (but (P, P+1))
      const long long c1 = clock64();
      if (tid == 32 && blockIdx.x == 0) g_fprof[9] += (unsigned long long)(c1 - c0);
      if (sp && tid == 32 && P < 4) g_sprof[P][4] = c1;
      if (ahead) asm volatile("bar.sync 2, %0;" ::"n"(FK_THREADS) : "memory");   // (P, P+1) from warp 0
      // trailing rank-8 update of blocks (I, J), P < I < nbr, I <= J < nb, but (P+1, P+1)
      const int nblk = (nrows_b == ncb) ? ncb * (ncb + 1) / 2 : nrows_b * ncb - nrows_b * (nrows_b - 1) / 2;
      auto decode = [&](int blk, int& I, int& Jb) {
        if (nrows_b == ncb) {
          int J = tri_col(blk);
          I = P + 1 + (blk - J * (J + 1) / 2);
          Jb = P + 1 + J;
        } else {
          // band rows: row r of the band has ncb - r blocks
          int r = 0, rem = blk;
          while (rem >= ncb - r) { rem -= ncb - r; ++r; }
          I = P + 1 + r;
          Jb = I + rem;
        }
      };
      // the 9 warps outside warp 0's SM sub-partition (warp % 4 != 0); warps 4
      // and 8 stay out so their DMMAs do not share warp 0's FP64 pipe (its
      // dependent pivot chain runs 2-3x slower otherwise).  blk 0 = (P+1, P+1)
      // is warp 0's.
      const int wk = warp - 1 - (warp >> 2);
      for (int blk = ((warp & 3) ? 1 + wk : nblk); blk < nblk; blk += 2 * NWK) {
        const int blk2 = blk + NWK;
        const bool two = blk2 < nblk;
        int I0, J0, I1 = 0, J1 = 0;
        decode(blk, I0, J0);
        if (two) decode(blk2, I1, J1);
        const double* pa0 = Wb + lay(P, I0) + g * 8 + t;
        const double* pb0 = Wb + lay(P, J0) + g * 8 + t;
        double* pc0 = Wb + lay(I0, J0) + 2 * t * 8 + g;
        double c0r[2];
        cfrag_load(pc0, t, c0r);
        double a00, a01, b00, b01;
        frag_pair(pa0, g, a00, a01);
        frag_pair(pb0, g, b00, b01);
        a00 = -a00; a01 = -a01;
        double c1r[2] = {0.0, 0.0}, a10 = 0.0, a11 = 0.0, b10 = 0.0, b11 = 0.0;
        double* pc1 = pc0;
        if (two) {
          const double* pa1 = Wb + lay(P, I1) + g * 8 + t;
          const double* pb1 = Wb + lay(P, J1) + g * 8 + t;
          pc1 = Wb + lay(I1, J1) + 2 * t * 8 + g;
          cfrag_load(pc1, t, c1r);
          frag_pair(pa1, g, a10, a11);
          frag_pair(pb1, g, b10, b11);
          a10 = -a10; a11 = -a11;
        }
        dmma(c0r, a00, b00);
        if (two) dmma(c1r, a10, b10);
        dmma(c0r, a01, b01);
        if (two) dmma(c1r, a11, b11);
        cfrag_store(pc0, t, c0r);
        if (two) cfrag_store(pc1, t, c1r);
      }
      if (tid == 32 && blockIdx.x == 0) g_fprof[10] += (unsigned long long)(clock64() - c1);
      if (sp && tid == 32 && P < 4) g_sprof[P][5] = clock64();
    }
    __syncthreads();
    if (sp && tid == 0 && P < 4) g_sprof[P][6] = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) g_fprof[11] += 1;
    if (*flag) return false;
    hook(P);
  }
  return true;
}

// Rank-(8 (P1-P0)) update of the trailing blocks after a band of block rows
// [P0, P1) is final: C(I, J) -= sum_P R(P, I)^T R(P, J) for P1 <= I <= J < nb.
// Each element sees the same DMMA chain (P ascending, k4 0 then 4) as P1-P0
// separate rank-8 steps, so the result is bitwise the unbanded one.
// A warp takes a 2 x 2 group of blocks (I0, I1) x (J0, J1): four independent
// accumulator chains, and each fragment it loads feeds two DMMAs (5 shared
// loads per 4 DMMAs with the C fragments, against 9 for blocks taken one or
// two at a time; those ran at ~45 cycles per DMMA per sub-partition, 3x the
// pipe's 16).  On diagonal groups the (I1, J0) block lies below the diagonal:
// it is computed and dropped.
template <typename Lay>
__device__ void band_trailing_update(double* Wb, int nb, int P0, int P1, Lay lay) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int tn = nb - P1;
  const int G = (tn + 1) >> 1;                 // group rows / columns
  const int ngroups = G * (G + 1) / 2;
  for (int gidx = warp; gidx < ngroups; gidx += FK_NW) {
    const int gj = tri_col(gidx), gi = gidx - gj * (gj + 1) / 2;
    const int I[2] = {P1 + 2 * gi, P1 + 2 * gi + 1};
    const int J[2] = {P1 + 2 * gj, P1 + 2 * gj + 1};
    bool live[2][2];
    double c[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        live[x][y] = I[x] <= J[y] && J[y] < nb;
        const double* pc = Wb + lay(live[x][y] ? I[x] : P1, live[x][y] ? J[y] : P1) + 2 * t * 8 + g;
        cfrag_load(pc, t, c[x][y]);
        if (!live[x][y]) { c[x][y][0] = 0.0; c[x][y][1] = 0.0; }
      }
#pragma unroll
    for (int q = 0; q < 4; ++q) {   // bands are at most 4 block rows: unrolled, loads hoisted
      const int P = P0 + q;
      if (P >= P1) break;
      double a[2][2], bb[2][2];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int Ix = I[x] < nb ? I[x] : P1;
        const int Jx = J[x] < nb ? J[x] : P1;
        frag_pair(Wb + lay(P, Ix) + g * 8 + t, g, a[x][0], a[x][1]);
        frag_pair(Wb + lay(P, Jx) + g * 8 + t, g, bb[x][0], bb[x][1]);
        a[x][0] = -a[x][0];
        a[x][1] = -a[x][1];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) dmma(c[x][y], a[x][h], bb[y][h]);
    }
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
        if (live[x][y]) {
          cfrag_store(Wb + lay(I[x], J[y]) + 2 * t * 8 + g, t, c[x][y]);
        }
  }
}

// Banded right-looking Cholesky of the nb x nb block upper triangle: bands of
// 4 block rows (32 pivots) are factored with in-band rank-8 steps, then the
// rest of the matrix gets one rank-32 update per band (4x fewer barriers and
// 4x more DMMA per block load than rank-8 steps over the whole matrix).
// `nbr` limits the factorization to block rows [0, nbr).
template <typename Lay, typename Hook = NoRowHook>
__device__ bool chol_banded(double* Wb, int n, int nb, int nbr, int off, double* inv, double& smin, FState& fs,
                            Lay lay, int* flag, Hook hook = Hook()) {
  for (int P0 = 0; P0 < nbr; P0 += 4) {
    const int P1 = min(nbr, P0 + 4);
    if (!chol_blocked(Wb, n, nb, P0, P1, off, inv, smin, fs, lay, flag, hook)) return false;
    if (P1 < nbr) {
      band_trailing_update(Wb, nb, P0, P1, lay);
      __syncthreads();
    }
  }
  return true;
}

__device__ void store_blocked(const double* Wb, int n, int off, double* Rk, int ldr) {
  // n <= 256; a warp per column pair, all shared loads of the pair before the stores
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 2 * warp; c0 < n; c0 += 2 * FK_NW) {
    double v[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + h, i = lane + 32 * u;
        v[h][u] = (c < n && i <= c) ? Wb[belem(i, c)] : 0.0;
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + h, i = lane + 32 * u;
        if (c < n && i <= c) Rk[(int64_t)(c + off) * ldr + off + i] = v[h][u];
      }
  }
}

// identity padding for rows / columns [n, 8 ceil(n/8)) of a block-packed matrix
__device__ void pad_blocked(double* Wb, int n) {
  const int np = (n + 7) & ~7;
  if (np == n) return;
  for (int e = threadIdx.x; e < (np - n) * np; e += FK_THREADS) {
    const int c = e % np, i = n + e / np;    // row i >= n
    if (c >= i) Wb[belem(i, c)] = (i == c) ? 1.0 : 0.0;
    else Wb[belem(c, i)] = 0.0;              // column i >= n, row c < i
  }
}

// Packed n x n upper W (rows/cols offset by `off` in R) -> Rk columns.
__device__ void store_packed(const double* W, int n, int off, double* Rk, int ldr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = warp; c < n; c += FK_NW)
    for (int i = lane; i <= c; i += 32) Rk[(int64_t)(c + off) * ldr + off + i] = W[pk(i, c)];
}

constexpr int FK_PANEL = 32;
constexpr int FK_BAND_K = 768;   // banded global path: the 32-row band fits in shared memory

// 256 < k <= 768: right-looking Cholesky by 32-row bands with the working
// matrix W (upper triangle, column-major k x k, L2 resident).  Per band:
// stage rows [r0, r0+32) x cols [r0, k) in shared memory (band layout),
// factor them with in-band rank-8 steps (chol_banded), write them to Rk, then
// apply the rank-32 update to the trailing upper triangle of W with DMMA
// (fragments of the band from shared memory, C read-modify-write in L2).
__device__ bool chol_bands_global(double* W, int k, double* Wb, double* Rk, int ldr, double* inv, double& smin,
                                  FState& fs, int* flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const LayoutBand4 band;
  for (int r0 = 0; r0 < k; r0 += FK_PANEL) {
    const int n = k - r0;                 // order of the remaining matrix
    const int nb = (n + 7) >> 3;
    const int nbr = min(4, nb);
    for (int r = warp; r < 8 * nbr; r += FK_NW)
      for (int c = r + lane; c < 8 * nb; c += 32) {
        double x = (c == r) ? 1.0 : 0.0;   // identity padding past n
        if (c < n && r < n) x = W[(int64_t)(r0 + c) * k + r0 + r];
        Wb[band(r >> 3, c >> 3) + (c & 7) * 8 + (r & 7)] = x;
      }
    __syncthreads();
    if (!chol_banded(Wb, n, nb, nbr, r0, inv, smin, fs, LayoutBand4(), flag)) return false;
    for (int r = warp; r < min(FK_PANEL, n); r += FK_NW)
      for (int c = r + lane; c < n; c += 32)
        Rk[(int64_t)(r0 + c) * ldr + r0 + r] = Wb[band(r >> 3, c >> 3) + (c & 7) * 8 + (r & 7)];
    if (nb > 4) {
      // trailing blocks (I, J), 4 <= I <= J < nb (band-relative), two per iteration
      const int tn = nb - 4;
      const int nblk = tn * (tn + 1) / 2;
      auto decode = [&](int blk, int& I, int& J) {
        J = tri_col(blk);
        I = 4 + blk - J * (J + 1) / 2;
        J += 4;
      };
      for (int blk = warp; blk < nblk; blk += 2 * FK_NW) {
        const int blk2 = blk + FK_NW;
        const bool two = blk2 < nblk;
        int I0, J0, I1 = 4, J1 = 4;
        decode(blk, I0, J0);
        if (two) decode(blk2, I1, J1);
        // C fragment (row g, cols 2t, 2t+1) of block (I, J): W(r0 + 8I + g, r0 + 8J + 2t + e)
        const int ri0 = 8 * I0 + g, ri1 = 8 * I1 + g;
        double c0[2], c1[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cj0 = 8 * J0 + 2 * t + e, cj1 = 8 * J1 + 2 * t + e;
          c0[e] = (ri0 < n && cj0 < n) ? W[(int64_t)(r0 + cj0) * k + r0 + ri0] : 0.0;
          c1[e] = (two && ri1 < n && cj1 < n) ? W[(int64_t)(r0 + cj1) * k + r0 + ri1] : 0.0;
        }
#pragma unroll
        for (int P = 0; P < 4; ++P) {
          const double* pa0 = Wb + band(P, I0) + g * 8 + t;
          const double* pb0 = Wb + band(P, J0) + g * 8 + t;
          const double* pa1 = Wb + band(P, I1) + g * 8 + t;
          const double* pb1 = Wb + band(P, J1) + g * 8 + t;
          double a00, a01, b00, b01, a10, a11, b10, b11;
          frag_pair(pa0, g, a00, a01);
          frag_pair(pb0, g, b00, b01);
          frag_pair(pa1, g, a10, a11);
          frag_pair(pb1, g, b10, b11);
          a00 = -a00; a01 = -a01; a10 = -a10; a11 = -a11;
          dmma(c0, a00, b00);
          dmma(c1, a10, b10);
          dmma(c0, a01, b01);
          dmma(c1, a11, b11);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cj0 = 8 * J0 + 2 * t + e, cj1 = 8 * J1 + 2 * t + e;
          if (ri0 < n && cj0 < n && ri0 <= cj0) W[(int64_t)(r0 + cj0) * k + r0 + ri0] = c0[e];
          if (two && ri1 < n && cj1 < n && ri1 <= cj1) W[(int64_t)(r0 + cj1) * k + r0 + ri1] = c1[e];
        }
      }
    }
    __syncthreads();   // W updates (global, this CTA) and the band area before the next band
  }
  return true;
}


__device__ __forceinline__ void fmark(int slot) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fprof[slot] = t;
  }
}

// ---------------------------------------------------------------------------
// Band-cluster Cholesky (96 < k <= 256, see factor_launch).  One attempt runs
// on a thread-block cluster of C = ceil(k / 32) CTAs; CTA r owns band r --
// rows [32r, 32r + 32) x columns [32r, k) of the upper triangle -- in its
// shared memory:
//   1. load its band of X + sigma I (every load of the band in flight at once);
//   2. for b = 0 .. r-1: apply the rows of band b, block row by block row, as
//      rank-8 DMMA updates of its band (per element: b, then P ascending, k4 0
//      then 4 -- the chain of the single-CTA banded path).  The rows are read
//      straight from band b's shared memory (DSMEM, ld.shared::cluster) once
//      band b has counted them into this CTA's row counter for b (a cluster-
//      scope release store): the next band takes every block row as it
//      finishes, the later bands take a band once it is complete;
//   3. factor its band with the in-band blocked steps (chol_banded); the hook
//      counts each finished block row into the later bands' counters, from a
//      worker thread (warp 0 runs the pivot chain).  A breakdown or an abort
//      is counted too (+15), so later bands stop instead of waiting;
//   4. write its rows of R to Rk;
//   5. agree on the outcome: every CTA stores its record into every CTA's
//      shared memory (DSMEM), one cluster barrier, the lowest band that did
//      not hold decides (its pivot is the reference's first breakdown).
// The single-CTA path runs the Schur complement of band 0 and seven rank-32
// band updates (~60 us of DMMA at k = 256) on one SM between the bands; here
// they run on C SMs while the bands factor, and the serial part is the last
// block row's hand-over plus the in-band steps.  Counters carry the attempt
// number (seq * 16 + rows), so a retry never reads an earlier attempt's count.
// A cluster guarantees the C CTAs are co-resident, so waiting on a lower
// band always terminates (a band never waits on a higher one).
constexpr int FC_LD = 36;   // staged band: column stride (conflict-free DMMA fragment loads)
constexpr int FC_LD8 = 12;  // one staged block row (8 rows): column stride, conflict-free fragment loads

// chol_blocked hook of the band-cluster path: block row P of this band is
// final -> count it in every later band's row counter for this band
struct BandRowHook {
  unsigned* crows;
  int r, C;
  unsigned seq;
  __device__ __forceinline__ void operator()(int P) const {
    // the next band takes every block row as it finishes; the later bands read
    // the band only once it is complete (their DSMEM reads would otherwise
    // compete with this band's own shared-memory traffic)
    if (threadIdx.x == FK_THREADS - 32) {   // a worker warp: warp 0 runs the pivot chain
      const unsigned v = seq * 16u + (unsigned)(P + 1);
      if (r + 1 < C) dsmem_st_release(crows + r, r + 1, v);
      if (P == 3)
        for (int d = r + 2; d < C; ++d) dsmem_st_release(crows + r, d, v);
    }
  }
};
enum { BAND_OK = 1, BAND_BREAKDOWN = 2, BAND_ABORT = 3, BAND_UPSTREAM = 4 };

__host__ __device__ inline int64_t cluster_work_doubles(int k) {
  const int nb = (k + 7) / 8;
  return (int64_t)256 * nb + (int64_t)FC_LD * 8 * nb;   // band (4 x nb blocks) + staged rows
}

__device__ bool chol_attempt_band_cluster(const double* __restrict__ Xg, int k, double sigma, double* smem_w,
                                          double* Rk, int ldr, double* inv, double& smin, FState& fs, int* flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r = fs.crank, C = fs.csize;
  const int r0 = 32 * r;
  const int n = k - r0;                  // order of the trailing matrix from this band on
  const int nb = (n + 7) >> 3;
  const int nbr = min(4, nb);
  const int nrow = min(32, n);
  double* Wb = smem_w;                   // the band, LayoutBand4
  double* stg = smem_w + 256 * nb;       // one block row of an earlier band: stg[c * FC_LD8 + ii]
  const LayoutBand4 band;
  __shared__ int s_state;
  const unsigned seq = fs.seq + 1;       // uniform over the cluster (every CTA runs every attempt)
  cmark(fs, 0);

  // ---- 1. the band of X + sigma I (X symmetric: X(r0 + i, r0 + c) = Xg[(r0 + i) k + r0 + c])
  {
    constexpr int NL = (32 * 256 + FK_THREADS - 1) / FK_THREADS;
    double v[NL];
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int e = tid + FK_THREADS * u, i = e >> 8, c = e & 255;
      v[u] = (i < 32 && i <= c && c < n && i < n) ? __ldg(Xg + (int64_t)(r0 + i) * k + r0 + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NL; ++u) {
      const int e = tid + FK_THREADS * u, i = e >> 8, c = e & 255;
      if (i < 8 * nbr && i <= c && c < 8 * nb)
        Wb[band(i >> 3, c >> 3) + (c & 7) * 8 + (i & 7)] = (c == i) ? (i < n ? __dadd_rn(v[u], sigma) : 1.0) : v[u];
    }
  }
  __syncthreads();
  cmark(fs, 1);

  // ---- 2. the updates of the earlier bands, block row by block row as they
  // are published: rows 8P .. 8P + 7 of band b are read straight from band b's
  // shared memory (DSMEM) and applied as a rank-8 update, while band b goes on
  // with its next pivots; only its last block row's hand-over is serial
  int state = BAND_OK;
  for (int b = 0; b < r && state == BAND_OK; ++b) {
    const int offc = r0 - 32 * b;                      // this band's column 0 among band b's columns
    const uint32_t rbase = dsmem_addr(smem_w, b);      // band b's work area (same offset in every CTA)
    for (int P = 0; P < 4; ++P) {
      if (tid == 0) {
        const unsigned want = seq * 16u + (unsigned)(b == r - 1 ? P + 1 : 4);
        while (true) {
          const unsigned v = ld_acquire_cluster(fs.crows + b);
          if ((v >> 4) != seq) continue;              // an earlier attempt's count
          if ((v & 15u) == 15u) { s_state = BAND_UPSTREAM; break; }
          if (v >= want) { s_state = BAND_OK; break; }
        }
      }
      __syncthreads();
      if (s_state != BAND_OK) { state = BAND_UPSTREAM; break; }
      if (b == r - 1 && P == 3) cmark(fs, 2);
      {
        // stg[c * FC_LD8 + ii] = R(32b + 8P + ii, r0 + c): lanes over 4 columns x 8 rows (64 contiguous doubles)
        constexpr int NE = (64 * 32 + FK_THREADS - 1) / FK_THREADS;
        double v[NE];
#pragma unroll
        for (int u = 0; u < NE; ++u) {
          const int e = tid + FK_THREADS * u, c = e >> 3, ii = e & 7, cp = offc + c;
          v[u] = (c < n) ? dsmem_ld(rbase + 8u * (uint32_t)(band(P, cp >> 3) + (cp & 7) * 8 + ii)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NE; ++u) {
          const int e = tid + FK_THREADS * u, c = e >> 3, ii = e & 7;
          if (c < 8 * nb) stg[c * FC_LD8 + ii] = v[u];
        }
      }
      __syncthreads();
      // C(I, J) -= A(P, I)^T B(P, J) over the band's blocks I <= J: a warp
      // takes a 2 x 2 group (four accumulator chains, each fragment feeds two DMMAs)
      const int G = (nb + 1) >> 1;
      const int ngr = G + (nbr > 2 ? G - 1 : 0);
      for (int gidx = warp; gidx < ngr; gidx += FK_NW) {
        const int gi = gidx < G ? 0 : 1;
        const int gj = gidx < G ? gidx : gidx - G + 1;
        const int I[2] = {2 * gi, 2 * gi + 1}, J[2] = {2 * gj, 2 * gj + 1};
        bool live[2][2];
        double c[2][2][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            live[x][y] = I[x] < nbr && I[x] <= J[y] && J[y] < nb;
            const double* pc = Wb + band(live[x][y] ? I[x] : 0, live[x][y] ? J[y] : 0) + 2 * t * 8 + g;
            cfrag_load(pc, t, c[x][y]);
            if (!live[x][y]) { c[x][y][0] = 0.0; c[x][y][1] = 0.0; }
          }
        const int ci[2] = {min(I[0], nb - 1), min(I[1], nb - 1)};
        const int cj[2] = {min(J[0], nb - 1), min(J[1], nb - 1)};
        double a[2][2], bb[2][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            a[x][h] = -stg[(8 * ci[x] + g) * FC_LD8 + 4 * h + t];
            bb[x][h] = stg[(8 * cj[x] + g) * FC_LD8 + 4 * h + t];
          }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) dmma(c[x][y], a[x][h], bb[y][h]);
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
            if (live[x][y]) cfrag_store(Wb + band(I[x], J[y]) + 2 * t * 8 + g, t, c[x][y]);
      }
      __syncthreads();
    }
  }

  // ---- 3. the band's own 32 pivots; each finished block row is published to
  // the later bands (their row counters, DSMEM release stores) by a worker
  // thread, so warp 0's pivot chain never waits on it
  cmark(fs, 3);
  if (state == BAND_OK) {
    if (!chol_banded(Wb, n, nb, nbr, r0, inv, smin, fs, band, flag, BandRowHook{fs.crows, r, C, seq}))
      state = fs.aborted ? BAND_ABORT : BAND_BREAKDOWN;
  }
  if (state != BAND_OK && threadIdx.x == FK_THREADS - 32)
    for (int d = r + 1; d < C; ++d) dsmem_st_release(fs.crows + r, d, seq * 16u + 15u);

  // ---- 4. rows r0 .. r0 + nrow - 1 of R (the later bands read them from shared memory)
  cmark(fs, 4);
  if (state == BAND_OK) {
    for (int c = warp; c < n; c += FK_NW)
      if (lane < nrow && lane <= c)
        Rk[(int64_t)(r0 + c) * ldr + r0 + lane] = Wb[band(lane >> 3, c >> 3) + (c & 7) * 8 + (lane & 7)];
  }
  cmark(fs, 5);

  // ---- 5. the attempt's outcome, agreed over the cluster
  const int slot = (int)(seq & 1u) * 32;
  if (tid == 0) {
    for (int d = 0; d < C; ++d) {
      dsmem_st(fs.crec + slot + 4 * r + 0, d, (double)state);
      dsmem_st(fs.crec + slot + 4 * r + 1, d, (double)fs.pivot_index);
      dsmem_st(fs.crec + slot + 4 * r + 2, d, fs.pivot_value);
      dsmem_st(fs.crec + slot + 4 * r + 3, d, smin);
    }
  }
  cluster_sync_all();
  if (tid == 0) {
    int res = BAND_OK;
    double sm = INFINITY;
    for (int b = 0; b < C; ++b) {
      const double* rec = fs.crec + slot + 4 * b;
      const int sb = (int)rec[0];
      if (sb == BAND_OK) { sm = fmin(sm, rec[3]); continue; }
      res = sb;
      if (sb == BAND_BREAKDOWN) { fs.pivot_index = (int)rec[1]; fs.pivot_value = rec[2]; }
      break;
    }
    fs.aborted = (res == BAND_ABORT) ? 1 : 0;
    fs.seq = seq;
    smin = sm;
    s_state = res;
  }
  __syncthreads();
  cmark(fs, 6);
  return s_state == BAND_OK;
}

// One factorization attempt of X + sigma I; on success the factor is in Rk
// (upper triangle; the caller zeroes the rest).  `smem_w` is the shared work
// area, `gW` the global fallback for k > FK_BIG_K.  X is symmetric: Xs in shared
// memory for k <= 128, else Xg in global memory, read-only for the kernel and
// read through ld.global.nc (generic loads from one SM run ~4x slower,
// profiles/r01_single_sm_io.jsonl).
__device__ __noinline__ bool chol_attempt(const double* __restrict__ Xs, const double* __restrict__ Xg, int k,
                             double sigma, double* smem_w, double* gW,
                             double* Rk, int ldr, double* rowbuf, FState& fs, int* flag) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double smin = INFINITY;
  bool ok;
  if (fs.csize > 1) {
    ok = chol_attempt_band_cluster(Xg, k, sigma, smem_w, Rk, ldr, rowbuf, smin, fs, flag);
  } else if (k <= FK_SMEM_K) {
    double* Wb = smem_w;
    for (int c = warp; c < k; c += FK_NW)
      for (int i = lane; i <= c; i += 32) {
        double x = Xs[c * k + i];
        if (i == c) x = __dadd_rn(x, sigma);
        Wb[belem(i, c)] = x;
      }
    pad_blocked(Wb, k);
    __syncthreads();
    fmark(2);
    const int nb = (k + 7) >> 3;
    ok = g_banded ? chol_banded(Wb, k, nb, nb, 0, rowbuf, smin, fs, LayoutUpper(), flag)
                  : chol_blocked(Wb, k, nb, 0, nb, 0, rowbuf, smin, fs, LayoutUpper(), flag);
    fmark(3);
    if (ok) store_blocked(Wb, k, 0, Rk, ldr);
    fmark(4);
  } else if (k > FK_BIG_K && k <= FK_BAND_K) {
    double* W = gW;   // k x k upper (column-major): X + sigma I, factored in place by bands
    for (int c = warp; c < k; c += FK_NW)
      for (int i = lane; i <= c; i += 32) {
        double x = __ldg(Xg + (int64_t)c * k + i);
        if (i == c) x = __dadd_rn(x, sigma);
        W[(int64_t)c * k + i] = x;
      }
    __syncthreads();
    ok = chol_bands_global(W, k, smem_w, Rk, ldr, rowbuf, smin, fs, flag);
  } else if (k > FK_BIG_K) {
    double* W = gW;
    for (int c = warp; c < k; c += FK_NW)
      for (int i = lane; i <= c; i += 32) {
        double x = __ldg(Xg + (int64_t)c * k + i);
        if (i == c) x = __dadd_rn(x, sigma);
        W[pk(i, c)] = x;
      }
    __syncthreads();
    ok = chol_packed(W, k, 0, rowbuf, smin, fs);
    if (ok) store_packed(W, k, 0, Rk, ldr);
  } else {
    // ---- stage 1: block rows 0..3 (rows 0..31) as a band, updates kept inside the band
    fmark(2);
    const int b = FK_PANEL;
    const int nb = (k + 7) >> 3;
    double* Wb = smem_w;
    const LayoutBand4 band;
    // (8 nb <= 256 columns: one batch of 8 loads per lane and row, all in
    // flight before the stores)
    for (int r = warp; r < b; r += FK_NW) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = r + lane + 32 * u;
        v[u] = (c < 8 * nb && c < k) ? __ldg(Xg + (int64_t)r * k + c) : 0.0;   // = X(r, c) by symmetry
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = r + lane + 32 * u;
        if (c < 8 * nb) Wb[band(r >> 3, c >> 3) + (c & 7) * 8 + (r & 7)] = (c == r) ? __dadd_rn(v[u], sigma) : v[u];
      }
    }
    __syncthreads();
    ok = chol_banded(Wb, k, nb, 4, 0, rowbuf, smin, fs, LayoutBand4(), flag);
    if (ok) {
      // band rows are final rows of R
      // (a warp per column, lanes over the 32 band rows: coalesced)
      for (int c = warp; c < k; c += FK_NW)
        if (lane <= c) Rk[(int64_t)c * ldr + lane] = Wb[band(lane >> 3, c >> 3) + (c & 7) * 8 + (lane & 7)];
      __syncthreads();
      fmark(3);
      if (spec_should_stop(fs)) return false;
      // ---- stage 2: S = X22 + sigma I - R12^T R12 (block upper, n = k - 32) with DMMA.
      // A warp takes 2 x 2 groups of S blocks (four accumulator chains; each
      // R12 fragment, read from the band in shared memory, feeds two DMMAs) and
      // loads its X22 values as C fragments straight from L2 at the start of
      // the group, so their latency hides under the DMMA chains.  S's block
      // layout overlays the band for its first block columns: the groups that
      // touch them (group columns <= GJO) are kept in registers and stored
      // after a barrier; the others are stored at once.
      const int n = k - b;
      double* S = smem_w;
      const int nbs = (n + 7) / 8;
      const int nblk = nbs * (nbs + 1) / 2;
      const int nov = min(nblk, 4 * nb);          // S blocks inside the band area
      const int g = lane >> 2, t = lane & 3;
      const int G = (nbs + 1) >> 1;               // group rows / columns
      const int ngroups = G * (G + 1) / 2;
      int GJO = -1;                               // last group column that can touch the overlay
      while (GJO + 1 < G && (2 * (GJO + 1)) * (2 * (GJO + 1) + 1) / 2 < nov) ++GJO;
      const int nog = (GJO + 1) * (GJO + 2) / 2;  // groups gidx < nog are kept
      // one group: v[x][y][e] = S values of blocks (2gi + x, 2gj + y), fragment (row g, col 2t + e)
      auto sgroup = [&](int gidx, double (&v)[2][2][2]) {
        const int gj = tri_col(gidx), gi = gidx - gj * (gj + 1) / 2;
        double acc[2][2][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * (2 * gi + x) + g, c = 8 * (2 * gj + y) + 2 * t + e;   // trailing coordinates
              v[x][y][e] = (i <= c && c < n) ? __ldg(Xg + (int64_t)(b + c) * k + b + i) : 0.0;
              acc[x][y][e] = 0.0;
            }
        const int I0 = min(2 * gi, nbs - 1), I1 = min(2 * gi + 1, nbs - 1);
        const int J0 = min(2 * gj, nbs - 1), J1 = min(2 * gj + 1, nbs - 1);
        const int Ic[2] = {I0, I1}, Jc[2] = {J0, J1};
#pragma unroll
        for (int P = 0; P < FK_PANEL / 8; ++P) {   // band block row P: k-steps rows t, 4 + t
          double fa[2][2], fb[2][2];
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            frag_pair(Wb + band(P, b / 8 + Ic[x]) + g * 8 + t, g, fa[x][0], fa[x][1]);
            frag_pair(Wb + band(P, b / 8 + Jc[x]) + g * 8 + t, g, fb[x][0], fb[x][1]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
              for (int y = 0; y < 2; ++y) dmma(acc[x][y], fa[x][h], fb[y][h]);
        }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * (2 * gi + x) + g, c = 8 * (2 * gj + y) + 2 * t + e;
              double xv = v[x][y][e];
              if (i == c) xv = __dadd_rn(xv, sigma);
              v[x][y][e] = xv - acc[x][y][e];
            }
      };
      auto gstore = [&](int gidx, const double (&v)[2][2][2]) {
        const int gj = tri_col(gidx), gi = gidx - gj * (gj + 1) / 2;
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * (2 * gi + x) + g, c = 8 * (2 * gj + y) + 2 * t + e;
              if (i <= c && c < n) S[belem(i, c)] = v[x][y][e];
            }
      };
      // kept groups per warp, bounded at the largest overlay (nov <= 4 (FK_BIG_K / 8))
      constexpr int NOV_MAX = 4 * (FK_BIG_K / 8);
      constexpr int GJO_MAX = [] { int j = -1; while ((2 * (j + 1)) * (2 * (j + 1) + 1) / 2 < NOV_MAX) ++j; return j; }();
      constexpr int KG = ((GJO_MAX + 1) * (GJO_MAX + 2) / 2 + FK_NW - 1) / FK_NW;
      double keep[KG][2][2][2];
#pragma unroll
      for (int j = 0; j < KG; ++j) {
        const int gidx = warp + FK_NW * j;
        if (gidx < nog) sgroup(gidx, keep[j]);
      }
      for (int gidx = nog + warp; gidx < ngroups; gidx += FK_NW) {
        double v[2][2][2];
        sgroup(gidx, v);
        gstore(gidx, v);
      }
      __syncthreads();   // every read of the band is done
#pragma unroll
      for (int j = 0; j < KG; ++j) {
        const int gidx = warp + FK_NW * j;
        if (gidx < nog) gstore(gidx, keep[j]);
      }
      pad_blocked(S, n);
      __syncthreads();
      fmark(4);
      ok = g_banded ? chol_banded(S, n, nbs, nbs, b, rowbuf, smin, fs, LayoutUpper(), flag)
                    : chol_blocked(S, n, nbs, 0, nbs, b, rowbuf, smin, fs, LayoutUpper(), flag);
      fmark(5);
      if (ok) store_blocked(S, n, b, Rk, ldr);
    }
  }
  if (tid == 0) {
    const double margin = (ok ? smin : fs.pivot_value) / fs.diag_max;
    if (fs.attempts == 0) fs.plain_margin = margin;
    fs.attempts += 1;
    if (ok) fs.min_pivot = smin;
  }
  __syncthreads();
  return ok;
}

// One X v product row block for the power iteration: rows [i0, i0 + nr) of X
// (row i at Xr + (i - i0) k), lanes striding the row, butterfly sums -- the
// same per-row operation order wherever the rows come from.
template <int MR>
__device__ __forceinline__ void matvec_rows(const double* Xr, int i0, int nr, int k, const double* vec, double* wv,
                                            bool global) {
  const int lane = threadIdx.x & 31;
  double acc[MR];
#pragma unroll
  for (int r = 0; r < MR; ++r) acc[r] = 0.0;
  for (int c = lane; c < k; c += 32) {
    const double vc = vec[c];
#pragma unroll
    for (int r = 0; r < MR; ++r)
      if (r < nr) acc[r] += (global ? __ldg(Xr + (int64_t)r * k + c) : Xr[(int64_t)r * k + c]) * vc;
  }
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    const double sr = warp_sum(acc[r]);
    if (lane == 0 && r < nr) wv[i0 + r] = sr;
  }
}

// Power iteration of spectral_norm_estimate (kernels.py:126-178) for X in
// shared memory (k <= 128) on warp 0 alone: lane l owns rows l, l + 32, ...
// (NR = ceil(k/32) rows), reads column j of the symmetric X (consecutive lanes,
// consecutive addresses) against the broadcast v[j], and the two dot products
// of an iteration are warp sums -- no block barrier inside the loop.  The
// block-wide version spent ~4000 cycles per iteration at k = 64 on four
// 384-thread barriers and per-row warp reductions; this one ~600.  The caller
// has set vec = 1/sqrt(k).  Returns the estimate (or `fro` with est_flag set).
template <int NR>
__device__ double power_iter_warp(const double* __restrict__ X, int k, double tol, int max_iter, double* vec,
                                  FState& fs, double fro) {
  const int lane = threadIdx.x & 31;
  double vr[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) vr[r] = (lane + 32 * r < k) ? vec[lane + 32 * r] : 0.0;
  bool have_prev = false;
  double prev = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    double acc[NR][2];
#pragma unroll
    for (int r = 0; r < NR; ++r) { acc[r][0] = 0.0; acc[r][1] = 0.0; }
    int j = 0;
    for (; j + 1 < k; j += 2) {   // two accumulator chains per row (even / odd columns)
      const double v0 = vec[j], v1 = vec[j + 1];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int i = lane + 32 * r;
        if (i < k) {
          acc[r][0] += X[(int64_t)j * k + i] * v0;
          acc[r][1] += X[(int64_t)(j + 1) * k + i] * v1;
        }
      }
    }
    if (j < k) {
      const double v0 = vec[j];
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (lane + 32 * r < k) acc[r][0] += X[(int64_t)j * k + lane + 32 * r] * v0;
    }
    double ww = 0.0, vw = 0.0, w[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      w[r] = acc[r][0] + acc[r][1];
      ww += w[r] * w[r];
      vw += vr[r] * w[r];
    }
    const double nw = sqrt(warp_sum(ww));
    const double lam = warp_sum(vw);
    if (nw == 0.0) {
      if (lane == 0) fs.est_flag = 1;
      return fro;
    }
    __syncwarp();   // every lane has read vec for this product
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      vr[r] = w[r] / nw;
      if (lane + 32 * r < k) vec[lane + 32 * r] = vr[r];
    }
    __syncwarp();
    if (have_prev && fabs(lam - prev) <= tol * fabs(lam)) {
      if (lane == 0) g_fprof[8] = it + 1;   // iterations of the last estimate (profiling)
      return fabs(lam);
    }
    prev = lam;
    have_prev = true;
  }
  if (lane == 0) { fs.est_flag = 2; g_fprof[8] = max_iter; }
  return fro;
}

// spectral_norm_estimate (kernels.py:126-178) on the full symmetric X.
// Returns the estimate; sets fs.est_flag (1 stalled, 2 not converged) and
// fs.code = CQR_ASYMMETRIC on the asymmetry ValueError.
// GX (k > 128, X in global memory): X was formed symmetric by construction
// (factor_prep_kernel mirrors the lower triangle), so the reference's asymmetry
// check cannot fire and ||X||_F comes from the prep kernel's partials (fs.fro);
// each X v streams X through the shared work area `ring` with cp.async.bulk,
// two row chunks in flight per warp (one SM pulls ~80 B/clk that way against
// ~30 B/clk with loads, profiles/r01_single_sm_io.jsonl).
template <bool GX>
__device__ double norm_estimate(const double* __restrict__ X, int k, double tol, int max_iter, double* vec,
                                double* wv, double* red, FState& fs, double* ring, int ring_doubles) {
  const int tid = threadIdx.x;
  double fro;
  if (!GX) {
    double loc = 0.0, la = 0.0;
    for (int c = tid >> 5; c < k; c += FK_NW)
#pragma unroll 4
      for (int i = tid & 31; i < k; i += 32) {
        const double x = X[(int64_t)c * k + i];
        loc += x * x;
        const double d = x - X[(int64_t)i * k + c];
        la += d * d;
      }
    fro = sqrt(block_sum(loc, red));
    const double asym = sqrt(block_sum(la, red));
    if (fro == 0.0) return 0.0;
    if (asym > 1e-8 * fro) {
      if (tid == 0) fs.code = CQR_ASYMMETRIC;
      return fro;
    }
  } else {
    fro = fs.fro;
    if (fro == 0.0) return 0.0;
  }
  const double v0 = 1.0 / sqrt((double)k);
  for (int i = tid; i < k; i += FK_THREADS) vec[i] = v0;
  const int warp = tid >> 5, lane = tid & 31;
  // ring: 2 stages per warp of R rows (k even: rows are whole 16-byte units)
  constexpr int RMAX = 8;
  const int R = GX && (k % 2 == 0) ? min(RMAX, ring_doubles / (2 * FK_NW * k)) : 0;
  __shared__ __align__(8) uint64_t rbar[2 * FK_NW];
  if (R > 0 && tid == 0) {
    for (int j = 0; j < 2 * FK_NW; ++j) mbar_init(&rbar[j], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (!GX) {
    // X in shared memory: the whole iteration on warp 0, the result broadcast through red
    if (warp == 0) {
      double res;
      switch ((k + 31) >> 5) {
        case 1: res = power_iter_warp<1>(X, k, tol, max_iter, vec, fs, fro); break;
        case 2: res = power_iter_warp<2>(X, k, tol, max_iter, vec, fs, fro); break;
        case 3: res = power_iter_warp<3>(X, k, tol, max_iter, vec, fs, fro); break;
        default: res = power_iter_warp<4>(X, k, tol, max_iter, vec, fs, fro); break;
      }
      if (lane == 0) red[0] = res;
    }
    __syncthreads();
    const double res = red[0];
    __syncthreads();   // red is reused by the caller's reductions
    return res;
  }
  const int nch = R > 0 ? (k + R - 1) / R : 0;   // row chunks per product
  uint32_t uses[2] = {0u, 0u};                    // this warp's stage uses (phase parity)
  auto issue = [&](int ch, int st) {              // lane 0: chunk ch into this warp's stage st
    const int r0 = ch * R, nr = min(R, k - r0);
    double* dst = ring + (int64_t)(2 * warp + st) * R * k;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&rbar[2 * warp + st], (uint32_t)(nr * k * 8));
    bulk_g2s(dst, X + (int64_t)r0 * k, (uint32_t)(nr * k * 8), &rbar[2 * warp + st]);
  };
  bool have_prev = false;
  double prev = 0.0;
  double result = fro;
  bool finished = false;
  for (int it = 0; it < max_iter && !finished; ++it) {
    if (R > 0) {
      // w = X v, chunk ch = warp + FK_NW q of the rows, stage q & 1 of this warp
      if (lane == 0) {
        if (warp < nch) issue(warp, 0);
        if (warp + FK_NW < nch) issue(warp + FK_NW, 1);
      }
      __syncthreads();   // vec is ready
      for (int q = 0; warp + FK_NW * q < nch; ++q) {
        const int ch = warp + FK_NW * q, st = q & 1;
        mbar_wait(&rbar[2 * warp + st], uses[st] & 1u);
        ++uses[st];
        const int r0 = ch * R, nr = min(R, k - r0);
        matvec_rows<RMAX>(ring + (int64_t)(2 * warp + st) * R * k, r0, nr, k, vec, wv, false);
        __syncwarp();
        if (lane == 0 && ch + 2 * FK_NW < nch) issue(ch + 2 * FK_NW, st);
      }
    } else {
      __syncthreads();
      // warp w owns rows w, w + FK_NW, ... (4 rows in flight)
      for (int i0 = warp * 4; i0 < k; i0 += 4 * FK_NW)
        matvec_rows<4>(X + (int64_t)i0 * k, i0, min(4, k - i0), k, vec, wv, GX);
    }
    __syncthreads();
    // ||w||^2 and v.w in one two-value reduction
    double ww = 0.0, vw = 0.0;
    for (int i = tid; i < k; i += FK_THREADS) {
      ww += wv[i] * wv[i];
      vw += vec[i] * wv[i];
    }
    ww = warp_sum(ww);
    vw = warp_sum(vw);
    if (lane == 0) { red[warp] = ww; red[FK_NW + warp] = vw; }
    __syncthreads();
    double nw2 = 0.0, lam = 0.0;
#pragma unroll
    for (int w = 0; w < FK_NW; ++w) { nw2 += red[w]; lam += red[FK_NW + w]; }
    const double nw = sqrt(nw2);
    if (nw == 0.0) {
      if (tid == 0) fs.est_flag = 1;
      result = fro;
      finished = true;
      break;
    }
    for (int i = tid; i < k; i += FK_THREADS) vec[i] = wv[i] / nw;
    __syncthreads();   // also: red is rewritten next iteration only after this
    if (have_prev && fabs(lam - prev) <= tol * fabs(lam)) {
      if (tid == 0) g_fprof[8] = it + 1;   // iterations of the last estimate (profiling; one CTA runs it)
      result = fabs(lam);
      finished = true;
      break;
    }
    prev = lam;
    have_prev = true;
  }
  if (!finished) {
    if (tid == 0) { fs.est_flag = 2; g_fprof[8] = max_iter; }
    result = fro;
  }
  __syncthreads();   // every stage consumed: the barriers can go
  if (R > 0 && tid == 0)
    for (int j = 0; j < 2 * FK_NW; ++j) asm volatile("mbarrier.inval.shared.b64 [%0];" ::"r"(smem_u32(&rbar[j])) : "memory");
  __syncthreads();
  return result;
}

// Band-cluster groups: the same power iteration with the rows of X spread over
// the cluster.  CTA r keeps rows [32r, 32r + 32) of X in shared memory (loaded
// once), forms its part of w = X v with matvec_rows (the per-row operation
// order of the single-CTA version), stores it into every CTA's copy of w
// (DSMEM; two buffers alternating by iteration, so one cluster barrier per
// iteration suffices), and every CTA then runs the single-CTA version's
// reductions on the whole w: each CTA computes the same bits, and the same
// bits as norm_estimate<true>.  Per iteration this is one 64 KB local matvec
// instead of streaming all of X (512 KB at k = 256) through one SM.
__device__ double norm_estimate_cluster(const double* __restrict__ X, int k, double tol, int max_iter, double* vec,
                                        double* red, FState& fs, double* work) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = fs.crank, C = fs.csize;
  const int r0 = 32 * r, nr = min(32, k - r0);
  const double fro = fs.fro;
  if (fro == 0.0) return 0.0;
  const int kp = (int)round_up(k, 8);
  double* Xr = work;                       // nr x k, row-major (row i = column r0 + i of the symmetric X)
  double* wb = work + 32 * kp;             // two w buffers of kp
  for (int e0 = tid; e0 < nr * k; e0 += 8 * FK_THREADS) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * FK_THREADS;
      v[u] = (e < nr * k) ? __ldg(X + (int64_t)r0 * k + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * FK_THREADS;
      if (e < nr * k) Xr[(e / k) * k + e % k] = v[u];
    }
  }
  const double v0 = 1.0 / sqrt((double)k);
  for (int i = tid; i < k; i += FK_THREADS) vec[i] = v0;
  __syncthreads();
  bool have_prev = false;
  double prev = 0.0, result = fro;
  bool finished = false;
  for (int it = 0; it < max_iter && !finished; ++it) {
    double* wv = wb + (it & 1) * kp;
    // this CTA's rows: warp w takes rows w, w + 12, w + 24 (one matvec_rows call each)
    for (int i = warp; i < nr; i += FK_NW) matvec_rows<1>(Xr + (int64_t)i * k, r0 + i, 1, k, vec, wv, false);
    __syncthreads();
    if (tid < 32 * C) {
      const int d = tid >> 5, i = tid & 31;
      if (i < nr) dsmem_st(wv + r0 + i, d, wv[r0 + i]);
    }
    cluster_sync_all();
    double ww = 0.0, vw = 0.0;
    for (int i = tid; i < k; i += FK_THREADS) {
      ww += wv[i] * wv[i];
      vw += vec[i] * wv[i];
    }
    ww = warp_sum(ww);
    vw = warp_sum(vw);
    if (lane == 0) { red[warp] = ww; red[FK_NW + warp] = vw; }
    __syncthreads();
    double nw2 = 0.0, lam = 0.0;
#pragma unroll
    for (int w = 0; w < FK_NW; ++w) { nw2 += red[w]; lam += red[FK_NW + w]; }
    const double nw = sqrt(nw2);
    if (nw == 0.0) {
      if (tid == 0) fs.est_flag = 1;
      result = fro;
      finished = true;
      break;
    }
    for (int i = tid; i < k; i += FK_THREADS) vec[i] = wv[i] / nw;
    __syncthreads();
    if (have_prev && fabs(lam - prev) <= tol * fabs(lam)) {
      if (tid == 0 && blockIdx.x == 0) g_fprof[8] = it + 1;
      result = fabs(lam);
      finished = true;
      break;
    }
    prev = lam;
    have_prev = true;
  }
  if (!finished) {
    if (tid == 0) { fs.est_flag = 2; if (blockIdx.x == 0) g_fprof[8] = max_iter; }
    result = fro;
  }
  // no CTA may leave (and reuse its w buffers or exit) while another can still store into them
  cluster_sync_all();
  return result;
}

// X in shared memory (k <= 128) or global memory; `ring` is the shared work area
__device__ __forceinline__ double norm_estimate_x(const double* Xs, const double* Xg, int k, double tol, int max_iter,
                                                  double* vec, double* wv, double* red, FState& fs, double* ring,
                                                  int ring_doubles) {
  if (fs.csize > 1) return norm_estimate_cluster(Xg, k, tol, max_iter, vec, red, fs, ring);
  return (k <= FK_SMEM_K) ? norm_estimate<false>(Xs, k, tol, max_iter, vec, wv, red, fs, ring, ring_doubles)
                          : norm_estimate<true>(Xg, k, tol, max_iter, vec, wv, red, fs, ring, ring_doubles);
}

// doubles of the factor kernel's shared work area (after X for k <= 128)
__host__ __device__ inline int64_t work_doubles(int k) {
  auto blocked = [](int n) { const int nb = (n + 7) / 8; return (int64_t)nb * (nb + 1) / 2 * 64; };
  if (k <= FK_SMEM_K) return blocked(k);
  if (k <= FK_BIG_K) return (int64_t)FK_PANEL * k > blocked(k - FK_PANEL) ? (int64_t)FK_PANEL * k : blocked(k - FK_PANEL);
  if (k <= FK_BAND_K) return (int64_t)FK_PANEL * round_up(k, 8);
  return 0;
}

// k > 128: X = G (or G - Bt^T Bt), symmetric from the lower triangle, formed in
// global memory by many CTAs ahead of the single-CTA factorization (one CTA
// per 32 x 32 tile of the lower triangle; the mirrored half goes through
// shared memory so both stores are coalesced).  Each tile also leaves its
// share of ||X - I||_F^2, the max diagonal of G and ||X||_F^2 in a.part.
constexpr int FP_THREADS = 256;

__global__ void __launch_bounds__(FP_THREADS) factor_prep_kernel(FactorArgs a) {
  if (a.gate != nullptr && *a.gate != CQR_FACTORED) return;
  __shared__ double tile[32][33];   // tile[col][row]
  __shared__ double red[FP_THREADS / 32][3];
  const int k = a.k;
  const int b = blockIdx.x;
  int ti = 0;
  while ((ti + 1) * (ti + 2) / 2 <= b) ++ti;
  const int tj = b - ti * (ti + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* X = a.X;
  const bool upd = (a.policy == CQR_POLICY_UPDATE && a.q > 0);
  double loc = 0.0, dml = -INFINITY, f2 = 0.0;
  const int r = 32 * ti + lane;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int cl = warp + 8 * s, c = 32 * tj + cl;
    double x = 0.0;
    if (r < k && c < k && r >= c) {
      const double gv = a.G[(int64_t)c * a.ldg + r];
      x = gv;
      if (upd) {
        const double* br = a.Bt + (int64_t)r * a.ldbt;
        const double* bc = a.Bt + (int64_t)c * a.ldbt;
        double d = 0.0;
        for (int l = 0; l < a.q; ++l) d += br[l] * bc[l];
        x = x - d;
      }
      X[(int64_t)c * k + r] = x;
      const double d = x - ((r == c) ? 1.0 : 0.0);
      loc += ((r == c) ? 1.0 : 2.0) * (d * d);
      f2 += ((r == c) ? 1.0 : 2.0) * (x * x);
      if (r == c) dml = fmax(dml, gv);
    }
    tile[cl][lane] = x;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int rl = warp + 8 * s, rr = 32 * ti + rl, c = 32 * tj + lane;
    if (rr < k && c < k && rr > c) X[(int64_t)rr * k + c] = tile[lane][rl];
  }
  // fixed-order reductions: lanes by xor tree, warps in index order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    loc += __shfl_xor_sync(0xffffffffu, loc, o);
    f2 += __shfl_xor_sync(0xffffffffu, f2, o);
    dml = fmax(dml, __shfl_xor_sync(0xffffffffu, dml, o));
  }
  if (lane == 0) { red[warp][0] = loc; red[warp][1] = dml; red[warp][2] = f2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e2 = 0.0, dm = -INFINITY, ff = 0.0;
#pragma unroll
    for (int w = 0; w < FP_THREADS / 32; ++w) { e2 += red[w][0]; dm = fmax(dm, red[w][1]); ff += red[w][2]; }
    a.part[3 * b] = e2;
    a.part[3 * b + 1] = dm;
    a.part[3 * b + 2] = ff;
  }
}

__global__ void __launch_bounds__(FK_THREADS, 1) factor_kernel(FactorArgs a) {
  if (a.gate != nullptr && *a.gate != CQR_FACTORED) {
    // gated off (the previous pass did not factor): record it, touch nothing else
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.st->code = CQR_SKIPPED;
      if (a.stm != nullptr) { a.stm->code = CQR_SKIPPED; __threadfence_system(); }
    }
    return;
  }
  extern __shared__ __align__(16) double fsm[];
  __shared__ FState fs;
  __shared__ int sflag;
  const int k = a.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kpad = (int)round_up(k, 8);
  double* red = fsm;
  double* rowbuf = fsm + 32;
  double* vec = rowbuf + kpad;
  double* wv = vec + kpad;
  // band-cluster path: a group of C CTAs (one cluster) per attempt chain
  const int C = a.ncl > 1 ? a.ncl : 1;
  // k <= 128 on one CTA: X itself lives in shared memory (k^2 doubles) before the work area
  const bool xs = (k <= FK_SMEM_K) && C == 1;
  double* Xs = wv + kpad;                // X in shared memory (xs)
  const double* Xg = a.X;                // X in global memory (formed by factor_prep_kernel)
  double* Wsm = xs ? Xs + (int64_t)k * k : wv + kpad;   // shared work area
  const int group = (int)blockIdx.x / C, crank = (int)blockIdx.x - group * C;
  const int wdoubles = C > 1 ? (int)cluster_work_doubles(k) : (int)work_doubles(k);
  __shared__ double crec[2 * 8 * 4];
  __shared__ unsigned crows[8];
  // speculative group 1 (RECOMPUTE): private R, work matrix and shift list; X
  // in global memory (k > 128) is formed identically by both groups
  const bool spec1 = a.spec && group == 1;
  double* Rkx = spec1 ? a.Rk1 : a.Rk;
  const int ldrx = spec1 ? a.ldr1 : a.ldr;
  double* gWx = spec1 ? a.W1 : a.W;
  double* shx = spec1 ? a.shifts1 : a.shifts;

  if (tid == 0) {
    fs.code = CQR_FACTORED; fs.retries = 0; fs.n_shifts = 0; fs.pivot_index = -1; fs.est_calls = 0;
    fs.est_flag = 0; fs.escalations = 0; fs.singular_index = -1;
    fs.pivot_value = 0.0; fs.err = 0.0; fs.norm_est = 0.0; fs.last_shift = 0.0; fs.min_pivot_rel = 0.0;
    fs.sigma = 0.0; fs.attempts = 0; fs.plain_margin = 0.0; fs.diag_max = 0.0; fs.min_pivot = 0.0; fs.fro = 0.0;
    fs.spec_flag = nullptr; fs.spec_done = 0; fs.aborted = 0;
    if (spec1) {
      fs.spec_flag = reinterpret_cast<const volatile unsigned long long*>(a.pub);
      fs.spec_done = (0xC9F0A5ull << 40) | ((unsigned long long)a.epoch << 2) | 1ull;
    }
    fs.crank = crank; fs.csize = C; fs.seq = 0;
    fs.crec = crec;
    fs.crows = crows;
  }
  if (tid < 8) crows[tid] = 0u;
  // every CTA's row counters are zero before any band can publish into them
  if (C > 1) cluster_sync_all();

  if (tid == 0 && blockIdx.x == 0) { g_fprof[9] = 0; g_fprof[10] = 0; g_fprof[11] = 0; g_fprof[12] = 0; }
  fmark(0);
  // ---- 1. X = G (or G - Bt^T Bt), symmetric by construction from the lower triangle
  //         (lower triangle read column by column: coalesced)
  //         and 2. err = ||X - I||_F in the same sweep.  k <= 128: here, into
  //         shared memory; loads are batched 16 per thread before any store
  //         (the L2 latency, not bandwidth, bounds this phase).  k > 128: by
  //         factor_prep_kernel ahead of this kernel.
  if (xs && a.policy == CQR_POLICY_UPDATE && a.q > 0 && a.bt_stage) {
    // deflated X = G - Bt^T Bt (algorithms.py:358-366).  Bt (q x k) is staged
    // in the work area first (one coalesced sweep, latency overlapped across
    // all threads; column stride q + 1 against bank conflicts), then each
    // thread forms its elements' q-long dot products from shared memory with
    // eight accumulator chains, added in a fixed order.  One thread per element
    // streaming the chain from L2 took ~20 us at q = 256 (~40 at 496).
    const int q = a.q, ldb = q + 1;
    double* bts = Wsm + wdoubles;   // the launch sized shared memory for it (a.bt_stage)
    for (int base = tid; base < k * q; base += 8 * FK_THREADS) {
      double v[8];   // all loads of the batch in flight before any store
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * FK_THREADS;
        v[u] = (e < k * q) ? a.Bt[(int64_t)(e / q) * a.ldbt + e % q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * FK_THREADS;
        if (e < k * q) bts[(e / q) * ldb + e % q] = v[u];
      }
    }
    __syncthreads();
    for (int e = tid; e < k * k; e += FK_THREADS) {
      const int r = e % k, c = e / k;
      if (r < c) continue;
      const double* br = bts + r * ldb;
      const double* bc = bts + c * ldb;
      double d[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int l = 0;
      for (; l + 8 <= q; l += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) d[u] = fma(br[l + u], bc[l + u], d[u]);
      }
      for (; l < q; ++l) d[0] = fma(br[l], bc[l], d[0]);
      const double dd = ((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7]));
      const double x = a.G[(int64_t)c * a.ldg + r] - dd;
      Xs[(int64_t)c * k + r] = x;
      Xs[(int64_t)r * k + c] = x;
    }
    __syncthreads();
    double loc = 0.0;
    for (int e = tid; e < k * k; e += FK_THREADS) {
      const int r = e % k, c = e / k;
      if (r < c) continue;
      const double dd = Xs[(int64_t)c * k + r] - ((r == c) ? 1.0 : 0.0);
      loc += ((r == c) ? 1.0 : 2.0) * (dd * dd);
    }
    const double err = sqrt(block_sum(loc, red));
    double dml = -INFINITY;
    for (int j = tid; j < k; j += FK_THREADS) dml = fmax(dml, a.G[(int64_t)j * a.ldg + j]);
    const double dm = block_max(dml, red);
    if (tid == 0) {
      fs.err = err;
      fs.diag_max = dm;
    }
  } else if (xs) {
    const int kk32 = k * k;
    double loc = 0.0;
    for (int base = tid; base < kk32; base += 16 * FK_THREADS) {
      double v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int e = base + j * FK_THREADS;
        const int r = e % k, c = e / k;
        v[j] = (e < kk32 && r >= c) ? a.G[(int64_t)c * a.ldg + r] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int e = base + j * FK_THREADS;
        const int r = e % k, c = e / k;
        if (e < kk32 && r >= c) {
          double x = v[j];
          if (a.policy == CQR_POLICY_UPDATE && a.q > 0) {
            const double* br = a.Bt + (int64_t)r * a.ldbt;
            const double* bc = a.Bt + (int64_t)c * a.ldbt;
            double d = 0.0;
            for (int l = 0; l < a.q; ++l) d += br[l] * bc[l];
            x = x - d;
          }
          Xs[(int64_t)c * k + r] = x;
          Xs[(int64_t)r * k + c] = x;
          const double d = x - ((r == c) ? 1.0 : 0.0);
          loc += ((r == c) ? 1.0 : 2.0) * (d * d);
        }
      }
    }
    __syncthreads();
    const double err = sqrt(block_sum(loc, red));
    // decision-margin scale: max diag of the undeflated Gram (for updates the
    // deflated X is itself at rounding level when the block is dependent)
    double dml = -INFINITY;
    for (int j = tid; j < k; j += FK_THREADS) dml = fmax(dml, a.G[(int64_t)j * a.ldg + j]);
    const double dm = block_max(dml, red);
    if (tid == 0) {
      fs.err = err;
      fs.diag_max = dm;
    }
  } else {
    // X was formed in global memory by factor_prep_kernel; its per-tile
    // partials are combined here in tile order (fixed, so deterministic).  The
    // partials are loaded by all threads at once (one thread walking them took
    // ~2.7 us of dependent L2 round trips at k = 256), then summed by thread 0.
    const int nt = (k + 31) / 32, ntiles = nt * (nt + 1) / 2;
    double* pp = rowbuf;   // rowbuf | vec | wv: 3 kpad doubles, free here
    const int chunk = kpad;  // tiles per pass (3 doubles each)
    double e2 = 0.0, dm = -INFINITY, ff = 0.0;
    for (int b0 = 0; b0 < ntiles; b0 += chunk) {
      const int nb = min(chunk, ntiles - b0);
      for (int e = tid; e < 3 * nb; e += FK_THREADS) pp[e] = a.part[3 * b0 + e];
      __syncthreads();
      if (tid == 0)
        for (int b = 0; b < nb; ++b) {
          e2 += pp[3 * b];
          dm = fmax(dm, pp[3 * b + 1]);
          ff += pp[3 * b + 2];
        }
      __syncthreads();
    }
    if (tid == 0) {
      fs.err = sqrt(e2);
      fs.diag_max = dm;
      fs.fro = sqrt(ff);
    }
  }
  __syncthreads();
  const double err = fs.err;
  fmark(1);
  // `while not err < tol: if its == max_iter: ...` (algorithms.py:341-343):
  // convergence is tested before the iteration cap.
  bool done = false;
  if (a.check_tol && err < a.tol) {
    if (tid == 0) fs.code = CQR_CONVERGED;
    done = true;
  } else if (a.stop) {
    if (tid == 0) fs.code = CQR_CAPPED;
    done = true;
  }

  // ---- 3. factorization attempts per policy
  bool ok = false;
  double sigma = 0.0;
  if (!done) {
    const double u2 = 2.0 * a.u;
    switch (a.policy) {
      case CQR_POLICY_PLAIN:
        ok = chol_attempt(Xs, Xg, k, 0.0, Wsm, a.W, a.Rk, a.ldr, rowbuf, fs, &sflag);
        break;
      case CQR_POLICY_FIXED_SHIFT:
        sigma = a.fixed_shift;
        if (tid == 0) { a.shifts[0] = sigma; fs.n_shifts = 1; }
        ok = chol_attempt(Xs, Xg, k, sigma, Wsm, a.W, a.Rk, a.ldr, rowbuf, fs, &sflag);
        break;
      case CQR_POLICY_ESTIMATE: {
        const double est = norm_estimate_x(Xs, Xg, k, a.est_tol, a.est_max_iter, vec, wv, red, fs, Wsm, wdoubles);
        __syncthreads();
        if (tid == 0) {
          if (fs.code != CQR_ASYMMETRIC) fs.code = CQR_ESTIMATED;
          fs.norm_est = est;
          fs.est_calls = 1;
        }
        done = true;
        break;
      }
      case CQR_POLICY_SHIFT_ONCE: {
        const double est = norm_estimate_x(Xs, Xg, k, a.est_tol, a.est_max_iter, vec, wv, red, fs, Wsm, wdoubles);
        __syncthreads();
        if (fs.code == CQR_ASYMMETRIC) { done = true; break; }
        sigma = shift_value(a.m_global, a.shift_width, est, a.u);
        if (tid == 0) { fs.est_calls = 1; fs.norm_est = est; a.shifts[0] = sigma; fs.n_shifts = 1; }
        ok = chol_attempt(Xs, Xg, k, sigma, Wsm, a.W, a.Rk, a.ldr, rowbuf, fs, &sflag);
        break;
      }
      case CQR_POLICY_RECOMPUTE: {
        if (spec1) {
          // the branch after a failed plain attempt, run ahead on a second SM;
          // the plain attempt's record (attempt 1, its margin) is merged later
          if (tid == 0) fs.attempts = 1;
          __syncthreads();
        } else {
          ok = chol_attempt(Xs, Xg, k, 0.0, Wsm, a.W, a.Rk, a.ldr, rowbuf, fs, &sflag);
          if (ok || a.spec) break;
        }
        const double est = norm_estimate_x(Xs, Xg, k, a.est_tol, a.est_max_iter, vec, wv, red, fs, Wsm, wdoubles);
        __syncthreads();
        if (fs.code == CQR_ASYMMETRIC) { done = true; break; }
        // (cluster groups poll inside the band steps only: an abort there is
        // published with the band and agreed on by the whole cluster)
        if (C == 1 && spec_should_stop(fs)) { done = true; break; }
        sigma = shift_value(a.m_global, a.shift_width, est, a.u);
        if (tid == 0) { fs.est_calls = 1; fs.norm_est = est; }
        int retries = 0, nsh = 0;
        while (true) {
          ++retries;
          if (retries > a.max_shift_attempts) {
            if (tid == 0) { fs.code = CQR_SHIFT_LIMIT; fs.retries = retries - 1; fs.last_shift = sigma; }
            done = true;
            break;
          }
          if (tid == 0) shx[nsh] = sigma;
          ++nsh;
          ok = chol_attempt(Xs, Xg, k, sigma, Wsm, gWx, Rkx, ldrx, rowbuf, fs, &sflag);
          if (ok) break;
          if (fs.aborted) { done = true; break; }   // speculative CTA: the plain attempt held
          if (tid == 0) fs.escalations += 1;
          sigma = py_max(a.esc * sigma, u2);
        }
        if (tid == 0) { fs.n_shifts = nsh; if (!done) fs.retries = retries; }
        break;
      }
      case CQR_POLICY_UPDATE: {
        int retries = 0, nsh = 0;
        sigma = 0.0;
        while (true) {
          ok = chol_attempt(Xs, Xg, k, sigma, Wsm, a.W, a.Rk, a.ldr, rowbuf, fs, &sflag);
          if (ok) break;
          ++retries;
          if (retries > a.max_shift_attempts) {
            if (tid == 0) { fs.code = CQR_SHIFT_LIMIT; fs.retries = retries - 1; fs.last_shift = sigma; }
            done = true;
            break;
          }
          if (sigma == 0.0) {
            const double est = norm_estimate_x(Xs, Xg, k, a.est_tol, a.est_max_iter, vec, wv, red, fs, Wsm, wdoubles);
            __syncthreads();
            if (fs.code == CQR_ASYMMETRIC) { done = true; break; }
            if (tid == 0) { fs.est_calls += 1; fs.norm_est = est; }
            sigma = shift_value(a.m_global, a.shift_width, est, a.u);
          } else {
            if (tid == 0) fs.escalations += 1;
            sigma = a.esc * sigma;
          }
          sigma = py_max(sigma, u2);
          if (tid == 0) a.shifts[nsh] = sigma;
          ++nsh;
        }
        if (tid == 0) { fs.n_shifts = nsh; if (!done) fs.retries = retries; }
        break;
      }
      default:
        break;
    }
    __syncthreads();
    if (a.spec && a.policy == CQR_POLICY_RECOMPUTE && !spec1) {
      // ---- group 0 publishes its outcome (pub: [flag, plain_margin, pivot_value,
      // pivot_index]) for group 1's polls and for the finish kernel, which takes
      // group 1's result when the plain attempt broke down.  Nobody waits on it.
      if (tid == 0 && crank == 0) {
        if (!ok) {
          a.pub[1] = fs.plain_margin;
          a.pub[2] = fs.pivot_value;
          a.pub[3] = (double)fs.pivot_index;
        }
        __threadfence();
        *reinterpret_cast<volatile unsigned long long*>(a.pub) =
            (0xC9F0A5ull << 40) | ((unsigned long long)a.epoch << 2) | (ok ? 1ull : 2ull);
      }
      if (!ok) return;   // the pass continues with group 1's result
    }
    if (!done && !ok) {
      if (tid == 0) fs.code = CQR_BREAKDOWN;
      done = true;
    }
  }

  // the group's rank 0 completes the pass: group 0 into Rk and the status,
  // the speculative group 1 into its private Rk1 and status record (pub)
  if (crank != 0) return;
  double* Ro = spec1 ? a.Rk1 : a.Rk;
  const int ldo = spec1 ? a.ldr1 : a.ldr;
  if (!done) {
    // ---- 4. TriangularSingularError check, decision margin, zero lower part + padding of Rk
    double tl = -INFINITY, zl = INFINITY;
    for (int j = tid; j < k; j += FK_THREADS) {
      tl = fmax(tl, __dadd_rn(xs ? Xs[(int64_t)j * k + j] : __ldg(Xg + (int64_t)j * k + j), sigma));
      if (__ldcg(Ro + (int64_t)j * ldo + j) == 0.0) zl = fmin(zl, (double)j);
    }
    const double top = block_max(tl, red);
    const double zfirst = -block_max(-zl, red);
    if (tid == 0) {
      if (zfirst < INFINITY) { fs.code = CQR_TRI_SINGULAR; fs.singular_index = (int)zfirst; }
      fs.min_pivot_rel = fs.min_pivot / top;
    }
    // k <= 256: only the lower parts of the 8 x 8 diagonal blocks here; the
    // blocks below them are zeroed by factor_finish_kernel (which never reads them)
    const int KP = (int)round_up(k, 32);
    for (int c = warp; c < k; c += FK_NW) {
      const int iend = (k <= 256) ? min(KP, (c | 7) + 1) : KP;
      for (int i = c + 1 + lane; i < iend; i += 32) Ro[(int64_t)c * ldo + i] = 0.0;
    }
  }

  __syncthreads();
  fmark(6);
  if (tid == 0) {
    cqr_factor_status rec{};
    rec.code = fs.code;
    rec.retries = fs.retries;
    rec.n_shifts = fs.n_shifts;
    rec.pivot_index = fs.pivot_index;
    rec.pivot_value = fs.pivot_value;
    rec.err = fs.err;
    rec.norm_est = fs.norm_est;
    rec.last_shift = fs.last_shift;
    rec.min_pivot_rel = fs.min_pivot_rel;
    rec.est_calls = fs.est_calls;
    rec.est_flag = fs.est_flag;
    rec.escalations = fs.escalations;
    rec.singular_index = fs.singular_index;
    rec.plain_margin = fs.plain_margin;
    rec.diag_max = fs.diag_max;
    *(spec1 ? reinterpret_cast<cqr_factor_status*>(a.pub + PUB_ST1) : a.st) = rec;
    if (!spec1 && a.stm != nullptr) {
      // host-mapped mirror: the host reads the pass's outcome without a D2H copy.
      // No system fence: kernel completion and the host's event wait order these
      // stores before the host's read (as for cqr_store_to_host)
      *a.stm = rec;
      for (int i = 0; i < fs.n_shifts; ++i) a.shm[i] = a.shifts[i];
    }
  }
}

// ---------------------------------------------------------------------------
// Speculative RECOMPUTE launches: group 0 (the plain attempt) and group 1 (the
// estimate and the shifted attempts) never wait on each other.  The finish
// kernel, stream-ordered after both, takes group 1's result when group 0's
// published flag says the plain attempt broke down.
__device__ __forceinline__ bool spec_selected(const FactorArgs& a) {
  if (!a.spec) return false;
  const unsigned long long f = *reinterpret_cast<const volatile unsigned long long*>(a.pub);
  return (f >> 2) == ((0xC9F0A5ull << 38) | (unsigned long long)a.epoch) && (f & 3ull) == 2ull;
}
// one thread: the pass's status from group 1's record plus the plain attempt's
// margin and breakdown (what the reference records for the failed attempt,
// algorithms.py:344-349), the shift list, the host-mapped mirrors
__device__ void spec_merge_status(const FactorArgs& a) {
  cqr_factor_status s = *reinterpret_cast<const cqr_factor_status*>(a.pub + PUB_ST1);
  s.plain_margin = a.pub[1];
  if (s.pivot_index < 0) { s.pivot_value = a.pub[2]; s.pivot_index = (int)a.pub[3]; }
  *a.st = s;
  for (int i = 0; i < s.n_shifts; ++i) a.shifts[i] = a.shifts1[i];
  if (a.stm != nullptr) {   // (kernel completion orders these before the host's read)
    *a.stm = s;
    for (int i = 0; i < s.n_shifts; ++i) a.shm[i] = a.shifts1[i];
  }
}

// ---------------------------------------------------------------------------
// finish: two CTAs per 8-column block J (one for B/Racc, one for Rinv),
// everything in 8x8 blocks with DMMA
//   B(:, J)     += Bt Racc_old(:, J)                      (algorithms.py:445)
//   Racc(I, J)   = sum_{L=I..J} Rk(I, L) Racc_old(L, J)   (kernels.py:103-114, triu)
//   Rinv(I, J)   = inv(R_II) (delta_IJ - sum_{L>I} R(I, L) Rinv(L, J)),
//                  block back substitution I = J .. 0    (kernels.py:85-100)
// Rk / Racc are column-major (ldr, rows >= k zero); rows/cols >= k of the
// last block act as identity.  Rinv goes straight into coefficient tiles.
constexpr int FF_WARPS = 8;

// A fragment of block (I, L) of a column-major matrix: A[m][kk] = M(8I+m, 8L+kk)
__device__ __forceinline__ double frag_a(const double* M, int ldm, int I, int L, int g, int t, int h) {
  return M[(int64_t)(8 * L + t + 4 * h) * ldm + 8 * I + g];
}
// B fragment of block (L, J): B[kk][n] = M(8L+kk, 8J+n)
__device__ __forceinline__ double frag_b(const double* M, int ldm, int L, int J, int g, int t, int h) {
  return M[(int64_t)(8 * J + g) * ldm + 8 * L + t + 4 * h];
}

__global__ void __launch_bounds__(FF_WARPS * 32) factor_finish_kernel(FactorArgs a) {
  // Two independent CTA roles per 8-column block J, run side by side:
  //   role 1 (blockIdx >= nblk): B += Bt Racc_old(:, J); Racc(:, J) <- Rk Racc_old(:, J)
  //   role 0: inverses of the diagonal blocks, Rinv(:, J) by block back substitution
  // sOld (Racc_old(:, J), role 1) and sX (Rinv(I, J) blocks, role 0) share storage
  __shared__ double sU[256 * 9];
  __shared__ double sInv[32][64];      // inv(R_II), column-major 8x8
  __shared__ double sPart[FF_WARPS][64];
  double (*sOld)[9] = reinterpret_cast<double (*)[9]>(sU);   // rows (<= 256) x 8, padded
  double (*sX)[64] = reinterpret_cast<double (*)[64]>(sU);   // 32 blocks, column-major 8x8
  const bool sel1 = spec_selected(a);
  if (sel1 && blockIdx.x == 0 && threadIdx.x == 0) spec_merge_status(a);
  const cqr_factor_status* st = sel1 ? reinterpret_cast<const cqr_factor_status*>(a.pub + PUB_ST1) : a.st;
  if (st->code != CQR_FACTORED) return;
  const int k = a.k;
  const int nblk = (k + 7) / 8;
  const int role = (int)blockIdx.x / nblk;
  const int J = (int)blockIdx.x - role * nblk;
  const bool prof = (J == nblk - 1 && threadIdx.x == 0);   // the longest column block
  long long fc0 = prof ? clock64() : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int ldr = a.ldr;                       // Rk, Racc
  const double* R = sel1 ? a.Rk1 : a.Rk;       // the selected factor (read only here)
  const int ldR = sel1 ? a.ldr1 : a.ldr;
  const int nrow = 8 * J + 8;          // rows 0 .. 8J+7 of the column block

  if (role == 1) {
    // ---- stage Racc_old(:, J) (rows < nrow) and update B with it
    for (int e = threadIdx.x; e < nrow * 8; e += FF_WARPS * 32) {
      const int r = e % nrow, cl = e / nrow, c = 8 * J + cl;
      sOld[r][cl] = (c < k) ? a.Racc[(int64_t)c * ldr + r] : ((r == c) ? 1.0 : 0.0);
    }
    __syncthreads();
    if (a.update_b && a.q > 0) {
      for (int e = threadIdx.x; e < a.q * 8; e += FF_WARPS * 32) {
        const int i = e % a.q, cl = e / a.q, c = 8 * J + cl;
        if (c >= k) continue;
        double s = 0.0;
        for (int l = 0; l <= c; ++l) s += a.Bt[(int64_t)l * a.ldbt + i] * sOld[l][cl];
        a.B[(int64_t)c * a.ldb + i] = a.B[(int64_t)c * a.ldb + i] + s;
      }
    }
    if (!a.accumulate) return;
    // ---- Racc(I, J) = sum_L Rk(I, L) Racc_old(L, J): warps over I.  Only this
    // CTA reads or writes column block J of Racc (its old values are staged)
    for (int I = warp; I <= J; I += FF_WARPS) {
      double c2[2] = {0.0, 0.0};
      const int ra = 8 * I + g;
      // Rk(I, L) fragments come from L2: load 4 L steps at once so the
      // latencies overlap (the DMMA order over L is unchanged)
      for (int L0 = I; L0 <= J; L0 += 4) {
        double av[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int L = L0 + j, ca = 8 * L + t + 4 * h;
            av[j][h] = (L <= J) ? ((ra < k && ca < k) ? R[(int64_t)ca * ldR + ra] : ((ra == ca) ? 1.0 : 0.0)) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int L = L0 + j;
          if (L > J) break;
#pragma unroll
          for (int h = 0; h < 2; ++h) dmma(c2, av[j][h], sOld[8 * L + t + 4 * h][g]);
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        if (c < k && r < k) a.Racc[(int64_t)c * ldr + r] = (r <= c) ? c2[e] : 0.0;
      }
    }
    if (prof) g_fprof[13] = (unsigned long long)(clock64() - fc0);
    return;
  }
  // ---- zero Rk below the diagonal blocks in column block J (rows 8J+8 .. KP);
  // group 1's factor is copied into Rk (the pass's R) on the way
  {
    const int KP = (int)round_up(k, 32);
    for (int e = threadIdx.x; e < 8 * KP; e += FF_WARPS * 32) {
      const int cl = e / KP, i = e % KP, c = 8 * J + cl;
      if (c >= k) continue;
      if (i >= nrow) a.Rk[(int64_t)c * ldr + i] = 0.0;
      else if (sel1) a.Rk[(int64_t)c * ldr + i] = R[(int64_t)c * ldR + i];
    }
  }
  // ---- inverses of the diagonal blocks I <= J (warp per block, lanes 0..7 one column each)
  // all 32 lanes: lane = 8 * sub + cl handles block I = warp + 8 (4 i + sub)
  // column cl (four blocks per warp at once); the 8 diagonal reciprocals are
  // independent divisions, so the substitution chain itself is FMA only
  for (int I0 = warp; I0 <= J; I0 += 4 * FF_WARPS) {
    const int I = I0 + FF_WARPS * (lane >> 3);
    const int cl = lane & 7;
    if (I <= J) {
      double rr[8][8];   // R_II(r, l), upper part
      double dinv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int l = r + 1; l < 8; ++l) {
          const int ri = 8 * I + r, cj = 8 * I + l;
          rr[r][l] = (ri < k && cj < k) ? R[(int64_t)cj * ldR + ri] : 0.0;
        }
        const int di = 8 * I + r;
        dinv[r] = 1.0 / ((di < k) ? R[(int64_t)di * ldR + di] : 1.0);
      }
      // column cl of inv(R_II): back substitution R_II x = e_cl
      double x[8];
#pragma unroll
      for (int r = 7; r >= 0; --r) {
        double sacc = (r == cl) ? 1.0 : 0.0;
#pragma unroll
        for (int l = r + 1; l < 8; ++l) sacc -= rr[r][l] * x[l];
        x[r] = (r <= cl) ? sacc * dinv[r] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) sInv[I][cl * 8 + r] = x[r];
    }
  }
  __syncthreads();
  if (prof) g_fprof[14] = (unsigned long long)(clock64() - fc0);
  // ---- R^-1(:, J) by right-looking block back substitution.  Warp w owns the
  // block rows I' = w + 8 s; acc[s] collects sum_{L > I'} R(I', L) X_L as each
  // X_L is published (L descending), so step I only waits for X_{I+1}'s term
  // of row I: one barrier and four dependent DMMAs per step, against two
  // barriers, a partial-sum reduction and 8x8 products over all L before.
  // R(I', L) fragments are loaded two steps ahead.
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { acc[j][0] = 0.0; acc[j][1] = 0.0; }
  auto load_col = [&](int L, double (&fr)[4][2]) {   // R(I', L) for this warp's rows I' < L
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int Ip = warp + FF_WARPS * j;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ra = 8 * Ip + g, ca = 8 * L + t + 4 * h;
        fr[j][h] = (L >= 0 && Ip < L && ra < k && ca < k) ? R[(int64_t)ca * ldR + ra] : 0.0;
      }
    }
  };
  double (*sM)[64] = sPart;   // the owner warp's M, column-major
  auto step = [&](int I, const double (&fr)[4][2]) {
    if (warp == (I & (FF_WARPS - 1))) {
      // X_I = inv(R_II) (delta_IJ I - S_I)
      const int sl = I / FF_WARPS;
      double s0 = acc[0][0], s1 = acc[0][1];
#pragma unroll
      for (int j = 1; j < 4; ++j)
        if (sl == j) { s0 = acc[j][0]; s1 = acc[j][1]; }
      sM[warp][(2 * t) * 8 + g] = ((I == J && g == 2 * t) ? 1.0 : 0.0) - s0;
      sM[warp][(2 * t + 1) * 8 + g] = ((I == J && g == 2 * t + 1) ? 1.0 : 0.0) - s1;
      __syncwarp();
      double x2[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) dmma(x2, sInv[I][(t + 4 * h) * 8 + g], sM[warp][g * 8 + t + 4 * h]);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        const double v = (I == J && g > 2 * t + e) ? 0.0 : x2[e];
        sX[I][(2 * t + e) * 8 + g] = v;
        if (r < k && c < k) a.Rinv[coeff_off(r, c, k)] = v;
      }
    }
    __syncthreads();   // X_I is published
    // X_I's term for every row above it, the highest first (row I - 1 is on
    // the critical path: its owner computes X_{I-1} next)
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      const int Ip = warp + FF_WARPS * j;
      if (Ip < I) {
#pragma unroll
        for (int h = 0; h < 2; ++h) dmma(acc[j], fr[j][h], sX[I][g * 8 + t + 4 * h]);
      }
    }
  };
  // two fragment sets used alternately, each reloaded right after its step for
  // the step after next (no register moves that would wait on the loads)
  double fr0[4][2], fr1[4][2];
  load_col(J, fr0);
  load_col(J - 1, fr1);
  for (int I = J; I >= 0; I -= 2) {
    step(I, fr0);
    load_col(I - 2, fr0);
    if (I >= 1) {
      step(I - 1, fr1);
      load_col(I - 3, fr1);
    }
  }
  if (prof) g_fprof[15] = (unsigned long long)(clock64() - fc0);
}

// generic (k > 256) finish: one warp per column, R columns staged through
// shared memory.  Same operations as factor_finish_kernel.
constexpr int FW_WARPS = 8;

__global__ void __launch_bounds__(FW_WARPS * 32) factor_finish_wide_kernel(FactorArgs a) {
  extern __shared__ __align__(16) double ffs[];
  const bool sel1 = spec_selected(a);
  if (sel1 && blockIdx.x == 0 && threadIdx.x == 0) spec_merge_status(a);
  const cqr_factor_status* st = sel1 ? reinterpret_cast<const cqr_factor_status*>(a.pub + PUB_ST1) : a.st;
  if (st->code != CQR_FACTORED) return;
  const int k = a.k;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int c0 = blockIdx.x * FW_WARPS;
  const int c = c0 + wl;
  const bool active = c < k;
  double* col = ffs + (size_t)wl * k;                 // per-warp column scratch
  double* rbuf = ffs + (size_t)FW_WARPS * k;          // 2 x k: staged column of R
  const int ldr = a.ldr;
  const int KP = (int)round_up(k, 32);
  const double* R = sel1 ? a.Rk1 : a.Rk;       // the selected factor
  const int ldR = sel1 ? a.ldr1 : a.ldr;
  if (active && sel1)
    for (int i = lane; i < KP; i += 32) a.Rk[(int64_t)c * ldr + i] = R[(int64_t)c * ldR + i];
  if (active) {
    // old Racc column c
    for (int l = lane; l <= c; l += 32) col[l] = a.Racc[(int64_t)c * ldr + l];
    __syncwarp();
    if (a.update_b && a.q > 0) {
      for (int i = lane; i < a.q; i += 32) {
        double s = 0.0;
        for (int l = 0; l <= c; ++l) s += a.Bt[(int64_t)l * a.ldbt + i] * col[l];
        a.B[(int64_t)c * a.ldb + i] = a.B[(int64_t)c * a.ldb + i] + s;
      }
    }
    if (a.accumulate) {
      // new(i) = sum_{l=i..c} R(i,l) old(l): lanes own rows i, loop over l (coalesced columns of R)
      for (int i0 = 0; i0 <= c; i0 += 32) {
        const int i = i0 + lane;
        double s = 0.0;
#pragma unroll 8
        for (int l = i0; l <= c; ++l) {
          const double r = (i <= l) ? R[(int64_t)l * ldR + i] : 0.0;
          s += r * col[l];
        }
        if (i <= c) a.Racc[(int64_t)c * ldr + i] = s;
      }
      for (int i = c + 1 + lane; i < KP; i += 32) a.Racc[(int64_t)c * ldr + i] = 0.0;
    }
    __syncwarp();
    // inverse column: acc = e_c
    for (int l = lane; l <= c; l += 32) col[l] = (l == c) ? 1.0 : 0.0;
  }
  // back substitution for the CTA's columns together: step i uses column i of R,
  // staged in shared memory (double buffered, next column prefetched into
  // registers while the current step computes)
  const int cmax = min(c0 + FW_WARPS - 1, k - 1);
  const int nthr = FW_WARPS * 32;
  for (int l = threadIdx.x; l <= cmax; l += nthr) rbuf[l] = R[(int64_t)cmax * ldR + l];
  int cur = 0;
  double* out = a.Rinv + coeff_off(0, active ? c : 0, k);
  for (int i = cmax; i >= 0; --i) {
    __syncthreads();
    const double* rc = rbuf + cur * k;
    // prefetch column i-1 (rows 0..i-1)
    double pre[4];
    int npre = 0;
    if (i > 0)
      for (int l = threadIdx.x; l < i && npre < 4; l += nthr) pre[npre++] = R[(int64_t)(i - 1) * ldR + l];
    if (active && c >= i) {
      const double x = col[i] / rc[i];
      if (lane == 0) out[(i / CT_K) * CT_TILE + i % CT_K] = x;
      for (int l = lane; l < i; l += 32) col[l] -= rc[l] * x;
    }
    if (i > 0) {
      double* rn = rbuf + (cur ^ 1) * k;
      int q = 0;
      for (int l = threadIdx.x; l < i && q < 4; l += nthr) rn[l] = pre[q++];
      for (int l = threadIdx.x + 4 * nthr; l < i; l += nthr) rn[l] = R[(int64_t)(i - 1) * ldR + l];
    }
    cur ^= 1;
  }
  if (active)
    for (int i = c + 1 + lane; i < KP; i += 32) out[(i / CT_K) * CT_TILE + i % CT_K] = 0.0;
}

static int g_cluster_mode = 1;   // host: band-cluster path for 96 < k <= 256 (cqr_debug_factor_cluster)

int factor_set_cluster(int on) {
  g_cluster_mode = (on >= 0 && on <= 2) ? on : 1;
  return 0;
}

int factor_set_banded(int on) {
  const int v = on ? 1 : 0;
  return cudaMemcpyToSymbol(g_banded, &v, sizeof(int)) == cudaSuccess ? 0 : -1;
}

int factor_cluster_profile(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_cprof, sizeof(g_cprof)) == cudaSuccess ? 0 : -1;
}

// diagnostics: per-step stamps of CTA `cta` (-1: off); out = [4][8] stamps
int factor_step_profile(int cta, long long* out) {
  if (out != nullptr) return cudaMemcpyFromSymbol(out, g_sprof, sizeof(g_sprof)) == cudaSuccess ? 0 : -1;
  return cudaMemcpyToSymbol(g_sprof_cta, &cta, sizeof(int)) == cudaSuccess ? 0 : -1;
}

int factor_profile(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_fprof, sizeof(g_fprof)) == cudaSuccess ? 0 : -1;
}

size_t factor_workspace_bytes(int k) {
  // X (k^2) | W + Ri (k (k+1)) | speculative CTA: Rk1 (k x round_up(k, 32)), W1 (k (k+1)), shifts1 (1024), pub (64)
  // | prep partials (3 per 32 x 32 tile of the lower triangle)
  const size_t kk = (size_t)k;
  const size_t nt = (kk + 31) / 32;
  return (kk * kk + 2 * kk * (kk + 1) + kk * (size_t)round_up(k, 32) + 1024 + 64 + 2 * nt * (nt + 1)) * sizeof(double) + 512;
}

cudaError_t factor_launch(FactorArgs& a, cudaStream_t stream) {
  if (a.k < 1 || a.k > FK_MAX_K) return cudaErrorInvalidValue;
  const int kpad = (int)round_up(a.k, 8);
  size_t smem = (32 + 3 * (size_t)kpad) * sizeof(double);
  // k <= 128: X, then the block-packed triangle; 128 < k <= 256: the band or the
  // trailing triangle; k <= 768: one 32-row band (work_doubles)
  smem += ((a.k <= FK_SMEM_K ? (size_t)a.k * a.k : 0) + (size_t)work_doubles(a.k)) * sizeof(double);
  // update policy, k <= 128: room to stage Bt (q x k, column stride q + 1) for the deflation
  a.bt_stage = 0;
  if (a.policy == CQR_POLICY_UPDATE && a.q > 0 && a.k <= FK_SMEM_K) {
    const size_t extra = (size_t)a.k * (a.q + 1) * sizeof(double);
    if (smem + extra <= 220 * 1024) { smem += extra; a.bt_stage = 1; }
  }
  {
    const size_t mx = 220 * 1024;  // <= 227 KB minus the static shared state
    cudaError_t e = smem_attr((const void*)factor_kernel, mx);
    if (e == cudaSuccess) e = smem_attr((const void*)factor_finish_wide_kernel, mx);
    if (e != cudaSuccess) return e;
  }
  static unsigned epoch = 0;
  a.epoch = ++epoch;   // tags the speculative handshake of this launch (no reset launch needed)
  // band-cluster path: one cluster of ceil(k / 32) CTAs per attempt chain (band r on
  // CTA r) for 128 < k <= 256, and from 96 < k for the policies that run a norm
  // estimate (its distributed power iteration is where 4 bands gain: k = 128
  // shifted calls 121 -> 105 us; a plain k = 128 call measured 0.095 -> 0.103 ms
  // in config 2, and with 2-3 bands the hand-overs cost what the cluster
  // distributes).  Mode 2 (diagnostics): from 64 < k for every policy but the
  // update policy's deflation, which stays on the single CTA at k <= 128.
  const bool est_policy = a.policy == CQR_POLICY_SHIFT_ONCE || a.policy == CQR_POLICY_RECOMPUTE ||
                          a.policy == CQR_POLICY_ESTIMATE;
  const bool small_ok = !(a.policy == CQR_POLICY_UPDATE && a.q > 0);
  const int kmin = !small_ok ? FK_SMEM_K : (g_cluster_mode == 2 ? 64 : (est_policy ? 96 : FK_SMEM_K));
  a.ncl = (g_cluster_mode && a.k > kmin && a.k <= FK_BIG_K) ? (a.k + 31) / 32 : 1;
  if (a.k > FK_SMEM_K || a.ncl > 1) {
    const int nt = (a.k + 31) / 32;
    factor_prep_kernel<<<nt * (nt + 1) / 2, FP_THREADS, 0, stream>>>(a);
  }
  if (a.ncl > 1) {
    smem = (32 + 3 * (size_t)kpad + (size_t)cluster_work_doubles(a.k)) * sizeof(double);
  }
  // The speculative RECOMPUTE launch runs two groups (plain; estimate + shifted
  // attempts) side by side; neither waits on the other (the finish kernel
  // merges), so they need not be co-scheduled.  Within a group the band
  // hand-over does wait, and the cluster guarantees co-residency.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.spec ? 2 : 1) * a.ncl);
  cfg.blockDim = dim3(FK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.ncl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.ncl > 1 ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, factor_kernel, a);
  if (e != cudaSuccess) return e;
  const int blocks = (a.k + 7) / 8;
  if (a.k <= 256) {
    factor_finish_kernel<<<2 * blocks, FF_WARPS * 32, 0, stream>>>(a);   // two roles per column block
  } else {
    factor_finish_wide_kernel<<<(a.k + FW_WARPS - 1) / FW_WARPS, FW_WARPS * 32,
                                (size_t)(FW_WARPS + 2) * a.k * sizeof(double), stream>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace cqr
