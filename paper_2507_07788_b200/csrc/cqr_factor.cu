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
// Storage: X (the symmetric input) is kept in a k x k global workspace (L2
// resident) so shifted retries can restart from it; the Cholesky factor W and
// the inverse accumulator Ri are packed upper triangles, in shared memory for
// k <= 128 (2 x 66 KB) and in global workspace otherwise.  The Cholesky is
// right-looking (row j scaled, rank-1 trailing update), the inverse is the
// row-by-row back substitution R Rinv = I with rank-1 updates; both need two
// block barriers per step.  All reductions use a fixed order, so results are
// bitwise reproducible run to run.
#include <cmath>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int FK_THREADS = 512;
constexpr int FK_NW = FK_THREADS / 32;
constexpr int FK_SMEM_K = 128;
constexpr int FK_MAX_K = 2048;

__host__ __device__ __forceinline__ int64_t pk(int i, int c) { return (int64_t)c * (c + 1) / 2 + i; }

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

// compute_shift (kernels.py:194): ((11 * N) * u) * norm, then Python max with 2u.
__device__ __forceinline__ double shift_value(int64_t m, int64_t w, double norm, double u) {
  const double N = (double)(m * w + w * (w + 1));
  const double s = __dmul_rn(__dmul_rn(__dmul_rn(11.0, N), u), norm);
  return py_max(s, 2.0 * u);
}

struct FState {
  int code, retries, n_shifts, pivot_index, est_calls, est_flag, escalations, singular_index;
  double pivot_value, err, norm_est, last_shift, min_pivot_rel, sigma;
};

// One factorization attempt of X + sigma I into the packed upper factor W.
// Returns true on success; on breakdown records the pivot in fs (thread 0).
__device__ bool chol_attempt(const double* __restrict__ X, int k, double sigma, double* W, double* rowbuf,
                             FState& fs) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = warp; c < k; c += FK_NW)
    for (int i = lane; i <= c; i += 32) {
      double x = X[(int64_t)c * k + i];
      if (i == c) x = __dadd_rn(x, sigma);
      W[pk(i, c)] = x;
    }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double s = W[pk(j, j)];
    if (!(s > 0.0)) {
      if (tid == 0) { fs.pivot_index = j; fs.pivot_value = s; }
      __syncthreads();
      return false;
    }
    const double d = sqrt(s);
    for (int c = j + 1 + tid; c < k; c += FK_THREADS) {
      const double v = W[pk(j, c)] / d;
      W[pk(j, c)] = v;
      rowbuf[c] = v;
    }
    __syncthreads();
    if (tid == 0) W[pk(j, j)] = d;
    for (int c = j + 1 + warp; c < k; c += FK_NW) {
      const double rc = rowbuf[c];
      double* col = W + pk(0, c);
      for (int i = j + 1 + lane; i <= c; i += 32) col[i] -= rowbuf[i] * rc;
    }
    __syncthreads();
  }
  return true;
}

// spectral_norm_estimate (kernels.py:126-178) on the full symmetric X.
// Returns the estimate; sets fs.est_flag (1 stalled, 2 not converged) and
// fs.code = CQR_ASYMMETRIC on the asymmetry ValueError.
__device__ double norm_estimate(const double* __restrict__ X, int k, double tol, int max_iter, double* vec,
                                double* wv, double* red, FState& fs) {
  const int tid = threadIdx.x;
  const int64_t kk = (int64_t)k * k;
  double loc = 0.0, la = 0.0;
  for (int64_t e = tid; e < kk; e += FK_THREADS) {
    const double x = X[e];
    loc += x * x;
    const int i = (int)(e % k), c = (int)(e / k);
    const double d = x - X[(int64_t)i * k + c];
    la += d * d;
  }
  const double fro = sqrt(block_sum(loc, red));
  const double asym = sqrt(block_sum(la, red));
  if (fro == 0.0) return 0.0;
  if (asym > 1e-8 * fro) {
    if (tid == 0) fs.code = CQR_ASYMMETRIC;
    return fro;
  }
  const double v0 = 1.0 / sqrt((double)k);
  for (int i = tid; i < k; i += FK_THREADS) vec[i] = v0;
  __syncthreads();
  bool have_prev = false;
  double prev = 0.0;
  for (int it = 0; it < max_iter; ++it) {
    double nw_loc = 0.0;
    for (int i = tid; i < k; i += FK_THREADS) {
      double s = 0.0;
      for (int c = 0; c < k; ++c) s += X[(int64_t)c * k + i] * vec[c];
      wv[i] = s;
      nw_loc += s * s;
    }
    const double nw = sqrt(block_sum(nw_loc, red));
    if (nw == 0.0) {
      if (tid == 0) fs.est_flag = 1;
      return fro;
    }
    double vw_loc = 0.0;
    for (int i = tid; i < k; i += FK_THREADS) vw_loc += vec[i] * wv[i];
    const double lam = block_sum(vw_loc, red);
    for (int i = tid; i < k; i += FK_THREADS) vec[i] = wv[i] / nw;
    __syncthreads();
    if (have_prev && fabs(lam - prev) <= tol * fabs(lam)) return fabs(lam);
    prev = lam;
    have_prev = true;
  }
  if (tid == 0) fs.est_flag = 2;
  return fro;
}

__global__ void __launch_bounds__(FK_THREADS) factor_kernel(FactorArgs a) {
  extern __shared__ __align__(16) double fsm[];
  __shared__ FState fs;
  const int k = a.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kpad = (int)round_up(k, 2);
  const int64_t npk = pk(0, k);  // k (k+1) / 2
  double* red = fsm;
  double* rowbuf = fsm + 32;
  double* vec = rowbuf + kpad;
  double* wv = vec + kpad;
  double* W = (k <= FK_SMEM_K) ? wv + kpad : a.W;
  double* Ri = (k <= FK_SMEM_K) ? W + npk : a.Ri;
  double* X = a.X;

  if (tid == 0) {
    fs.code = CQR_FACTORED; fs.retries = 0; fs.n_shifts = 0; fs.pivot_index = -1; fs.est_calls = 0;
    fs.est_flag = 0; fs.escalations = 0; fs.singular_index = -1;
    fs.pivot_value = 0.0; fs.err = 0.0; fs.norm_est = 0.0; fs.last_shift = 0.0; fs.min_pivot_rel = 0.0;
    fs.sigma = 0.0;
  }

  // ---- 1. X = G (or G - Bt^T Bt), symmetric by construction from the lower triangle
  const int64_t kk = (int64_t)k * k;
  for (int64_t e = tid; e < kk; e += FK_THREADS) {
    const int i = (int)(e % k), c = (int)(e / k);
    const int r = max(i, c), cc = min(i, c);
    double x = a.G[(int64_t)cc * a.ldg + r];
    if (a.policy == CQR_POLICY_UPDATE && a.q > 0) {
      const double* br = a.Bt + (int64_t)r * a.ldbt;
      const double* bc = a.Bt + (int64_t)cc * a.ldbt;
      double d = 0.0;
      for (int l = 0; l < a.q; ++l) d += br[l] * bc[l];
      x = x - d;
    }
    X[e] = x;
  }
  __syncthreads();

  // ---- 2. err = ||X - I||_F
  double loc = 0.0;
  for (int64_t e = tid; e < kk; e += FK_THREADS) {
    const double d = X[e] - (((e % k) == (e / k)) ? 1.0 : 0.0);
    loc += d * d;
  }
  const double err = sqrt(block_sum(loc, red));
  if (tid == 0) fs.err = err;

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
        ok = chol_attempt(X, k, 0.0, W, rowbuf, fs);
        break;
      case CQR_POLICY_SHIFT_ONCE: {
        const double est = norm_estimate(X, k, a.est_tol, a.est_max_iter, vec, wv, red, fs);
        __syncthreads();
        if (fs.code == CQR_ASYMMETRIC) { done = true; break; }
        sigma = shift_value(a.m_global, a.shift_width, est, a.u);
        if (tid == 0) { fs.est_calls = 1; fs.norm_est = est; a.shifts[0] = sigma; fs.n_shifts = 1; }
        ok = chol_attempt(X, k, sigma, W, rowbuf, fs);
        break;
      }
      case CQR_POLICY_RECOMPUTE: {
        ok = chol_attempt(X, k, 0.0, W, rowbuf, fs);
        if (ok) break;
        const double est = norm_estimate(X, k, a.est_tol, a.est_max_iter, vec, wv, red, fs);
        __syncthreads();
        if (fs.code == CQR_ASYMMETRIC) { done = true; break; }
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
          if (tid == 0) a.shifts[nsh] = sigma;
          ++nsh;
          ok = chol_attempt(X, k, sigma, W, rowbuf, fs);
          if (ok) break;
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
          ok = chol_attempt(X, k, sigma, W, rowbuf, fs);
          if (ok) break;
          ++retries;
          if (retries > a.max_shift_attempts) {
            if (tid == 0) { fs.code = CQR_SHIFT_LIMIT; fs.retries = retries - 1; fs.last_shift = sigma; }
            done = true;
            break;
          }
          if (sigma == 0.0) {
            const double est = norm_estimate(X, k, a.est_tol, a.est_max_iter, vec, wv, red, fs);
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
    if (!done && !ok) {
      if (tid == 0) fs.code = CQR_BREAKDOWN;
      done = true;
    }
  }

  if (!done) {
    // ---- 4. triangular inverse (zero diagonal -> TriangularSingularError)
    if (tid == 0) {
      for (int j = 0; j < k; ++j)
        if (W[pk(j, j)] == 0.0) { fs.code = CQR_TRI_SINGULAR; fs.singular_index = j; break; }
      double top = -INFINITY, mn = INFINITY;
      for (int j = 0; j < k; ++j) {
        const double xd = __dadd_rn(X[(int64_t)j * k + j], sigma);
        top = fmax(top, xd);
        const double d = W[pk(j, j)];
        mn = fmin(mn, d * d);
      }
      fs.min_pivot_rel = mn / top;
    }
    __syncthreads();
    if (fs.code == CQR_TRI_SINGULAR) done = true;
  }

  if (!done) {
    for (int64_t e = tid; e < npk; e += FK_THREADS) Ri[e] = 0.0;
    __syncthreads();
    for (int l = k - 1; l >= 0; --l) {
      const double rll = W[pk(l, l)];
      for (int c = l + tid; c < k; c += FK_THREADS) {
        const double v = (((c == l) ? 1.0 : 0.0) - Ri[pk(l, c)]) / rll;
        Ri[pk(l, c)] = v;
        rowbuf[c] = v;
      }
      __syncthreads();
      const double* rcol = W + pk(0, l);  // column l of R: rows 0..l
      for (int c = l + warp; c < k; c += FK_NW) {
        const double rc = rowbuf[c];
        double* col = Ri + pk(0, c);
        for (int i = lane; i < l; i += 32) col[i] += rcol[i] * rc;
      }
      __syncthreads();
    }
    // with R Rinv = I solved as Rinv(i,c) = (delta - sum_{l>i} R(i,l) Rinv(l,c)) / R(i,i),
    // the accumulator above holds +sum; rows were finalized as (delta - acc) / R(i,i).

    // ---- 5. write Rk and Rinv (ldr rows, zero below the diagonal and in the padding)
    const int KP = (int)round_up(k, 32);
    for (int64_t e = tid; e < (int64_t)KP * k; e += FK_THREADS) {
      const int i = (int)(e % KP), c = (int)(e / KP);
      const bool up = (i <= c);
      a.Rk[(int64_t)c * a.ldr + i] = up ? W[pk(i, c)] : 0.0;
      a.Rinv[(int64_t)c * a.ldr + i] = up ? Ri[pk(i, c)] : 0.0;
    }
    __syncthreads();

    // ---- 6. B <- B + Bt Racc_old  (q x k), before Racc changes
    if (a.update_b && a.q > 0) {
      for (int64_t e = tid; e < (int64_t)a.q * k; e += FK_THREADS) {
        const int i = (int)(e % a.q), j = (int)(e / a.q);
        double s = 0.0;
        for (int l = 0; l <= j; ++l) s += a.Bt[(int64_t)l * a.ldbt + i] * a.Racc[(int64_t)j * a.ldr + l];
        a.B[(int64_t)j * a.ldb + i] = a.B[(int64_t)j * a.ldb + i] + s;
      }
      __syncthreads();
    }

    // ---- 7. Racc <- triu(Rk Racc); staged through X (no longer needed)
    if (a.accumulate) {
      for (int64_t e = tid; e < kk; e += FK_THREADS) {
        const int i = (int)(e % k), c = (int)(e / k);
        double s = 0.0;
        if (i <= c)
          for (int l = i; l <= c; ++l) s += W[pk(i, l)] * a.Racc[(int64_t)c * a.ldr + l];
        X[e] = s;
      }
      __syncthreads();
      for (int64_t e = tid; e < kk; e += FK_THREADS) {
        const int i = (int)(e % k), c = (int)(e / k);
        a.Racc[(int64_t)c * a.ldr + i] = X[e];
      }
    }
  }

  __syncthreads();
  if (tid == 0) {
    cqr_factor_status* st = a.st;
    st->code = fs.code;
    st->retries = fs.retries;
    st->n_shifts = fs.n_shifts;
    st->pivot_index = fs.pivot_index;
    st->pivot_value = fs.pivot_value;
    st->err = fs.err;
    st->norm_est = fs.norm_est;
    st->last_shift = fs.last_shift;
    st->min_pivot_rel = fs.min_pivot_rel;
    st->est_calls = fs.est_calls;
    st->est_flag = fs.est_flag;
    st->escalations = fs.escalations;
    st->singular_index = fs.singular_index;
  }
}

size_t factor_workspace_bytes(int k) {
  size_t b = (size_t)k * k * sizeof(double);
  if (k > FK_SMEM_K) b += 2 * (size_t)pk(0, k) * sizeof(double) + 256;
  return b + 256;
}

cudaError_t factor_launch(FactorArgs& a, cudaStream_t stream) {
  if (a.k < 1 || a.k > FK_MAX_K) return cudaErrorInvalidValue;
  const int kpad = (int)round_up(a.k, 2);
  size_t smem = (32 + 3 * (size_t)kpad) * sizeof(double);
  if (a.k <= FK_SMEM_K) smem += 2 * (size_t)pk(0, a.k) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    const int mx = (int)((32 + 3 * FK_MAX_K) * sizeof(double) + 2 * pk(0, FK_SMEM_K) * sizeof(double));
    cudaError_t e = cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  factor_kernel<<<1, FK_THREADS, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace cqr
