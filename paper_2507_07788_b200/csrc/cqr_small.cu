// Standalone k x k kernels of the reference's kernel API (kernels.py:85-123):
// triangular inverse, triangular product, Frobenius norm.  The drivers never
// call these -- the factor kernel (cqr_factor.cu) does the same work inside its
// one launch per pass -- they back `paper_2507_07788_b200.kernels` so that code
// written against the reference's kernel functions runs on the device.
//
// All matrices column-major.  One CTA per launch: these are O(k^3) at k <= a few
// hundred, latency bound, and a fixed-order single-CTA reduction keeps the
// Frobenius norm bitwise reproducible.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int SM_THREADS = 256;

// X = R^-1 by back substitution, one thread per column j (column j of R^-1
// depends only on R): x_i = (delta_ij - sum_{l=i+1..j} R_il x_l) / R_ii for
// i = j .. 0.  The strictly lower part of the output is exactly zero
// (kernels.py:100: np.triu).  The caller has checked the diagonal for zeros
// (kernels.py:94-96).
__global__ void __launch_bounds__(SM_THREADS) tri_inverse_kernel(const double* __restrict__ R, int ldr, int n,
                                                                  double* __restrict__ X, int ldx) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double* x = X + (int64_t)j * ldx;
    for (int i = j + 1; i < n; ++i) x[i] = 0.0;
    for (int i = j; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int l = i + 1; l <= j; ++l) s -= R[(int64_t)l * ldr + i] * x[l];
      x[i] = s / R[(int64_t)i * ldr + i];
    }
  }
}

// C = triu(A B) for upper-triangular A, B: C_ij = sum_{l=i..j} A_il B_lj
// (kernels.py:103-114), zero below the diagonal.
__global__ void __launch_bounds__(SM_THREADS) tri_multiply_kernel(const double* __restrict__ A, int lda,
                                                                   const double* __restrict__ B, int ldb, int n,
                                                                   double* __restrict__ C, int ldc) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    double s = 0.0;
    for (int l = i; l <= j; ++l) s += A[(int64_t)l * lda + i] * B[(int64_t)j * ldb + l];
    C[(int64_t)j * ldc + i] = s;
  }
}

// sqrt(sum x^2) over a rows x cols block, one CTA, fixed order (each thread a
// strided partial, then a tree over the CTA): reproducible bit for bit.
__global__ void __launch_bounds__(SM_THREADS) frobenius_kernel(const double* __restrict__ X, int ldx, int rows,
                                                                int cols, double* __restrict__ out) {
  __shared__ double part[SM_THREADS];
  const int64_t total = (int64_t)rows * cols;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < total; e += SM_THREADS) {
    const double v = X[(e / rows) * ldx + e % rows];
    s += v * v;
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = SM_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sqrt(part[0]);
}

// out[e] = ((parts[0][e] + parts[1][e]) + parts[2][e]) + ... : the per-rank
// partial sums of a row-sharded Gram added in rank order, so every rank gets
// bitwise the same matrix whatever the collective's internal algorithm, and
// bit-symmetric partials give a bit-symmetric sum (the two mirror elements
// see the same operands in the same order).
__global__ void sum_ranks_kernel(const double* __restrict__ parts, int nparts, int64_t n, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = parts[e];
    for (int r = 1; r < nparts; ++r) s += parts[(int64_t)r * n + e];
    out[e] = s;
  }
}

cudaError_t sum_ranks_launch(const double* parts, int nparts, int64_t n, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)imin64(ceil_div(n, SM_THREADS), 4 * num_sms());
  sum_ranks_kernel<<<blocks, SM_THREADS, 0, s>>>(parts, nparts, n, out);
  return cudaGetLastError();
}

// dst (mapped pinned host memory, seen through its device alias) = src, n
// doubles, written by the SMs as posted PCIe stores: a small result leaves the
// GPU without a copy-engine transfer, so it does not queue behind a large
// cudaMemcpy a caller runs on another stream (the e2e loader's D2H of Q).
// The host reads dst only after synchronizing with the stream (an event), and
// kernel completion makes the mapped stores visible to it; no per-thread
// system fence is needed (one per thread cost ~10 us at 512 KB).
__global__ void store_mapped_kernel(const double* __restrict__ src, int64_t n, double* dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

cudaError_t store_mapped_launch(const double* src, int64_t n, double* dst_dev_alias, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)imin64(ceil_div(n, SM_THREADS), 64);
  store_mapped_kernel<<<blocks, SM_THREADS, 0, s>>>(src, n, dst_dev_alias);
  return cudaGetLastError();
}

cudaError_t tri_inverse_launch(const double* R, int ldr, int n, double* X, int ldx, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  tri_inverse_kernel<<<(int)ceil_div(n, SM_THREADS), SM_THREADS, 0, s>>>(R, ldr, n, X, ldx);
  return cudaGetLastError();
}

cudaError_t tri_multiply_launch(const double* A, int lda, const double* B, int ldb, int n, double* C, int ldc,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int64_t total = (int64_t)n * n;
  const int blocks = (int)imin64(ceil_div(total, SM_THREADS), 1024);
  tri_multiply_kernel<<<blocks, SM_THREADS, 0, s>>>(A, lda, B, ldb, n, C, ldc);
  return cudaGetLastError();
}

cudaError_t frobenius_launch(const double* X, int ldx, int rows, int cols, double* out, cudaStream_t s) {
  frobenius_kernel<<<1, SM_THREADS, 0, s>>>(X, ldx, rows, cols, out);
  return cudaGetLastError();
}

}  // namespace cqr
