// Data-layout kernels for the row-quad interleaved (QI) tall layout and the
// tiled coefficient layout (include/cqr.h), plus the elementwise axpy.
//
//   QI tall array, m rows, ldk column capacity:  (r, c) -> (r/4)*4*ldk + 4c + r%4
//   coefficient tiles (k x n operand C / R^-1):  32 x 64 tiles, tile (kt, nt) at
//       (nt*nkt + kt) * 64*36, element (k, n) at +(n%64)*36 + k%32, zero padded
//
// Every thread moves whole 32-byte quads (one DRAM sector), so the strided
// side of each transpose still moves full sectors.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

// column-major (lds) -> QI (ldk); rows [m, m_pad) are zero-filled
__global__ void pack_tall_kernel(const double* __restrict__ src, int64_t lds, int64_t m, int k,
                                 double* __restrict__ dst, int64_t ldk, int64_t nq) {
  const int64_t total = nq * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e % nq, c = e / nq;
    const double* s = src + c * lds + 4 * q;
    double v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (4 * q + i < m) ? s[i] : 0.0;
    double2* d = reinterpret_cast<double2*>(dst + q * 4 * ldk + 4 * c);
    d[0] = make_double2(v[0], v[1]);
    d[1] = make_double2(v[2], v[3]);
  }
}

// QI (ldk) -> column-major (ldd), rows [0, m)
__global__ void unpack_tall_kernel(const double* __restrict__ src, int64_t ldk, int64_t m, int k,
                                   double* __restrict__ dst, int64_t ldd, int64_t nq) {
  const int64_t total = nq * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e % nq, c = e / nq;
    const double2* s = reinterpret_cast<const double2*>(src + q * 4 * ldk + 4 * c);
    const double2 a = s[0], b = s[1];
    double* d = dst + c * ldd + 4 * q;
    const double v[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * q + i < m) d[i] = v[i];
  }
}

// dst(:, j) = src(:, idx[j]) for j < n (idx == nullptr: idx[j] = j0 + j)
__global__ void gather_cols_kernel(const double* __restrict__ src, int64_t lds, const int* __restrict__ idx, int j0,
                                   double* __restrict__ dst, int64_t ldd, int dcol0, int n, int64_t nq) {
  const int64_t total = nq * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % n, q = e / n;
    const int c = idx ? idx[j] : j0 + (int)j;
    const double2* s = reinterpret_cast<const double2*>(src + q * 4 * lds + 4 * (int64_t)c);
    double2* d = reinterpret_cast<double2*>(dst + q * 4 * ldd + 4 * (dcol0 + j));
    d[0] = s[0];
    d[1] = s[1];
  }
}

// Y(:, 0:n) += alpha X(:, 0:n) with NumPy's two roundings y + (alpha x)
__global__ void axpy_qi_kernel(double* __restrict__ Y, int64_t ldy, double alpha, const double* __restrict__ X,
                               int64_t ldx, int n, int64_t nq) {
  const int64_t total = nq * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % n, q = e / n;
    double2* y = reinterpret_cast<double2*>(Y + q * 4 * ldy + 4 * j);
    const double2* x = reinterpret_cast<const double2*>(X + q * 4 * ldx + 4 * j);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 v = y[h];
      const double2 w = x[h];
      v.x = __dadd_rn(v.x, __dmul_rn(alpha, w.x));
      v.y = __dadd_rn(v.y, __dmul_rn(alpha, w.y));
      y[h] = v;
    }
  }
}

// column-major k x n (ld) -> coefficient tiles (zero padded)
__global__ void pack_coeff_kernel(const double* __restrict__ src, int ld, int k, int n, double* __restrict__ dst) {
  const int nkt = (int)ceil_div(k, CT_K), nnt = (int)ceil_div(n, CT_N);
  const int64_t total = (int64_t)nkt * nnt * CT_TILE;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e / CT_TILE;
    const int w = (int)(e % CT_TILE);
    const int nt = (int)(tile / nkt), kt = (int)(tile % nkt);
    const int nl = w / CT_LD, kl = w % CT_LD;
    const int kk = kt * CT_K + kl, nn = nt * CT_N + nl;
    dst[e] = (kl < CT_K && kk < k && nn < n) ? src[(int64_t)nn * ld + kk] : 0.0;
  }
}

static int grid_for(int64_t total) {
  int64_t b = ceil_div(total, 256);
  if (b > 32 * (int64_t)num_sms()) b = 32 * (int64_t)num_sms();
  return (int)(b < 1 ? 1 : b);
}

cudaError_t pack_tall_launch(const double* src, int64_t lds, int64_t m, int k, double* dst, int64_t ldk,
                             cudaStream_t s) {
  const int64_t nq = round_up(m, 16) / 4;
  if (nq * k == 0) return cudaSuccess;
  pack_tall_kernel<<<grid_for(nq * k), 256, 0, s>>>(src, lds, m, k, dst, ldk, nq);
  return cudaGetLastError();
}

cudaError_t unpack_tall_launch(const double* src, int64_t ldk, int64_t m, int k, double* dst, int64_t ldd,
                               cudaStream_t s) {
  const int64_t nq = ceil_div(m, 4);
  if (nq * k == 0) return cudaSuccess;
  unpack_tall_kernel<<<grid_for(nq * k), 256, 0, s>>>(src, ldk, m, k, dst, ldd, nq);
  return cudaGetLastError();
}

cudaError_t gather_cols_launch(const double* src, int64_t lds, const int* idx, int j0, double* dst, int64_t ldd,
                               int dcol0, int n, int64_t m, cudaStream_t s) {
  const int64_t nq = round_up(m, 16) / 4;
  if (nq * n == 0) return cudaSuccess;
  gather_cols_kernel<<<grid_for(nq * n), 256, 0, s>>>(src, lds, idx, j0, dst, ldd, dcol0, n, nq);
  return cudaGetLastError();
}

cudaError_t axpy_launch(double* Y, int64_t ldy, double alpha, const double* X, int64_t ldx, int64_t m, int n,
                        cudaStream_t s) {
  const int64_t nq = round_up(m, 16) / 4;
  if (nq * n == 0) return cudaSuccess;
  axpy_qi_kernel<<<grid_for(nq * n), 256, 0, s>>>(Y, ldy, alpha, X, ldx, n, nq);
  return cudaGetLastError();
}

cudaError_t pack_coeff_launch(const double* src, int ld, int k, int n, double* dst, cudaStream_t s) {
  const int64_t total = coeff_tiles_doubles(k, n);
  if (total == 0) return cudaSuccess;
  pack_coeff_kernel<<<grid_for(total), 256, 0, s>>>(src, ld, k, n, dst);
  return cudaGetLastError();
}

}  // namespace cqr
