// K2 building blocks: row-panel GEMM Y = X C (TRMM when C = R^-1 is upper
// triangular) and the in-place axpy.
//
// Replaces `DenseVectorArray.lincomb` (reference varray.py:157-163: X @ C plus
// a Fortran re-layout copy) and `DenseVectorArray.axpy` (varray.py:165-171).
//
// GEMM layout: CTA tile = 64 rows x 64 output columns, 4 consumer warps in a
// 2x2 grid of 32x32 register tiles, 1 producer warp.  The K dimension (columns
// of X) is streamed in chunks of 32: per chunk one stage holds X[64 rows, 32
// cols] (bulk copy per column, row stride 68 doubles) and C[32, 64 cols]
// (bulk copy per column, stride 36) -- both strides are 4 (mod 16) doubles so
// every DMMA fragment load is bank-conflict free.  CTAs are persistent over
// row tiles (grid.y) so the pipeline runs across tiles.  For upper-triangular
// C the K chunks and 8x8 blocks that only meet zeros are skipped, so a TRMM
// costs m k (k+1) flops instead of 2 m k^2.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int GM_BR = 64;            // rows per tile
constexpr int GM_KC = 32;            // K chunk
constexpr int GM_BN = 64;            // output columns per tile
constexpr int GM_LDX = GM_BR + 4;    // 68
constexpr int GM_LDC = GM_KC + 4;    // 36
constexpr int GM_STAGES = 3;
constexpr int GM_XS = GM_KC * GM_LDX;
constexpr int GM_CS = GM_BN * GM_LDC;
constexpr int GM_STAGE_DOUBLES = GM_XS + GM_CS;
constexpr int GM_THREADS = 160;

static size_t gemm_smem_bytes() { return GM_STAGES * GM_STAGE_DOUBLES * sizeof(double) + 2 * GM_STAGES * 8 + 64; }

// Column groups: for a triangular C the work of column tile j grows with j,
// so tiles j and T-1-j share a CTA (equal work per CTA); otherwise one tile
// per group.  CTAs are persistent over row tiles and run their group's
// column tiles back to back on each row tile (the second pass over the X
// row tile hits L2).
__device__ __forceinline__ int group_tiles(int grp, int T, int upper, int (&tiles)[2]) {
  if (!upper) { tiles[0] = grp; return 1; }
  tiles[0] = grp;
  if (T - 1 - grp != grp) { tiles[1] = T - 1 - grp; return 2; }
  return 1;
}

__global__ void __launch_bounds__(GM_THREADS, 2) gemm_kernel(GemmArgs args) {
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GM_STAGES * GM_STAGE_DOUBLES);
  uint64_t* empty = full + GM_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tiles[2];
  const int ntl = group_tiles(blockIdx.x, args.ntile_n, args.upper, tiles);

  if (threadIdx.x == 0) {
    for (int s = 0; s < GM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    int it = 0;
    for (int64_t rt = blockIdx.y; rt < args.nrow_tiles; rt += gridDim.y) {
      const int64_t r0 = rt * GM_BR;
      const int nrows = (int)imin64(GM_BR, args.rows - r0);
      const uint32_t xbytes = nrows * 8;
      for (int tl = 0; tl < ntl; ++tl) {
        const int n0 = tiles[tl] * GM_BN;
        const int ncols = min(GM_BN, args.n - n0);
        const int kend = args.upper ? min(args.kx, n0 + GM_BN) : args.kx;
        const int nchunks = (int)ceil_div(kend, GM_KC);
        for (int ch = 0; ch < nchunks; ++ch, ++it) {
          const int s = it % GM_STAGES;
          const uint32_t use = it / GM_STAGES;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
          const int kc = ch * GM_KC;
          const int nxc = min(GM_KC, args.kx - kc);
          double* Xs = smem + s * GM_STAGE_DOUBLES;
          double* Cs = Xs + GM_XS;
          if (lane == 0) mbar_arrive_expect_tx(&full[s], nxc * xbytes + ncols * (GM_KC * 8));
          __syncwarp();
          for (int c = lane; c < nxc; c += 32)
            bulk_g2s(Xs + c * GM_LDX, args.X + (int64_t)(kc + c) * args.ldx + r0, xbytes, &full[s]);
          for (int c = lane; c < ncols; c += 32)
            bulk_g2s(Cs + c * GM_LDC, args.C + (int64_t)(n0 + c) * args.ldc + kc, GM_KC * 8, &full[s]);
        }
      }
    }
    return;
  }

  const int wi = warp >> 1, wj = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
  int it = 0;
  for (int64_t rt = blockIdx.y; rt < args.nrow_tiles; rt += gridDim.y) {
    const int64_t r0 = rt * GM_BR;
    const int nrows = (int)imin64(GM_BR, args.rows - r0);
    for (int tl = 0; tl < ntl; ++tl) {
      const int n0 = tiles[tl] * GM_BN;
      const int kend = args.upper ? min(args.kx, n0 + GM_BN) : args.kx;
      const int nchunks = (int)ceil_div(kend, GM_KC);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
      for (int ch = 0; ch < nchunks; ++ch, ++it) {
        const int s = it % GM_STAGES;
        mbar_wait(&full[s], (it / GM_STAGES) & 1);
        const int kc = ch * GM_KC;
        const double* Xs = smem + s * GM_STAGE_DOUBLES;
        const double* Cs = Xs + GM_XS;
        const double* xp = Xs + t * GM_LDX + 32 * wi + g;
        const double* cp = Cs + (32 * wj + g) * GM_LDC + t;
        const bool tail = kc + GM_KC > args.kx;   // X columns past kx hold stale data
        const int colmax = n0 + 32 * wj + 31;     // last output column of this warp
#pragma unroll 2
        for (int ks = 0; ks < GM_KC / 4; ++ks) {
          const int k4 = kc + 4 * ks;
          if (args.upper && k4 > colmax) break;   // rest of the chunk multiplies zeros
          if (k4 >= args.kx) break;
          double a[4], b[4];
          const bool kval = !tail || (k4 + t < args.kx);
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = kval ? xp[4 * ks * GM_LDX + 8 * i] : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = cp[8 * j * GM_LDC + 4 * ks];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (args.upper && k4 > n0 + 32 * wj + 8 * j + 7) continue;  // block of zeros
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(acc[i][j], a[i], b[j]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // ---- store this tile (rows < rows, cols < n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 32 * wi + 8 * i + g;
        if (row >= nrows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = n0 + 32 * wj + 8 * j + 2 * t + e;
            if (col < args.n) args.Y[(int64_t)col * args.ldy + r0 + row] = acc[i][j][e];
          }
      }
    }
  }
}

cudaError_t gemm_launch(GemmArgs& a, cudaStream_t stream) {
  static bool attr_set = false;
  const size_t smem = gemm_smem_bytes();
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  a.ntile_n = (int)ceil_div(a.n, GM_BN);
  a.nrow_tiles = ceil_div(a.rows, GM_BR);
  if (a.nrow_tiles == 0 || a.n == 0) return cudaSuccess;
  const int ngroups = a.upper ? (a.ntile_n + 1) / 2 : a.ntile_n;
  // one full wave of 2 CTAs per SM
  int64_t gy = (2 * (int64_t)num_sms()) / ngroups;
  if (gy < 1) gy = 1;
  if (gy > a.nrow_tiles) gy = a.nrow_tiles;
  if (gy > 65535) gy = 65535;
  dim3 grid(ngroups, (unsigned)gy);
  gemm_kernel<<<grid, GM_THREADS, smem, stream>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ axpy
__global__ void axpy_kernel(double* __restrict__ Y, int64_t ldy, double alpha, const double* __restrict__ X,
                            int64_t ldx, int64_t rows2, int n) {
  const int64_t total = rows2 * n;  // in double2 units
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows2, r = e % rows2;
    double2* y = reinterpret_cast<double2*>(Y + j * ldy) + r;
    const double2 x = reinterpret_cast<const double2*>(X + j * ldx)[r];
    double2 v = *y;
    // y + (alpha x) with two roundings, as NumPy's `data += alpha * other`
    v.x = __dadd_rn(v.x, __dmul_rn(alpha, x.x));
    v.y = __dadd_rn(v.y, __dmul_rn(alpha, x.y));
    *y = v;
  }
}

cudaError_t axpy_launch(double* Y, int64_t ldy, double alpha, const double* X, int64_t ldx, int64_t rows, int n,
                        cudaStream_t stream) {
  const int64_t rows2 = rows / 2;
  const int64_t total = rows2 * n;
  if (total == 0) return cudaSuccess;
  int blocks = (int)imin64(ceil_div(total, 256), 16 * num_sms());
  axpy_kernel<<<blocks, 256, 0, stream>>>(Y, ldy, alpha, X, ldx, rows2, n);
  return cudaGetLastError();
}

}  // namespace cqr
