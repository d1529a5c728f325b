// K2 building block: row-panel GEMM Y = X C on QI tall arrays (TRMM when
// C = R^-1 is upper triangular).
//
// Replaces `DenseVectorArray.lincomb` (reference varray.py:157-163: X @ C plus
// a Fortran re-layout copy).  CTA tile = 64 rows x 64 output columns, four
// consumer warps in a 2x2 grid of 32-row x (4 interleaved 8-column blocks)
// register tiles, one producer warp.
// The K dimension is streamed in chunks of 32 columns: per chunk one stage
// holds X[64 rows, 32 cols] (16 bulk copies of one 1 KB quad run each) and
// the 32 x 64 coefficient tile (one 18 KB bulk copy of the pre-tiled C,
// columns padded to 36 doubles).  Both fragment loads are bank-conflict free:
// A at quad offset 4*col + row%4, B at 36*col + k.  For a triangular C the K
// chunks and 8x8 blocks that only meet zeros are skipped (a TRMM costs
// m k (k+1) flops), and column tiles j and T-1-j share a CTA so every CTA
// gets the same work.  CTAs are persistent over row tiles in one wave of two
// CTAs per SM.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int GM_BR = 64;                 // rows per tile (16 quads)
constexpr int GM_KC = CT_K;               // K chunk (32)
constexpr int GM_BN = CT_N;               // output columns per tile (64)
constexpr int GM_XS = (GM_BR / 4) * GM_KC * 4;   // 2048 doubles
constexpr int GM_STAGES = 3;
constexpr int GM_STAGE_DOUBLES = GM_XS + CT_TILE;
constexpr int GM_THREADS = 160;

static size_t gemm_smem_bytes() { return GM_STAGES * GM_STAGE_DOUBLES * sizeof(double) + 2 * GM_STAGES * 8 + 64; }

__device__ __forceinline__ int group_tiles(int grp, int T, int upper, int (&tiles)[2]) {
  tiles[0] = grp;
  if (upper && T - 1 - grp != grp) { tiles[1] = T - 1 - grp; return 2; }
  return 1;
}

// 8-column block j (0..3) of warp column wj: wj = 0 owns blocks {0,3,4,7},
// wj = 1 owns {1,2,5,6}.  On the diagonal 64x64 block of a triangular C,
// block b needs b+1 k-octets, so both sets cost 18 -- the two warp columns
// (and the SM sub-partitions they run on) get equal DMMA work.
__device__ __forceinline__ int col_block(int j, int wj) { return 2 * j + (wj ^ (j & 1)); }

// Diagonal chunk CH (0/1) of a 64-column tile of an upper-triangular C for
// warp column WJ: every block/step condition is a compile-time constant, so
// no DMMA is issued for a zero block (predicated-off DMMAs still occupy the
// tensor pipe).  Block b is live at k4 step ks iff 4 CH + ks/2 <= b.
template <int WJ, int CH>
__device__ __forceinline__ void diag_chunk(double (&acc)[4][4][2], const double* xp, const double* cp) {
  constexpr int bmax = WJ == 0 ? 7 : 6;
#pragma unroll
  for (int ks = 0; ks < GM_KC / 4; ++ks) {
    if (4 * CH + ks / 2 > bmax) break;
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = xp[2 * i * (GM_KC * 4) + 16 * ks];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cb = 2 * j + (WJ ^ (j & 1));
      if (4 * CH + ks / 2 <= cb) b[j] = cp[8 * cb * CT_LD + 4 * ks];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cb = 2 * j + (WJ ^ (j & 1));
      if (4 * CH + ks / 2 > cb) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(acc[i][j], a[i], b[j]);
    }
  }
}

// JL = live 8-column blocks per warp column: 4 for tiles wider than 32 output
// columns, 2 for 17..32 (blocks 0..3 of the tile: j < 2 of both warp columns),
// 1 for <= 16 -- a skinny general C (the projection Q_in Bt of the update path)
// does not issue DMMAs for zero column blocks.  SUB: Y = Yin - X C (the
// projection and its subtraction, algorithms.py:442-444, in one pass; the same
// two roundings as lincomb + axpy).  The TRMM / full-width instance is <4, false>.
template <int JL, bool SUB>
__global__ void __launch_bounds__(GM_THREADS, 2) gemm_kernel(GemmArgs args) {
  if (args.gate != nullptr && *args.gate != 0) return;   // gated off
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GM_STAGES * GM_STAGE_DOUBLES);
  uint64_t* empty = full + GM_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tiles[2];
  const int ntl = group_tiles(blockIdx.x, args.ntile_n, args.upper, tiles);
  const int nkt = (int)ceil_div(args.kx, GM_KC);

  if (threadIdx.x == 0) {
    for (int s = 0; s < GM_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    int it = 0;
    for (int64_t rt = blockIdx.y; rt < args.nrow_tiles; rt += gridDim.y) {
      const int64_t r0 = rt * GM_BR;
      const int nq = (int)imin64(GM_BR, args.rows - r0) >> 2;
      for (int tl = 0; tl < ntl; ++tl) {
        const int nt = tiles[tl];
        const int kend = args.upper ? min(args.kx, (nt + 1) * GM_BN) : args.kx;
        const int nchunks = (int)ceil_div(kend, GM_KC);
        for (int ch = 0; ch < nchunks; ++ch, ++it) {
          const int s = it % GM_STAGES;
          const uint32_t use = it / GM_STAGES;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
          const int kc = ch * GM_KC;
          const int nxc = min(GM_KC, args.kx - kc);
          double* Xs = smem + s * GM_STAGE_DOUBLES;
          double* Cs = Xs + GM_XS;
          if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)nq * nxc * 32 + CT_TILE * 8);
          __syncwarp();
          const double* xb = args.X + (r0 >> 2) * 4 * args.ldx + 4 * (int64_t)kc;
          for (int q = lane; q < nq; q += 32)
            bulk_g2s_stream(Xs + q * (GM_KC * 4), xb + q * 4 * args.ldx, (uint32_t)nxc * 32, &full[s]);
          if (lane == 0)
            bulk_g2s(Cs, args.C + ((int64_t)nt * nkt + ch) * CT_TILE, CT_TILE * 8, &full[s]);
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
        // A fragment (row 32wi+8i+g, col kc+4ks+t): quad 8wi+2i+g/4, offset 4(4ks+t) + g%4
        const double* xp = Xs + (8 * wi + (g >> 2)) * (GM_KC * 4) + 4 * t + (g & 3);
        const double* cp = Cs + g * CT_LD + t;
        const bool tail = kc + GM_KC > args.kx;   // X columns past kx hold stale data
        const int colmax = n0 + 63 - 8 * wj;      // last output column of this warp
        if (!tail && (!args.upper || kc + GM_KC <= n0)) {
          // full chunk (no zero blocks, no stale columns): fully unrolled,
          // next k4 step's fragments loaded while this step's DMMAs issue
          double a[2][4], b[2][4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[0][i] = xp[2 * i * (GM_KC * 4)];
#pragma unroll
          for (int j = 0; j < JL; ++j) b[0][j] = cp[8 * col_block(j, wj) * CT_LD];
#pragma unroll
          for (int ks = 0; ks < GM_KC / 4; ++ks) {
            const int cur = ks & 1;
            if (ks + 1 < GM_KC / 4) {
#pragma unroll
              for (int i = 0; i < 4; ++i) a[cur ^ 1][i] = xp[2 * i * (GM_KC * 4) + 16 * (ks + 1)];
#pragma unroll
              for (int j = 0; j < JL; ++j) b[cur ^ 1][j] = cp[8 * col_block(j, wj) * CT_LD + 4 * (ks + 1)];
            }
#pragma unroll
            for (int j = 0; j < JL; ++j)
#pragma unroll
              for (int i = 0; i < 4; ++i) dmma(acc[i][j], a[cur][i], b[cur][j]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
          continue;
        }
        if (args.upper && !tail && kc >= n0) {
          const int ch = (kc - n0) >> 5;   // 0 or 1
          if (wj == 0) { if (ch == 0) diag_chunk<0, 0>(acc, xp, cp); else diag_chunk<0, 1>(acc, xp, cp); }
          else         { if (ch == 0) diag_chunk<1, 0>(acc, xp, cp); else diag_chunk<1, 1>(acc, xp, cp); }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
          continue;
        }
#pragma unroll 2
        for (int ks = 0; ks < GM_KC / 4; ++ks) {
          const int k4 = kc + 4 * ks;
          if (args.upper && k4 > colmax) break;   // rest of the chunk multiplies zeros
          if (k4 >= args.kx) break;
          double a[4], b[4];
          const bool kval = !tail || (k4 + t < args.kx);
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = kval ? xp[2 * i * (GM_KC * 4) + 16 * ks] : 0.0;
#pragma unroll
          for (int j = 0; j < JL; ++j) b[j] = cp[8 * col_block(j, wj) * CT_LD + 4 * ks];
#pragma unroll
          for (int j = 0; j < JL; ++j) {
            if (args.upper && k4 > n0 + 8 * col_block(j, wj) + 7) continue;  // block of zeros
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(acc[i][j], a[i], b[j]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // ---- store this tile (rows < nrows, cols < n) in the QI layout
      if constexpr (SUB) {
        // Y = Yin - X C: all of the lane's Yin values are requested before the
        // first store (the stores are volatile asm: interleaved, every load's
        // latency would be exposed)
        double yv[4][JL][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = 32 * wi + 8 * i + g;
          const double* yi = args.Yin + ((r0 + row) >> 2) * 4 * args.ldyin + (row & 3);
#pragma unroll
          for (int j = 0; j < JL; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = n0 + 8 * col_block(j, wj) + 2 * t + e;
              yv[i][j][e] = (row < nrows && col < args.n) ? yi[4 * (int64_t)col] : 0.0;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < JL; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[i][j][e] = __dsub_rn(yv[i][j][e], acc[i][j][e]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 32 * wi + 8 * i + g;
        if (row >= nrows) continue;
        double* yq = args.Y + ((r0 + row) >> 2) * 4 * args.ldy + (row & 3);
#pragma unroll
        for (int j = 0; j < JL; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = n0 + 8 * col_block(j, wj) + 2 * t + e;
            if (col < args.n) st_stream(yq + 4 * (int64_t)col, acc[i][j][e]);
          }
      }
    }
  }
}

template <int JL, bool SUB>
static cudaError_t gemm_launch_t(const GemmArgs& a, dim3 grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = smem_attr((const void*)gemm_kernel<JL, SUB>, smem);
  if (e != cudaSuccess) return e;
  gemm_kernel<JL, SUB><<<grid, GM_THREADS, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t gemm_launch(GemmArgs& a, cudaStream_t stream) {
  const size_t smem = gemm_smem_bytes();
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
  // skinny general C: only the live column blocks (the triangular path keeps
  // its compile-time block skips over the full tile)
  const int jl = (a.upper || a.n > 32) ? 4 : (a.n > 16 ? 2 : 1);
  if (a.Yin != nullptr) {
    if (a.upper) return cudaErrorInvalidValue;
    if (jl == 4) return gemm_launch_t<4, true>(a, grid, smem, stream);
    if (jl == 2) return gemm_launch_t<2, true>(a, grid, smem, stream);
    return gemm_launch_t<1, true>(a, grid, smem, stream);
  }
  if (jl == 4) return gemm_launch_t<4, false>(a, grid, smem, stream);
  if (jl == 2) return gemm_launch_t<2, false>(a, grid, smem, stream);
  return gemm_launch_t<1, false>(a, grid, smem, stream);
}

}  // namespace cqr
