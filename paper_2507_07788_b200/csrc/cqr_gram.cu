// K1: tall-skinny Gram kernels, G = A^T B over the local row shard.
//
// Replaces `DenseVectorArray.gramian` (reference varray.py:150-155): the self
// Gram X^T X (bit-symmetric by construction: only the lower triangle is
// computed and mirrored) and the cross Gram Q_in^T Q of the update path.
//
// Layout: A, B column-major fp64 (column j at A + j*lda), `rows` = m padded to
// 16 with zero rows.  The k x k output is cut into 64x64 CTA tiles (self: the
// lower-triangular tiles only); the rows are cut into `nsplit` contiguous
// ranges.  Grid = (tile, split): CTAs of one split run side by side and share
// the row panels through L2.  Each CTA streams 32-row panels of its column
// blocks into padded shared memory with cp.async.bulk (one bulk copy per
// column, row stride 36 doubles so the DMMA fragment loads are bank-conflict
// free), a 3-stage full/empty mbarrier ring fed by one producer warp, and 4
// consumer warps each own a 32x32 sub-tile held in registers (16 DMMA.8x8x4
// per 8 LDS.64).  On diagonal tiles blocks above the diagonal are skipped.
// Per-(split, tile) partials go to a workspace; `reduce` sums them in a fixed
// split order (deterministic, bitwise run-to-run) and writes G (+ mirror).
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int GR_BR = 32;           // rows per panel stage
constexpr int GR_LDP = GR_BR + 4;   // 36 == 4 (mod 16): conflict-free fragments
constexpr int GR_CT = 64;           // CTA tile edge
constexpr int GR_STAGES = 3;
constexpr int GR_STAGE_DOUBLES = 2 * GR_CT * GR_LDP;
constexpr int GR_THREADS = 160;     // 4 consumer warps + 1 producer warp

size_t gram_smem_bytes() { return GR_STAGES * GR_STAGE_DOUBLES * sizeof(double) + 2 * GR_STAGES * 8 + 64; }

__device__ __forceinline__ void tile_coords(int tile, bool self, int ntj, int& ti, int& tj) {
  if (self) {
    int t = tile, r = 0;
    while (t > r) { t -= r + 1; ++r; }
    ti = r; tj = t;
  } else {
    ti = tile / ntj; tj = tile % ntj;
  }
}

__global__ void __launch_bounds__(GR_THREADS) gram_kernel(GramArgs args) {
  extern __shared__ __align__(128) double smem[];
  double* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GR_STAGES * GR_STAGE_DOUBLES);
  uint64_t* empty = full + GR_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  int ti, tj;
  tile_coords(tile, args.self, args.ntile_j, ti, tj);
  const bool diag = args.self && ti == tj;
  const int ia0 = ti * GR_CT, jb0 = tj * GR_CT;
  const int ncolA = min(GR_CT, args.ka - ia0);
  const int ncolB = diag ? 0 : min(GR_CT, args.kb - jb0);

  const int64_t npan = args.npanels;
  const int64_t p_begin = npan * split / args.nsplit;
  const int64_t p_end = npan * (split + 1) / args.nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GR_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---------------- producer warp: bulk copies of the row panels
    int it = 0;
    for (int64_t p = p_begin; p < p_end; ++p, ++it) {
      const int s = it % GR_STAGES;
      const uint32_t use = it / GR_STAGES;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      const int64_t r0 = p * GR_BR;
      const int nrows = (int)imin64(GR_BR, args.rows - r0);
      const uint32_t bytes = nrows * 8;
      double* As = stage_base + s * GR_STAGE_DOUBLES;
      double* Bs = As + GR_CT * GR_LDP;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (ncolA + ncolB) * bytes);
      __syncwarp();
      for (int c = lane; c < ncolA; c += 32)
        bulk_g2s(As + c * GR_LDP, args.A + (int64_t)(ia0 + c) * args.lda + r0, bytes, &full[s]);
      for (int c = lane; c < ncolB; c += 32)
        bulk_g2s(Bs + c * GR_LDP, args.B + (int64_t)(jb0 + c) * args.ldb + r0, bytes, &full[s]);
    }
    return;
  }

  // ---------------- consumer warps
  const int wi = warp >> 1, wj = warp & 1;
  const bool idle = diag && wi < wj;            // sub-tile wholly above the diagonal
  const bool wdiag = diag && wi == wj;          // sub-tile on the diagonal
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }

  int it = 0;
  for (int64_t p = p_begin; p < p_end; ++p, ++it) {
    const int s = it % GR_STAGES;
    mbar_wait(&full[s], (it / GR_STAGES) & 1);
    const int64_t r0 = p * GR_BR;
    const int nk4 = (int)imin64(GR_BR, args.rows - r0) >> 2;
    const double* As = stage_base + s * GR_STAGE_DOUBLES;
    const double* Bs = diag ? As : As + GR_CT * GR_LDP;
    if (!idle) {
      const double* ap = As + (32 * wi + g) * GR_LDP + t;
      const double* bp = Bs + (32 * wj + g) * GR_LDP + t;
      if (wdiag) {
        for (int ks = 0; ks < nk4; ++ks) {
          double a[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = ap[8 * i * GR_LDP + 4 * ks];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) dmma(acc[i][j], a[i], a[j]);
        }
      } else {
        for (int ks = 0; ks < nk4; ++ks) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = ap[8 * i * GR_LDP + 4 * ks];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = bp[8 * j * GR_LDP + 4 * ks];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- partial tile -> workspace (tile-local column-major 64x64)
  double* out = args.ws + ((int64_t)split * args.ntiles + tile) * (GR_CT * GR_CT);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 32 * wi + 8 * i + g, col = 32 * wj + 8 * j + 2 * t + e;
        out[col * GR_CT + row] = acc[i][j][e];
      }
}

// Fixed-order sum of the split partials.  One thread per output element of
// the (lower) tile set; writes G and, for the self Gram, its mirror.
__global__ void gram_reduce_kernel(GramArgs args, double* G, int ldg) {
  const int64_t n_el = (int64_t)args.ka * args.kb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    const int gi = (int)(e % args.ka), gj = (int)(e / args.ka);
    if (args.self && gi < gj) continue;
    const int ti = gi / GR_CT, tj = gj / GR_CT;
    const int tile = args.self ? (ti * (ti + 1) / 2 + tj) : (ti * args.ntile_j + tj);
    const double* p = args.ws + (int64_t)tile * (GR_CT * GR_CT) + (gj % GR_CT) * GR_CT + (gi % GR_CT);
    const int64_t stride = (int64_t)args.ntiles * GR_CT * GR_CT;
    double s = 0.0;
    for (int sp = 0; sp < args.nsplit; ++sp) s += p[sp * stride];
    G[(int64_t)gj * ldg + gi] = s;
    if (args.self) G[(int64_t)gi * ldg + gj] = s;
  }
}

static int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

GramArgs gram_plan(const double* A, int64_t lda, int ka, const double* B, int64_t ldb, int kb, int64_t rows,
                   bool self) {
  GramArgs a{};
  a.A = A; a.lda = lda; a.ka = ka;
  a.B = self ? A : B; a.ldb = self ? lda : ldb; a.kb = self ? ka : kb;
  a.rows = rows;
  a.self = self ? 1 : 0;
  a.ntile_i = (int)ceil_div(ka, GR_CT);
  a.ntile_j = (int)ceil_div(a.kb, GR_CT);
  a.ntiles = self ? a.ntile_i * (a.ntile_i + 1) / 2 : a.ntile_i * a.ntile_j;
  a.npanels = ceil_div(rows, GR_BR);
  const int64_t target = 2 * (int64_t)num_sms();  // 2 CTAs per SM
  int64_t ns = ceil_div(target, a.ntiles);
  if (ns > a.npanels) ns = a.npanels;
  if (ns < 1) ns = 1;
  a.nsplit = (int)ns;
  return a;
}

size_t gram_workspace_bytes(const GramArgs& a) {
  return (size_t)a.nsplit * a.ntiles * GR_CT * GR_CT * sizeof(double);
}

cudaError_t gram_launch(GramArgs& a, double* G, int ldg, cudaStream_t stream) {
  static bool attr_set = false;
  const size_t smem = gram_smem_bytes();
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (a.rows > 0) {
    dim3 grid(a.ntiles, a.nsplit);
    gram_kernel<<<grid, GR_THREADS, smem, stream>>>(a);
  } else {
    a.nsplit = 0;
  }
  const int64_t n_el = (int64_t)a.ka * a.kb;
  int blocks = (int)imin64(ceil_div(n_el, 256), 4 * num_sms());
  if (blocks < 1) blocks = 1;
  gram_reduce_kernel<<<blocks, 256, 0, stream>>>(a, G, ldg);
  return cudaGetLastError();
}

}  // namespace cqr
