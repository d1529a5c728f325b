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

// Work items.  Non-self: one item per 64x64 tile.  Self (lower triangle of
// T x T tiles): items 0 .. T/2-1 pair diagonal tiles (p, T-1-p) -- two
// half-full tiles make one full CTA load -- item T/2 is the middle diagonal
// tile when T is odd, then the off-diagonal tiles (ti > tj) in row order.
// Every item reads two 64-column blocks (or one) and stores two 64x64 slots.
__host__ __device__ __forceinline__ int self_items(int T) { return (T + 1) / 2 + T * (T - 1) / 2; }

// item -> (column block of operand A, of operand B, kind); kind 0 = off, 1 = diag pair, 2 = single diag
__device__ __forceinline__ void item_blocks(int item, bool self, int T, int ntj, int& ba, int& bb, int& kind) {
  if (!self) { ba = item / ntj; bb = item % ntj; kind = 0; return; }
  const int nd = (T + 1) / 2;
  if (item < T / 2) { ba = item; bb = T - 1 - item; kind = 1; return; }
  if (item < nd) { ba = bb = item; kind = 2; return; }
  int t = item - nd, r = 1;
  while (t >= r) { t -= r; ++r; }
  ba = r; bb = t; kind = 0;
}

// tile (ti, tj) -> (item, slot) of the partial storage
__device__ __forceinline__ void tile_item(int ti, int tj, bool self, int T, int ntj, int& item, int& slot) {
  if (!self) { item = ti * ntj + tj; slot = 0; return; }
  if (ti == tj) {
    if (2 * ti + 1 == T) { item = ti; slot = 0; return; }      // middle single
    if (ti < T / 2) { item = ti; slot = 0; } else { item = T - 1 - ti; slot = 1; }
    return;
  }
  item = (T + 1) / 2 + ti * (ti - 1) / 2 + tj;
  slot = 0;
}

// 8 k4-steps of one 32x32 register sub-tile; DIAG skips blocks above the diagonal
template <bool DIAG>
__device__ __forceinline__ void subtile(double (&acc)[4][4][2], const double* ap, const double* bp, int ks0,
                                        int ks1, int kstep) {
  for (int ks = ks0; ks < ks1; ks += kstep) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = ap[8 * i * GR_LDP + 4 * ks];
    if (DIAG) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) dmma(acc[i][j], a[i], a[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bp[8 * j * GR_LDP + 4 * ks];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
}

__device__ __forceinline__ void store_acc(const double (&acc)[4][4][2], double* out, int r0, int c0, int g, int t) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) out[(c0 + 8 * j + 2 * t + e) * GR_CT + r0 + 8 * i + g] = acc[i][j][e];
}

__global__ void __launch_bounds__(GR_THREADS, 2) gram_kernel(GramArgs args) {
  extern __shared__ __align__(128) double smem[];
  double* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GR_STAGES * GR_STAGE_DOUBLES);
  uint64_t* empty = full + GR_STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x, split = blockIdx.y;
  const bool self = args.self != 0;
  int ba, bb, kind;
  item_blocks(item, self, args.ntile_i, args.ntile_j, ba, bb, kind);
  const int ia0 = ba * GR_CT, jb0 = bb * GR_CT;
  const int ncolA = min(GR_CT, args.ka - ia0);
  const int ncolB = (kind == 2) ? 0 : min(GR_CT, args.kb - jb0);

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

  // ---------------- consumer warps.  Roles (sub-tile = 32x32 of a 64x64 tile):
  //  off tile   : warp w -> sub-tile (w>>1, w&1) of tile (A, B)
  //  diag pair  : w0 -> A(0,0)+A(1,1), w1 -> A(1,0), w2 -> B(0,0)+B(1,1), w3 -> B(1,0)
  //  single diag: w0 -> (0,0), w2 -> (1,1), w1 / w3 -> (1,0) on even / odd k4 steps
  const int g = lane >> 2, t = lane & 3;
  double acc0[4][4][2], acc1[4][4][2];
  zero_acc(acc0);
  zero_acc(acc1);

  int it = 0;
  for (int64_t p = p_begin; p < p_end; ++p, ++it) {
    const int s = it % GR_STAGES;
    mbar_wait(&full[s], (it / GR_STAGES) & 1);
    const int64_t r0 = p * GR_BR;
    const int nk4 = (int)imin64(GR_BR, args.rows - r0) >> 2;
    const double* As = stage_base + s * GR_STAGE_DOUBLES;
    const double* Bs = As + GR_CT * GR_LDP;
    if (kind == 0) {
      const int wi = warp >> 1, wj = warp & 1;
      subtile<false>(acc0, As + (32 * wi + g) * GR_LDP + t, Bs + (32 * wj + g) * GR_LDP + t, 0, nk4, 1);
    } else if (kind == 1) {
      const double* T = (warp < 2) ? As : Bs;
      if ((warp & 1) == 0) {
        subtile<true>(acc0, T + g * GR_LDP + t, nullptr, 0, nk4, 1);
        subtile<true>(acc1, T + (32 + g) * GR_LDP + t, nullptr, 0, nk4, 1);
      } else {
        subtile<false>(acc0, T + (32 + g) * GR_LDP + t, T + g * GR_LDP + t, 0, nk4, 1);
      }
    } else {
      if (warp == 0) subtile<true>(acc0, As + g * GR_LDP + t, nullptr, 0, nk4, 1);
      else if (warp == 2) subtile<true>(acc0, As + (32 + g) * GR_LDP + t, nullptr, 0, nk4, 1);
      else subtile<false>(acc0, As + (32 + g) * GR_LDP + t, As + g * GR_LDP + t, warp == 1 ? 0 : 1, nk4, 2);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- partials -> workspace: item slots of 64x64 (tile-local column-major)
  double* out = args.ws + ((int64_t)split * args.nitems + item) * (2 * GR_CT * GR_CT);
  if (kind == 0) {
    store_acc(acc0, out, 32 * (warp >> 1), 32 * (warp & 1), g, t);
  } else if (kind == 1) {
    double* o = out + ((warp < 2) ? 0 : GR_CT * GR_CT);
    if ((warp & 1) == 0) {
      store_acc(acc0, o, 0, 0, g, t);
      store_acc(acc1, o, 32, 32, g, t);
    } else {
      store_acc(acc0, o, 32, 0, g, t);
    }
  } else {
    // (1,0) is split over warps 1 and 3: warp 3 parks its half in the second slot,
    // warp 1 adds it after the barrier (fixed order: deterministic)
    if (warp == 0) store_acc(acc0, out, 0, 0, g, t);
    if (warp == 2) store_acc(acc0, out, 32, 32, g, t);
    if (warp == 3) store_acc(acc0, out + GR_CT * GR_CT, 32, 0, g, t);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 1) {
      const double* o3 = out + GR_CT * GR_CT;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int idx = (8 * j + 2 * t + e) * GR_CT + 32 + 8 * i + g;
            out[idx] = acc0[i][j][e] + o3[idx];
          }
    }
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
    int item, slot;
    tile_item(ti, tj, args.self != 0, args.ntile_i, args.ntile_j, item, slot);
    const double* p = args.ws + ((int64_t)item * 2 + slot) * (GR_CT * GR_CT) + (gj % GR_CT) * GR_CT + (gi % GR_CT);
    const int64_t stride = (int64_t)args.nitems * 2 * GR_CT * GR_CT;
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
  a.nitems = self ? self_items(a.ntile_i) : a.ntiles;
  a.npanels = ceil_div(rows, GR_BR);
  // one full wave: 2 resident CTAs per SM, nsplit * nitems <= 2 * SMs
  const int64_t target = 2 * (int64_t)num_sms();
  int64_t ns = target / a.nitems;
  if (ns > a.npanels) ns = a.npanels;
  if (ns < 1) ns = 1;
  a.nsplit = (int)ns;
  return a;
}

size_t gram_workspace_bytes(const GramArgs& a) {
  return (size_t)a.nsplit * a.nitems * 2 * GR_CT * GR_CT * sizeof(double);
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
    dim3 grid(a.nitems, a.nsplit);
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
