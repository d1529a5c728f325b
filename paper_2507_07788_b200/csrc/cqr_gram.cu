// K1: tall-skinny Gram kernels, G = A^T B over the local row shard.
//
// Replaces `DenseVectorArray.gramian` (reference varray.py:150-155): the self
// Gram X^T X (bit-symmetric by construction: only the lower triangle is
// computed and mirrored) and the cross Gram Q_in^T Q of the update path.
//
// Layout: tall arrays are row-quad interleaved (cqr.h): element (r, c) at
// (r/4)*4*ldk + 4c + r%4, so a 32-row panel of a 64-column block is eight
// contiguous 2 KB runs (one run when the block spans the whole row) and the
// DMMA fragment loads from the staged copy are bank-conflict free without
// padding (lane (g, t) of a half-warp hits offset 4g + t (mod 16)).
//
// Work split: the k x k output is cut into 64x64 tiles; the self Gram pairs
// diagonal tiles (p, T-1-p) into one work item (two half tiles = one full
// load) and gives each off-diagonal tile its own item.  Rows are cut into
// `nsplit` contiguous ranges with nitems * nsplit <= 2 * SMs (one wave of two
// resident CTAs per SM).  Each CTA: one producer warp feeding a 3-stage
// full/empty mbarrier ring with cp.async.bulk (TMA bulk engine), four
// consumer warps each holding 32x32 register sub-tiles (16 DMMA.8x8x4 per 8
// LDS.64).  Per-(split, item) partials go to a workspace; `reduce` sums them
// in a fixed split order (deterministic, bitwise run-to-run).
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int GR_BR = 32;                       // rows per stage (8 quads)
constexpr int GR_CT = 64;                       // tile edge
constexpr int GR_QD = GR_CT * 4;                // doubles per quad of a 64-column block
constexpr int GR_BLK = (GR_BR / 4) * GR_QD;     // doubles per staged block (2048)
constexpr int GR_STAGES = 3;
constexpr int GR_STAGE_DOUBLES = 2 * GR_BLK;
constexpr int GR_THREADS = 160;                 // 4 consumer warps + 1 producer warp

size_t gram_smem_bytes() { return GR_STAGES * GR_STAGE_DOUBLES * sizeof(double) + 2 * GR_STAGES * 8 + 64; }

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

// k4-steps [ks0, ks1) (stride kstep) of one 32x32 register sub-tile.  ap / bp
// point at (column g, row t) of the sub-tile's A / B column range in a staged
// block; quad ks sits at +ks*GR_QD, the 8-column block i at +32*i.
template <bool DIAG>
__device__ __forceinline__ void subtile(double (&acc)[4][4][2], const double* ap, const double* bp, int ks0,
                                        int ks1, int kstep) {
  for (int ks = ks0; ks < ks1; ks += kstep) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = ap[ks * GR_QD + 32 * i];
    if (DIAG) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) dmma(acc[i][j], a[i], a[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bp[ks * GR_QD + 32 * j];
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

// stage rows [r0, r0 + nrows) of columns [c0, c0 + ncol) of a QI array into a
// dense [quad][64][4] block: one bulk copy per quad, or one in total when the
// block spans whole rows of the array
__device__ __forceinline__ void stage_block(double* dst, const double* src, int64_t ldk, int64_t r0, int nrows,
                                            int c0, int ncol, uint64_t* bar, int lane) {
  const int nq = nrows >> 2;
  const double* base = src + (r0 >> 2) * 4 * ldk + 4 * (int64_t)c0;
  if (ncol == GR_CT && ldk == GR_CT) {
    if (lane == 0) bulk_g2s_stream(dst, base, (uint32_t)nq * GR_QD * 8, bar);
  } else {
    for (int q = lane; q < nq; q += 32) bulk_g2s_stream(dst + q * GR_QD, base + q * 4 * ldk, (uint32_t)ncol * 32, bar);
  }
}

__global__ void __launch_bounds__(GR_THREADS, 2) gram_kernel(GramArgs args) {
  if (args.gate != nullptr && *args.gate != 0) return;   // gated off
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
  const bool narrowB = !self && ncolB <= 32;

  const int64_t npan = args.npanels;
  const int64_t p_begin = npan * split / args.nsplit;
  const int64_t p_end = npan * (split + 1) / args.nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GR_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 4) {
    // ---------------- producer warp
    int it = 0;
    for (int64_t p = p_begin; p < p_end; ++p, ++it) {
      const int s = it % GR_STAGES;
      const uint32_t use = it / GR_STAGES;
      if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
      const int64_t r0 = p * GR_BR;
      const int nrows = (int)imin64(GR_BR, args.rows - r0);
      double* As = stage_base + s * GR_STAGE_DOUBLES;
      double* Bs = As + GR_BLK;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(ncolA + ncolB) * nrows * 8);
      __syncwarp();
      stage_block(As, args.A, args.lda, r0, nrows, ia0, ncolA, &full[s], lane);
      if (ncolB) stage_block(Bs, args.B, args.ldb, r0, nrows, jb0, ncolB, &full[s], lane);
    }
    return;
  }

  // ---------------- consumer warps.  Roles (sub-tile = 32x32 of a 64x64 tile):
  //  off tile   : warp w -> sub-tile (w>>1, w&1) of tile (A, B)
  //  diag pair  : w0 -> A(0,0)+A(1,1), w1 -> A(1,0), w2 -> B(0,0)+B(1,1), w3 -> B(1,0)
  //  single diag: w0 -> (0,0), w2 -> (1,1), w1 / w3 -> (1,0) on even / odd k4 steps
  const int g = lane >> 2, t = lane & 3;
  const int fo = 4 * g + t;   // fragment offset inside a quad
  double acc0[4][4][2], acc1[4][4][2];
  zero_acc(acc0);
  zero_acc(acc1);

  int it = 0;
  for (int64_t p = p_begin; p < p_end; ++p, ++it) {
    const int s = it % GR_STAGES;
    mbar_wait(&full[s], (it / GR_STAGES) & 1);
    const int64_t r0 = p * GR_BR;
    const int nk4 = (int)imin64(GR_BR, args.rows - r0) >> 2;
    const double* As = stage_base + s * GR_STAGE_DOUBLES + fo;
    const double* Bs = As + GR_BLK;
    if (kind == 0 && narrowB) {
      // B has at most 32 columns (a skinny cross Gram: Q_in^T Q of the update
      // path): instead of two warps multiplying the tile's empty right half, the
      // k4 steps are split over warp pairs -- warps 0/1 take the even steps of
      // A sub-tiles 0/1, warps 2/3 the odd ones, summed below in a fixed order
      subtile<false>(acc0, As + 128 * (warp & 1), Bs, warp >> 1, nk4, 2);
    } else if (kind == 0) {
      const int wi = warp >> 1, wj = warp & 1;
      subtile<false>(acc0, As + 128 * wi, Bs + 128 * wj, 0, nk4, 1);
    } else if (kind == 1) {
      const double* T = (warp < 2) ? As : Bs;
      if ((warp & 1) == 0) {
        subtile<true>(acc0, T, nullptr, 0, nk4, 1);
        subtile<true>(acc1, T + 128, nullptr, 0, nk4, 1);
      } else {
        subtile<false>(acc0, T + 128, T, 0, nk4, 1);
      }
    } else {
      if (warp == 0) subtile<true>(acc0, As, nullptr, 0, nk4, 1);
      else if (warp == 2) subtile<true>(acc0, As + 128, nullptr, 0, nk4, 1);
      else subtile<false>(acc0, As + 128, As, warp == 1 ? 0 : 1, nk4, 2);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---------------- partials -> workspace: item slots of 64x64 (tile-local column-major)
  double* out = args.ws + ((int64_t)split * args.nitems + item) * (2 * GR_CT * GR_CT);
  if (kind == 0 && narrowB) {
    const int r0 = 32 * (warp & 1);
    if (warp >= 2) store_acc(acc0, out + GR_CT * GR_CT, r0, 0, g, t);   // odd steps parked in the second slot
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp < 2) {
      const double* o3 = out + GR_CT * GR_CT;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int idx = (8 * j + 2 * t + e) * GR_CT + r0 + 8 * i + g;
            out[idx] = acc0[i][j][e] + o3[idx];
          }
    }
  } else if (kind == 0) {
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
  if (args.gate != nullptr && *args.gate != 0) return;
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
  const size_t smem = gram_smem_bytes();
  {
    cudaError_t e = smem_attr((const void*)gram_kernel, smem);
    if (e != cudaSuccess) return e;
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
