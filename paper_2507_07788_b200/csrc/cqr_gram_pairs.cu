// K1 (v2): self Gram by block-row pairs, for k <= 256.
//
// Replaces `DenseVectorArray.gramian()` (reference varray.py:150-153) like
// cqr_gram.cu, with a schedule built for full-row panels:
//   * the lower triangle of the NB x NB grid of 8x8 blocks (NB = KP/8, KP =
//     k rounded up to a power of two >= 16) is cut into the NB/2 block-row
//     pairs (i, NB-1-i); every pair holds exactly NB+1 blocks, so one pair
//     per warp balances the DMMA work perfectly;
//   * a CTA (8 compute warps + a producer warp, one CTA per SM; for KP = 256
//     thread 0 issues the copies inline) owns 8 pairs -- the whole
//     triangle for KP <= 128 (KP < 128: several warps per pair, splitting
//     the k4 steps), half of it for KP = 256 (two CTAs per row range) -- and
//     streams 32-row panels of ALL k columns (QI layout: one bulk copy per
//     stage when ldk == KP), so X is read once (twice from L2 for KP = 256)
//     instead of once per 64x64 tile;
//   * per k4 step a warp loads the NB-i fragments of its columns once (the
//     two row fragments are among them) and issues NB+1 DMMA.8x8x4.
// Per-CTA partial triangles go to a workspace; a fixed-order reduce sums them.
#include "cqr_common.cuh"
#include "cqr_kernels.h"
#include "cqr_pairs.cuh"

namespace cqr {


template <int KP>
struct GPCfg {
  static constexpr int NB = KP / 8;
  static constexpr int PAIRS = NB / 2;
  static constexpr int ITEMS = (PAIRS > 8) ? PAIRS / 8 : 1;     // CTAs per row range
  static constexpr int WPP = (PAIRS >= 8) ? 1 : 8 / PAIRS;      // warps per pair
  // rows per stage: 32, more for narrow panels so a stage is >= 16 KB (bulk
  // copies below 16 KB stream measurably slower, profiles/r01_bulk_stream.jsonl)
  static constexpr int BR = (KP >= 64) ? 32 : 2048 / KP;
  static constexpr int STAGE = BR * KP;                         // doubles
  // ring depth: ~192 KB of panels in flight per SM (HBM latency x per-SM
  // bandwidth needs >= 64 KB outstanding), at most 8 stages
  static constexpr int S_FIT = (192 * 1024) / (STAGE * 8);
  static constexpr int STAGES = S_FIT > 8 ? 8 : (S_FIT < 3 ? 3 : S_FIT);
  // a dedicated producer warp (9 warps) where the consumers' registers allow
  // it; KP = 256 needs ~250 registers per thread, so thread 0 issues inline
  static constexpr bool PRODUCER = true;
  static constexpr int THREADS = PRODUCER ? 288 : 256;
};

template <int KP>
size_t gp_smem_bytes() {
  return (size_t)GPCfg<KP>::STAGES * GPCfg<KP>::STAGE * sizeof(double) + 2 * GPCfg<KP>::STAGES * 8 + 64;
}

template <int KP>
__global__ void __launch_bounds__(GPCfg<KP>::THREADS, 1) gram_pairs_kernel(const double* __restrict__ X, int64_t ldx, int k,
                                                                   int64_t rows, int nsplit, double* ws,
                                                                   const int* gate) {
  if (gate != nullptr && *gate != 0) return;   // gated off
  using C = GPCfg<KP>;
  constexpr int NB = C::NB;
  constexpr int GP_STAGES = C::STAGES;
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GP_STAGES * C::STAGE);
  uint64_t* empty = full + GP_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x % C::ITEMS, split = blockIdx.x / C::ITEMS;
  const int64_t npan = ceil_div(rows, C::BR);
  const int64_t p0 = npan * split / nsplit, p1 = npan * (split + 1) / nsplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GP_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t p, int st) {
    const int64_t r0 = p * C::BR;
    const int nq = (int)imin64(C::BR, rows - r0) >> 2;
    double* dst = smem + st * C::STAGE;
    const double* src = X + (r0 >> 2) * 4 * ldx;
    mbar_arrive_expect_tx(&full[st], (uint32_t)nq * k * 32);
    if (ldx == KP && k == KP) {
      bulk_g2s_stream(dst, src, (uint32_t)nq * KP * 32, &full[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s_stream(dst + q * 4 * KP, src + q * 4 * ldx, (uint32_t)k * 32, &full[st]);
    }
  };
  if constexpr (C::PRODUCER) {
    if (warp == 8) {
      // producer warp: refill each stage as soon as the 8 consumers release it
      if (lane == 0) {
        int it = 0;
        for (int64_t p = p0; p < p1; ++p, ++it) {
          const int s = it % GP_STAGES;
          if (it >= GP_STAGES) mbar_wait(&empty[s], ((it / GP_STAGES) - 1) & 1);
          issue(p, s);
        }
      }
      return;
    }
  }
  // inline producer (thread 0): D panels in flight, refills the stage of panel it-LAG
  constexpr int LAG = GP_STAGES >= 6 ? 2 : 1;
  constexpr int D = GP_STAGES - LAG;
  if (!C::PRODUCER && threadIdx.x == 0)
    for (int j = 0; j < D && p0 + j < p1; ++j) issue(p0 + j, j);

  const int g = lane >> 2, t = lane & 3;
  const int pair = item * 8 + warp / C::WPP;       // pair index handled by this warp
  const int sub = warp % C::WPP;                   // k4-step phase when several warps share a pair
  double acc[NB + 1][2];
#pragma unroll
  for (int c = 0; c <= NB; ++c) { acc[c][0] = 0.0; acc[c][1] = 0.0; }
  const double* fbase = smem + 4 * g + t;           // (column g, row t) of quad 0
  const bool active = pair < C::PAIRS;
  int it = 0;
  for (int64_t p = p0; p < p1; ++p, ++it) {
    const int s = it % GP_STAGES;
    if (!C::PRODUCER && threadIdx.x == 0 && p + D < p1) {
      // stage s2 last held panel it - LAG
      const int it2 = it + D;
      const int s2 = it2 % GP_STAGES;
      if (it2 >= GP_STAGES) mbar_wait(&empty[s2], ((it2 / GP_STAGES) - 1) & 1);
      issue(p + D, s2);
    }
    mbar_wait(&full[s], (it / GP_STAGES) & 1);
    const int nk4 = (int)imin64(C::BR, rows - p * C::BR) >> 2;
    if (active) {
      const double* fp = fbase + s * C::STAGE;
      // columns >= k of the staged panel hold stale data: only outputs in
      // rows/cols >= k see them, and those are never read back
      if constexpr (KP >= 256) {
        PairDispatch<NB, 0>::run_lean(pair, acc, fp, sub, nk4, C::WPP);
      } else {
        // full panels of narrow widths: fully unrolled (KP = 128 measured faster with the loop)
        if (KP <= 64 && nk4 == C::BR / 4)
          PairDispatch<NB, 0>::template run_fixed<C::BR / 4 / C::WPP>(pair, acc, fp, sub, C::WPP);
        else PairDispatch<NB, 0>::run(pair, acc, fp, sub, nk4, C::WPP);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- per-CTA partial (KP x KP column-major, lower triangle), warps in fixed order
  double* out = ws + ((int64_t)split * C::ITEMS + item) * KP * KP;
  for (int e = threadIdx.x; e < KP * KP; e += 256) out[e] = 0.0;
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int w = 0; w < 8; ++w) {
    if (warp == w && active) PairDispatch<NB, 0>::store(pair, acc, out, g, t);
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
}

static int gp_kp(int k) {
  if (k <= 16) return 16;
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  if (k <= 128) return 128;
  if (k <= 256) return 256;
  return 0;
}

bool gram_pairs_supported(int k) { return k >= 1 && gp_kp(k) != 0; }

static void gp_grid(int64_t rows, int kp, int& items, int& nsplit) {
  items = (kp == 256) ? 2 : 1;
  const int64_t npan = ceil_div(rows, (kp >= 64) ? 32 : 2048 / kp);
  int64_t ns = num_sms() / items;
  if (ns > npan) ns = npan;
  if (ns < 1) ns = 1;
  nsplit = (int)ns;
}

size_t gram_pairs_ws_bytes(int64_t rows, int k) {
  const int kp = gp_kp(k);
  if (!kp) return 0;
  int items, nsplit;
  gp_grid(rows, kp, items, nsplit);
  return (size_t)items * nsplit * kp * kp * sizeof(double) + 256;
}

template <int KP>
static cudaError_t launch_gp(const double* X, int64_t ldx, int k, int64_t rows, double* G, int ldg, double* ws,
                             cudaStream_t s, const int* gate) {
  const size_t smem = gp_smem_bytes<KP>();
  {
    cudaError_t e = smem_attr((const void*)gram_pairs_kernel<KP>, smem);
    if (e != cudaSuccess) return e;
  }
  int items, nsplit;
  gp_grid(rows, KP, items, nsplit);
  gram_pairs_kernel<KP><<<items * nsplit, GPCfg<KP>::THREADS, smem, s>>>(X, ldx, k, rows, nsplit, ws, gate);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_partials_reduce<<<gram_partials_reduce_blocks(k), PR_THREADS, 0, s>>>(ws, items * nsplit, KP, k, G, ldg,
                                                                                gate);
  return cudaGetLastError();
}

cudaError_t gram_pairs_launch(const double* X, int64_t ldx, int k, int64_t rows, double* G, int ldg, double* ws,
                              cudaStream_t s, const int* gate) {
  switch (gp_kp(k)) {
    case 16: return launch_gp<16>(X, ldx, k, rows, G, ldg, ws, s, gate);
    case 32: return launch_gp<32>(X, ldx, k, rows, G, ldg, ws, s, gate);
    case 64: return launch_gp<64>(X, ldx, k, rows, G, ldg, ws, s, gate);
    case 128: return launch_gp<128>(X, ldx, k, rows, G, ldg, ws, s, gate);
    case 256: return launch_gp<256>(X, ldx, k, rows, G, ldg, ws, s, gate);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace cqr
