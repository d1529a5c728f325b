// K2 fused pass for 33 <= k <= 64 and 97 <= k <= 128: Q = X R^-1 (R^-1
// upper triangular) and G = Q^T Q in one stream over X (Q may alias X).
//
// Replaces the lincomb + gramian pair of one iteration (reference
// algorithms.py:350,352 / :238,:240 / :211 + chol_qr2's second Gram) with one
// HBM read of X and one write of Q per pass (the unfused pair reads Q again).
//
// Warp-specialised, one CTA per SM, persistent over 32-row panels.  With
// NB = KP/8 column blocks and P = NB/2:
//   * P TRMM warps: warp c owns the column-block pair (c, NB-1-c) for all 32
//     rows of a panel -- every pair costs 2(NB+1) k4 steps, so the warps are
//     balanced -- reads the X panel from a TMA ring (XST stages) and writes
//     Q into a ring of Q panels in shared memory;
//   * P Gram warps: warp i owns the block-row pair (i, NB-1-i) of the lower
//     triangle (NB+1 blocks each) and accumulates it from the Q ring in
//     registers over the whole sweep; one lane of Gram warp 0 stores each Q
//     panel to HBM with bulk copies from the ring.
// Per 8 rows both halves issue NB(NB+1) DMMA.8x8x4, all from compile-time
// loops (no predicated-off DMMA occupies the tensor pipe).  The groups hand
// panels over through mbarriers only (no CTA-wide barrier in the sweep).
// Thread 0 issues the bulk copies.  Per-CTA partial triangles are summed in a
// fixed warp order, then over CTAs by gram_partials_reduce in a fixed order.
#include "cqr_common.cuh"
#include "cqr_kernels.h"
#include "cqr_pairs.cuh"

namespace cqr {

constexpr int FU_BR = 32;   // rows per panel = 8 k4 steps

template <int KP>
struct FuCfg {
  static constexpr int NB = KP / 8;
  static constexpr int PAIRS = NB / 2;        // TRMM warps = Gram warps
  // KP = 64: a dedicated producer warp issues the X copies; KP = 128 (16
  // compute warps, 128 registers each) keeps the producer inline on thread 0
  static constexpr bool PRODUCER = KP == 64;
  // KP = 64: a dedicated storer warp also writes the Q panels back to HBM
  // (otherwise one lane of Gram warp 0 does, and that warp paces the Gram side)
  static constexpr bool STORER = KP == 64;
  static constexpr int THREADS = 64 * PAIRS + (PRODUCER ? 32 : 0) + (STORER ? 32 : 0);
  static constexpr int NKT = KP / CT_K;       // 32-row coefficient k tiles
  static constexpr int NNT = KP / CT_N;       // 64-column coefficient n tiles
  static constexpr int STAGE = FU_BR * KP;    // doubles per panel
  static constexpr int XST = (KP == 64) ? 6 : 2;
  static constexpr int QB = (KP == 64) ? 4 : 1;
};

// coefficient tiles of R^-1 that hold upper-triangle entries (kt*32 < (nt+1)*64), packed in order
template <int KP>
__host__ __device__ constexpr int tile_slot(int kt, int nt) {
  int slot = 0;
  for (int n = 0; n < nt; ++n) slot += (FuCfg<KP>::NKT < 2 * (n + 1)) ? FuCfg<KP>::NKT : 2 * (n + 1);
  return slot + kt;
}
template <int KP>
__host__ __device__ constexpr int n_tiles_needed() {
  return tile_slot<KP>(0, FuCfg<KP>::NNT);
}
template <int KP>
__host__ __device__ constexpr size_t fused_smem_doubles() {
  return (size_t)n_tiles_needed<KP>() * CT_TILE + (size_t)(FuCfg<KP>::XST + FuCfg<KP>::QB) * FuCfg<KP>::STAGE;
}

// Q[32 rows, blocks CA and CB] of one panel; xp -> (row g, col t) of the
// staged X panel, rp -> (col g, k t) of the coefficient tile area.  The
// fragments of k4 step ks+1 are loaded before the DMMAs of step ks issue.
template <int KP, int CA, bool KFULL>
__device__ __forceinline__ void fu_trmm(double (&acc)[4][2][2], const double* xp, const double* rp, int t, int k) {
  constexpr int NB = KP / 8, CB = NB - 1 - CA;
  constexpr int NKA = 2 * (CA + 1), NKB = 2 * (CB + 1);
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int c = 0; c < 2; ++c) { acc[rb][c][0] = 0.0; acc[rb][c][1] = 0.0; }
  double a[2][4], bA[2], bB[2];
  auto load = [&](int ks, int buf) {
    const bool kv = KFULL || (4 * ks + t < k);   // X columns >= k of the stage are stale
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) a[buf][rb] = kv ? xp[rb * 8 * KP + 16 * ks] : 0.0;
    bB[buf] = rp[tile_slot<KP>(ks / 8, CB / 8) * CT_TILE + ((8 * CB) & 63) * CT_LD + 4 * (ks % 8)];
    if (ks < NKA) bA[buf] = rp[tile_slot<KP>(ks / 8, CA / 8) * CT_TILE + ((8 * CA) & 63) * CT_LD + 4 * (ks % 8)];
  };
  load(0, 0);
#pragma unroll
  for (int ks = 0; ks < NKB; ++ks) {
    const int cur = ks & 1;
    if (ks + 1 < NKB) load(ks + 1, cur ^ 1);
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) dmma(acc[rb][1], a[cur][rb], bB[cur]);
    if (ks < NKA) {
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) dmma(acc[rb][0], a[cur][rb], bA[cur]);
    }
  }
}

template <int KP, int C, bool KFULL>
struct TrmmDispatch {
  __device__ static void run(int pair, double (&acc)[4][2][2], const double* xp, const double* rp, int t, int k) {
    if (pair == C) fu_trmm<KP, C, KFULL>(acc, xp, rp, t, k);
    else TrmmDispatch<KP, C + 1, KFULL>::run(pair, acc, xp, rp, t, k);
  }
};
template <int KP, bool KFULL>
struct TrmmDispatch<KP, KP / 16, KFULL> {
  __device__ static void run(int, double (&)[4][2][2], const double*, const double*, int, int) {}
};

template <int KP, bool KFULL>
__global__ void __launch_bounds__(FuCfg<KP>::THREADS, 1)
    apply_gram_fused_kernel(const double* X, int64_t ldx, int k, const double* __restrict__ Rt, double* Q,
                            int64_t ldq, int64_t rows, double* __restrict__ ws, const int* gate) {
  if (gate != nullptr && *gate != 0) return;   // gated off
  using C = FuCfg<KP>;
  constexpr int NB = C::NB, P = C::PAIRS, XST = C::XST, QB = C::QB;
  // thread 0 keeps XD panels in flight and refills the stage of panel j-XLAG,
  // so warp 0 does not wait for the slowest TRMM warp every panel
  constexpr int XLAG = XST >= 6 ? 2 : 1, XD = XST - XLAG;
  extern __shared__ __align__(128) double smem[];
  double* rt_s = smem;                                   // R^-1 tiles
  double* xst = rt_s + n_tiles_needed<KP>() * CT_TILE;   // XST X panels
  double* qbuf = xst + XST * C::STAGE;                   // QB Q panels
  double* red = smem;                                    // KP x KP partial, after the sweep
  static_assert((size_t)KP * KP <= (size_t)n_tiles_needed<KP>() * CT_TILE + (size_t)XST * C::STAGE,
                "the partial must not overlap the Q ring");
  __shared__ __align__(8) uint64_t bars[2 * XST + 2 * QB + 1];
  uint64_t* xfull = bars;
  uint64_t* xempty = xfull + XST;
  uint64_t* qfull = xempty + XST;
  uint64_t* qempty = qfull + QB;
  uint64_t* rbar = qempty + QB;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t npan = ceil_div(rows, FU_BR);
  const int64_t mine = (npan > blockIdx.x) ? ceil_div(npan - blockIdx.x, gridDim.x) : 0;
  constexpr bool kfull = KFULL;   // k == KP

  if (tid == 0) {
    for (int s = 0; s < XST; ++s) { mbar_init(&xfull[s], 1); mbar_init(&xempty[s], P); }
    for (int s = 0; s < QB; ++s) { mbar_init(&qfull[s], 32 * P); mbar_init(&qempty[s], P + (C::STORER ? 1 : 0)); }
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t j, int st) {
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * FU_BR;
    const int nq = (int)imin64(FU_BR, rows - r0) >> 2;
    double* dst = xst + st * C::STAGE;
    const double* src = X + (r0 >> 2) * 4 * ldx;
    mbar_arrive_expect_tx(&xfull[st], (uint32_t)nq * k * 32);
    if (ldx == KP && kfull) {
      bulk_g2s_stream(dst, src, (uint32_t)nq * KP * 32, &xfull[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s_stream(dst + q * 4 * KP, src + q * 4 * ldx, (uint32_t)k * 32, &xfull[st]);
    }
  };
  if (tid == 0) {
    mbar_arrive_expect_tx(rbar, n_tiles_needed<KP>() * CT_TILE * 8);
    for (int nt = 0; nt < C::NNT; ++nt)
      for (int kt = 0; kt < min(C::NKT, 2 * (nt + 1)); ++kt)
        bulk_g2s(rt_s + tile_slot<KP>(kt, nt) * CT_TILE, Rt + ((int64_t)nt * C::NKT + kt) * CT_TILE, CT_TILE * 8,
                 rbar);
    if (!C::PRODUCER)
      for (int j = 0; j < XD && j < mine; ++j) issue(j, j);
  }
  if constexpr (C::PRODUCER) {
    if (warp == 2 * P) {
      if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t j = 0; j < mine; ++j) {
          if (j >= XST) mbar_wait(&xempty[s], ph ^ 1);
          issue(j, s);
          if (++s == XST) { s = 0; ph ^= 1; }
        }
      }
      return;
    }
  }
  if constexpr (C::STORER) {
    if (warp == 2 * P + 1) {
      // storer warp: Q panel j -> HBM as soon as the TRMM warps filled it; the
      // slot is released once the bulk engine has read it (one group in flight)
      if (lane == 0) {
        int qs = 0, prev = -1;
        uint32_t qph = 0;
        for (int64_t j = 0; j < mine; ++j) {
          mbar_wait(&qfull[qs], qph);
          const int64_t r0 = (blockIdx.x + j * gridDim.x) * FU_BR;
          const int nq = (int)imin64(FU_BR, rows - r0) >> 2;
          const double* src = qbuf + qs * C::STAGE;
          double* dst = Q + (r0 >> 2) * 4 * ldq;
          if (ldq == KP && KFULL) {
            bulk_s2g_stream(dst, src, (uint32_t)nq * KP * 32);
          } else {
            for (int q = 0; q < nq; ++q) bulk_s2g_stream(dst + q * 4 * ldq, src + q * 4 * KP, (uint32_t)k * 32);
          }
          bulk_commit();
          if (prev >= 0) {
            bulk_wait_read<1>();
            mbar_arrive(&qempty[prev]);
          }
          prev = qs;
          if (++qs == QB) { qs = 0; qph ^= 1; }
        }
        if (prev >= 0) {
          bulk_wait_read<0>();
          mbar_arrive(&qempty[prev]);
        }
        bulk_wait<0>();
      }
      return;
    }
  }

  if (warp < P) {
    // ---------------- TRMM warps
    const int cA = warp, cB = NB - 1 - warp;
    const double* rp = rt_s + g * CT_LD + t;
    mbar_wait(rbar, 0);
    int s = 0, qs = 0;          // ring slots of panel j
    uint32_t xph = 0, qph = 0;  // (j / XST) & 1, (j / QB) & 1
    for (int64_t j = 0; j < mine; ++j) {
      if (!C::PRODUCER && tid == 0 && j + XD < mine) {
        // stage s2 last held panel j - XLAG (released by every TRMM warp)
        const int64_t j2 = j + XD;
        const int s2 = (int)(j2 % XST);
        if (j2 >= XST) mbar_wait(&xempty[s2], (uint32_t)((j2 / XST) - 1) & 1);
        issue(j2, s2);
      }
      mbar_wait(&xfull[s], xph);
      const int64_t r0 = (blockIdx.x + j * gridDim.x) * FU_BR;
      const int nrows = (int)imin64(FU_BR, rows - r0);
      const double* xp = xst + s * C::STAGE + (g >> 2) * 4 * KP + 4 * t + (g & 3);
      double acc[4][2][2];
      TrmmDispatch<KP, 0, KFULL>::run(warp, acc, xp, rp, t, k);
      __syncwarp();
      if (lane == 0) mbar_arrive(&xempty[s]);
      // Q -> the Q ring (zeros past the last row / column); a Gram lane
      // stores the panel to HBM from there with one bulk copy per quad
      if (j >= QB) mbar_wait(&qempty[qs], qph ^ 1);
      double* qd = qbuf + qs * C::STAGE + (g >> 2) * 4 * KP + (g & 3);
      if (KFULL && nrows == FU_BR) {
#pragma unroll
        for (int rb = 0; rb < 4; ++rb)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int e0 = 0; e0 < 2; ++e0) {
              // lanes t >= 2 store e = 1 first: every half-warp then covers all 32 banks
              const int e = e0 ^ (t >> 1);
              qd[rb * 8 * KP + 4 * (8 * (c ? cB : cA) + 2 * t + e)] = e ? acc[rb][c][1] : acc[rb][c][0];
            }
      } else {
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int row = 8 * rb + g;
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int col = 8 * (c ? cB : cA) + 2 * t + e;
              qd[rb * 8 * KP + 4 * col] = (row < nrows && col < k) ? acc[rb][c][e] : 0.0;
            }
        }
      }
      fence_proxy_async_smem();  // the bulk store reads the ring through the async proxy
      mbar_arrive(&qfull[qs]);   // every lane: its own stores are released
      if (++s == XST) { s = 0; xph ^= 1; }
      if (++qs == QB) { qs = 0; qph ^= 1; }
    }
  } else {
    // ---------------- Gram warps
    const int pr = warp - P;
    const double* fb = qbuf + 4 * g + t;
    double gacc[NB + 1][2];
#pragma unroll
    for (int c = 0; c <= NB; ++c) { gacc[c][0] = 0.0; gacc[c][1] = 0.0; }
    int qs = 0;
    uint32_t qph = 0;
    const bool storer = !C::STORER && pr == 0 && lane == 0;
    for (int64_t j = 0; j < mine; ++j) {
      mbar_wait(&qfull[qs], qph);
      if (storer) {
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * FU_BR;
        const int nq = (int)imin64(FU_BR, rows - r0) >> 2;
        const double* src = qbuf + qs * C::STAGE;
        double* dst = Q + (r0 >> 2) * 4 * ldq;
        if (ldq == KP && KFULL) {
          bulk_s2g_stream(dst, src, (uint32_t)nq * KP * 32);
        } else {
          for (int q = 0; q < nq; ++q) bulk_s2g_stream(dst + q * 4 * ldq, src + q * 4 * KP, (uint32_t)k * 32);
        }
        bulk_commit();
      }
      PairDispatch<NB, 0>::template run<(KP == 64)>(pr, gacc, fb + qs * C::STAGE, 0, FU_BR / 4, 1);
      if (storer) bulk_wait_read<0>();   // the slot may be refilled once the store has read it
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (++qs == QB) { qs = 0; qph ^= 1; }
    }
    if (storer) bulk_wait<0>();
    // ---- per-CTA partial (KP x KP column-major, lower triangle), Gram warps in
    // fixed order.  Every TRMM warp finished with the tiles and X stages before
    // its last qfull arrive, and red (KP*KP doubles) ends before the Q ring.
    const int gt = tid - 32 * P;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * P) : "memory");
    for (int e = gt; e < KP * KP; e += 32 * P) red[e] = 0.0;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * P) : "memory");
    for (int w = 0; w < P; ++w) {
      if (pr == w) PairDispatch<NB, 0>::store(w, gacc, red, g, t);
      asm volatile("bar.sync 1, %0;" ::"r"(32 * P) : "memory");
    }
    double* out = ws + (int64_t)blockIdx.x * KP * KP;
    for (int e = gt; e < KP * KP; e += 32 * P) out[e] = red[e];
  }
}

// ---------------------------------------------------------------------------
// K2+K1 for k <= 64, register resident ("transposed TRMM"): each warp owns 8
// rows of a 64-row panel and computes Q^T = R^-T X^T for them, i.e. the DMMA
// takes A = R^-T (lane (g,t): R^-1[4ks+t][8j+g], the coefficient tiles as
// stored) and B = X^T (lane (g,t): X[r0+g][4ks+t], the staged QI panel).  The
// accumulator of column block j then holds, in lane (g,t),
//   qt[j][e] = Q[r0 + 2t + e][8j + g],
// which is exactly the A fragment (and the B fragment) of the Gram DMMA over
// the 4 rows {r0 + 2t + e : t} -- the k index of a DMMA is a row index here,
// and a Gram is a sum over rows in any order.  So the Gram of the fresh Q
// block is accumulated straight from the TRMM accumulators: no Q round trip
// through shared memory, no hand-over between warp groups.  Each lane's two
// values are consecutive in the QI layout (rows 2t, 2t+1 of one quad), so Q
// goes to HBM as one 16-byte store per lane per column block, two fully
// coalesced 256-byte runs per warp instruction.
// Per 8 rows a warp issues NB(NB+1) TRMM DMMAs (column block j needs K up to
// 8j+8) and NB(NB+1) Gram DMMAs (the NB(NB+1)/2 lower blocks, two row quads)
// from compile-time loops (no predicated-off DMMA); its Gram partial stays
// in registers (NB(NB+1) doubles per lane) for the whole sweep.
// Only the X panel and the R^-1 tiles live in shared memory: 88 LDS.64 per
// 144 DMMAs at k = 64, against ~1.0 LDS + 0.1 STS per DMMA in the two-group
// kernel above.
constexpr int RT_ROWS = 64;   // rows per staged panel (8 compute warps x 8 rows)

template <int KP>
struct RtCfg {
  static constexpr int NB = KP / 8;
  static constexpr int NKS = KP / 4;                      // k4 steps of the TRMM
  static constexpr int NKT = KP > CT_K ? KP / CT_K : 1;   // 32-row coefficient k tiles (one 64-wide n tile)
  static constexpr int NG = NB * (NB + 1) / 2;            // lower-triangle 8x8 blocks
  static constexpr int STAGE = RT_ROWS * KP;              // doubles per panel
  static constexpr int STAGES = KP >= 64 ? 5 : 8;
  static constexpr int THREADS = 256;                     // 8 compute warps
};
template <int KP>
__host__ __device__ constexpr size_t rt_smem_doubles() {
  return (size_t)RtCfg<KP>::NKT * CT_TILE + (size_t)RtCfg<KP>::STAGES * RtCfg<KP>::STAGE;
}

__device__ __forceinline__ void st_global_v2(double* p, double a, double b) {
#if CQR_L2_HINTS
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
#else
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
#endif
}

// TRMM = false: the same sweep as a plain self Gram of X (k <= 64): the
// fragments of the Gram DMMA are loaded straight from the staged panel (lane
// (g,t): X[r0 + t + 4e][8b + g], conflict-free), 16 LDS.64 per 72 DMMAs, and
// the warp's 36-block partial stays in registers.
template <int KP, bool KFULL, bool TRMM>
__global__ void __launch_bounds__(RtCfg<KP>::THREADS, 1)
    apply_gram_rt_kernel(const double* X, int64_t ldx, int k, const double* __restrict__ Rt, double* Q, int64_t ldq,
                         int64_t rows, double* __restrict__ ws, const int* gate) {
  if (gate != nullptr && *gate != 0) return;   // gated off
  using C = RtCfg<KP>;
  constexpr int NB = C::NB, NKS = C::NKS, ST = C::STAGES;
  // thread 0 keeps D panels in flight and refills the stage of panel j - LAG
  // (8 warps, no producer warp: a 9-warp CTA is capped at 168 registers per
  // thread, and the Gram partial alone takes 144 at k = 64)
  constexpr int LAG = 2, D = ST - LAG;
  extern __shared__ __align__(128) double smem[];
  double* rt_s = smem;                      // R^-1 coefficient tiles
  double* xst = smem + C::NKT * CT_TILE;    // ST X panels (QI, ldk = KP)
  __shared__ __align__(8) uint64_t bars[2 * ST + 1];
  uint64_t* full = bars;
  uint64_t* empty = bars + ST;
  uint64_t* rbar = bars + 2 * ST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t npan = ceil_div(rows, RT_ROWS);
  const int64_t mine = (npan > blockIdx.x) ? ceil_div(npan - blockIdx.x, gridDim.x) : 0;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t j, int st) {
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * RT_ROWS;
    const int nq = (int)imin64(RT_ROWS, rows - r0) >> 2;
    double* dst = xst + st * C::STAGE;
    const double* src = X + (r0 >> 2) * 4 * ldx;
    mbar_arrive_expect_tx(&full[st], (uint32_t)nq * k * 32);
    if (ldx == KP && KFULL) {
      bulk_g2s_stream(dst, src, (uint32_t)nq * KP * 32, &full[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s_stream(dst + q * 4 * KP, src + q * 4 * ldx, (uint32_t)k * 32, &full[st]);
    }
  };
  if (tid == 0) {
    if (TRMM) {
      mbar_arrive_expect_tx(rbar, C::NKT * CT_TILE * 8);
      for (int kt = 0; kt < C::NKT; ++kt)
        bulk_g2s(rt_s + kt * CT_TILE, Rt + (int64_t)kt * CT_TILE, CT_TILE * 8, rbar);
    }
    for (int j = 0; j < D && j < mine; ++j) issue(j, j);
  }

  // ---------------- compute warps: 8 rows of every panel each
  double gacc[C::NG][2];
#pragma unroll
  for (int b = 0; b < C::NG; ++b) { gacc[b][0] = 0.0; gacc[b][1] = 0.0; }
  // A fragments (R^-1[4ks+t][8j+g]) at rp[tile(ks) + 8j*CT_LD + 4(ks%8)]
  const double* rp = rt_s + g * CT_LD + t;
  if (TRMM) mbar_wait(rbar, 0);
  int s = 0;
  uint32_t ph = 0;
  for (int64_t j = 0; j < mine; ++j) {
    if (tid == 0 && j + D < mine) {
      // stage s2 last held panel j - LAG (released by all 8 warps)
      const int64_t j2 = j + D;
      const int s2 = (int)(j2 % ST);
      if (j2 >= ST) mbar_wait(&empty[s2], (uint32_t)((j2 / ST) - 1) & 1);
      issue(j2, s2);
    }
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * RT_ROWS + 8 * warp;
    const bool valid = r0 < rows;   // rows is a multiple of 16: a row octet is all in or all out
    mbar_wait(&full[s], ph);
    double qt[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) { qt[b][0] = 0.0; qt[b][1] = 0.0; }
    if (!TRMM && valid) {
      // Gram operands straight from the panel: rows r0 + t + 4e (quad 2*warp + e), column 8b + g
      const double* xp = xst + s * C::STAGE + 2 * warp * 4 * KP + 4 * g + t;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int b = 0; b < NB; ++b) qt[b][e] = (KFULL || 8 * b + g < k) ? xp[e * 4 * KP + 32 * b] : 0.0;
    }
    if (TRMM && valid) {
      // B fragments X[r0+g][4ks+t]: quad 2*warp + g/4 of the panel, conflict-free
      const double* xp = xst + s * C::STAGE + (2 * warp + (g >> 2)) * 4 * KP + 4 * t + (g & 3);
      double xb[2];
      xb[0] = (KFULL || t < k) ? xp[0] : 0.0;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int cur = ks & 1;
        if (ks + 1 < NKS) xb[cur ^ 1] = (KFULL || 4 * (ks + 1) + t < k) ? xp[16 * (ks + 1)] : 0.0;
        // column blocks j >= ks/2 see k4 step ks (R^-1 upper triangular)
#pragma unroll
        for (int b = ks / 2; b < NB; ++b) {
          const double ra = rp[(ks / 8) * CT_TILE + 8 * b * CT_LD + 4 * (ks % 8)];
          dmma(qt[b], ra, xb[cur]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // the panel is consumed: the producer may refill it
    if (++s == ST) { s = 0; ph ^= 1; }
    if (!valid) continue;
    if (TRMM && !KFULL) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (8 * b + g >= k) { qt[b][0] = 0.0; qt[b][1] = 0.0; }
    }
    // Q -> HBM: lane (g,t) holds rows 2t, 2t+1 (one quad, consecutive) of column 8b+g
    if (TRMM) {
      double* qd = Q + ((r0 >> 2) + (t >> 1)) * 4 * ldq + 4 * g + 2 * (t & 1);
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (KFULL || 8 * b + g < k) st_global_v2(qd + 32 * b, qt[b][0], qt[b][1]);
    }
    // Gram of the block: G(i, c) += sum over the 8 rows, two row quads
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) dmma(gacc[i * (i + 1) / 2 + c], qt[i][e], qt[c][e]);
    }
  }

  // ---- per-CTA partial (KP x KP column-major, lower triangle): warps in fixed order
  double* red = smem;
  __syncthreads();   // every warp is done with the tiles and panels
  for (int e = tid; e < KP * KP; e += 256) red[e] = 0.0;
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) red[(8 * c + 2 * t + e) * KP + 8 * i + g] += gacc[i * (i + 1) / 2 + c][e];
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
  double* out = ws + (int64_t)blockIdx.x * KP * KP;
  for (int e = tid; e < KP * KP; e += 256) out[e] = red[e];
}

static int fused_kp(int k) {
  if (k > 32 && k <= 64) return 64;
  if (k > 96 && k <= 128) return 128;
  return 0;   // k <= 32 and 65..96: unfused path
}
static int rt_kp(int k) {
  if (k < 1) return 0;
  if (k <= 16) return 16;
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  return 0;
}

// Fused-pass selection (cqr_set_fused):
//   2 (default) "auto": the register-resident kernel for k <= 64, the
//     two-kernel TRMM then Gram path otherwise;
//   1: every fused kernel (register-resident for k <= 64, the two-group
//     kernel for 97 <= k <= 128);
//   0: never fused.
// The two-group kernel is not the default for 97..128: there every pass is
// FP64-pipe bound and its split of one SM between two dependent warp groups
// costs more than the saved read of Q (k=128 fused 5.89 ms vs 2.21 + 2.10 ms
// at m=4M, tools/fused_probe.py).
static int g_fused_mode = 2;
void set_fused(int mode) { g_fused_mode = mode < 0 ? 0 : (mode > 2 ? 2 : mode); }
static int fused_variant(int k) {   // 0 none, 1 register-resident, 2 two-group
  if (g_fused_mode == 0 || k < 1) return 0;
  if (rt_kp(k)) return 1;
  if (g_fused_mode == 1 && fused_kp(k) == 128) return 2;
  return 0;
}
bool apply_gram_fused_supported(int k) { return fused_variant(k) != 0; }

static int fused_ctas(int64_t rows) {
  int64_t n = ceil_div(rows, FU_BR);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}
static int rt_ctas(int64_t rows) {
  int64_t n = ceil_div(rows, RT_ROWS);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

size_t apply_gram_fused_ws_bytes(int64_t rows, int k) {
  switch (fused_variant(k)) {
    case 1: return (size_t)rt_ctas(rows) * rt_kp(k) * rt_kp(k) * sizeof(double) + 256;
    case 2: return (size_t)fused_ctas(rows) * fused_kp(k) * fused_kp(k) * sizeof(double) + 256;
    default: return 0;
  }
}

template <int KP, bool TRMM>
static cudaError_t launch_rt(const double* X, int64_t ldx, int k, const double* Rt, double* Q, int64_t ldq,
                             int64_t rows, double* G, int ldg, double* ws, cudaStream_t s, const int* gate) {
  const size_t smem = rt_smem_doubles<KP>() * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)apply_gram_rt_kernel<KP, true, TRMM>, smem);
    if (e == cudaSuccess) e = smem_attr((const void*)apply_gram_rt_kernel<KP, false, TRMM>, smem);
    if (e != cudaSuccess) return e;
  }
  const int ctas = rt_ctas(rows);
  if (k == KP)
    apply_gram_rt_kernel<KP, true, TRMM><<<ctas, RtCfg<KP>::THREADS, smem, s>>>(X, ldx, k, Rt, Q, ldq, rows, ws, gate);
  else
    apply_gram_rt_kernel<KP, false, TRMM><<<ctas, RtCfg<KP>::THREADS, smem, s>>>(X, ldx, k, Rt, Q, ldq, rows, ws,
                                                                                gate);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_partials_reduce<<<gram_partials_reduce_blocks(k), PR_THREADS, 0, s>>>(ws, ctas, KP, k, G, ldg, gate);
  return cudaGetLastError();
}

template <int KP>
static cudaError_t launch_fused(const double* X, int64_t ldx, int k, const double* Rt, double* Q, int64_t ldq,
                                int64_t rows, double* G, int ldg, double* ws, cudaStream_t s, const int* gate) {
  const size_t smem = fused_smem_doubles<KP>() * sizeof(double);
  {
    cudaError_t e = smem_attr((const void*)apply_gram_fused_kernel<KP, true>, smem);
    if (e == cudaSuccess) e = smem_attr((const void*)apply_gram_fused_kernel<KP, false>, smem);
    if (e != cudaSuccess) return e;
  }
  const int ctas = fused_ctas(rows);
  if (k == KP)
    apply_gram_fused_kernel<KP, true><<<ctas, FuCfg<KP>::THREADS, smem, s>>>(X, ldx, k, Rt, Q, ldq, rows, ws, gate);
  else
    apply_gram_fused_kernel<KP, false><<<ctas, FuCfg<KP>::THREADS, smem, s>>>(X, ldx, k, Rt, Q, ldq, rows, ws, gate);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_partials_reduce<<<gram_partials_reduce_blocks(k), PR_THREADS, 0, s>>>(ws, ctas, KP, k, G, ldg, gate);
  return cudaGetLastError();
}

cudaError_t apply_gram_fused_launch(const double* X, int64_t ldx, int k, const double* Rinv_tiles, double* Q,
                                    int64_t ldq, int64_t rows, double* G, int ldg, double* ws, size_t ws_bytes,
                                    cudaStream_t stream, const int* gate) {
  (void)ws_bytes;
  if (fused_variant(k) == 1) {
    switch (rt_kp(k)) {
      case 16: return launch_rt<16, true>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream, gate);
      case 32: return launch_rt<32, true>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream, gate);
      case 64: return launch_rt<64, true>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream, gate);
      default: return cudaErrorNotSupported;
    }
  }
  if (fused_variant(k) == 2) return launch_fused<128>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream, gate);
  return cudaErrorNotSupported;
}

// ---- plain self Gram for k = 64 (K1): the register-resident sweep without the TRMM.
// Used for full 64-wide panels only: measured (tools/gram_probe.py) 4.27 ms vs
// 4.59 ms for the block-row pairs at m = 32M, k = 64, but slower for narrower
// or ragged widths, where the pass is HBM bound and the pairs kernel's
// dedicated producer warp streams better (k = 32: 0.48 vs 0.35 ms at 8M;
// k = 50: 1.50 vs 1.23 ms), and for short sweeps (m = 200k: 0.071 vs 0.058 ms).
bool gram_rt_supported(int k, int64_t rows) { return k == 64 && rows >= (int64_t(1) << 21); }
size_t gram_rt_ws_bytes(int64_t rows, int k) {
  return gram_rt_supported(k, rows) ? (size_t)rt_ctas(rows) * rt_kp(k) * rt_kp(k) * sizeof(double) + 256 : 0;
}
cudaError_t gram_rt_launch(const double* X, int64_t ldx, int k, int64_t rows, double* G, int ldg, double* ws,
                           cudaStream_t stream, const int* gate) {
  switch (rt_kp(k)) {
    case 16: return launch_rt<16, false>(X, ldx, k, nullptr, nullptr, 0, rows, G, ldg, ws, stream, gate);
    case 32: return launch_rt<32, false>(X, ldx, k, nullptr, nullptr, 0, rows, G, ldg, ws, stream, gate);
    case 64: return launch_rt<64, false>(X, ldx, k, nullptr, nullptr, 0, rows, G, ldg, ws, stream, gate);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace cqr
