// K2 fused pass for k <= 128: Q = X R^-1 (R^-1 upper triangular) and
// G = Q^T Q in one stream over X (Q may alias X).
//
// Replaces the lincomb + gramian pair of one iteration (reference
// algorithms.py:350,352 / :238,:240 / :211 + chol_qr2's second Gram) with one
// HBM read of X and one write of Q per pass (the unfused pair reads Q again).
//
// CTA = 8 consumer warps + 1 producer warp, persistent over row panels of BR
// rows (one wave, one CTA per SM).  At start the CTA loads the R^-1
// coefficient tiles it needs (upper part only) into shared memory.  Per
// panel: the producer stages X (QI layout: one run per quad) into a 2-stage
// ring; the consumers
//   1. compute the Q panel with DMMA -- warp w owns a row group and the
//      column-block pair (c, NC-1-c), so every warp gets the same triangular
//      work -- and store it to HBM straight from registers;
//   2. after a CTA barrier overwrite the staged X with Q (QI layout) and
//      accumulate the lower-triangular Gram from it (32x32 register
//      sub-tiles, diagonal ones skipping upper blocks, shared sub-tiles split
//      over k4 steps);
//   3. release the stage.
// Partials are summed inside the CTA in a fixed warp order and written once
// per CTA; gram_fused_reduce sums them over CTAs in a fixed order.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int FU_THREADS = 256;   // 8 warps; thread 0 also issues the bulk copies

template <int KP>
struct FusedCfg {
  static constexpr int NC = KP / 8;                       // 8-column blocks
  static constexpr int BR = (KP >= 128) ? 32 : 64;        // rows per panel
  static constexpr int NR = BR / 8;                       // 8-row blocks per panel
  static constexpr int PAIRS = NC / 2;                    // column-block pairs
  static constexpr int RGROUPS = 8 / PAIRS;               // row groups (warps = RGROUPS * PAIRS)
  static constexpr int RB = NR / RGROUPS;                 // row blocks per warp
  static constexpr int STAGE = BR * KP;                   // doubles per staged panel
  static constexpr int NKT = KP / CT_K;                   // coefficient k tiles
  static constexpr int NNT = (KP + CT_N - 1) / CT_N;      // coefficient n tiles
  static constexpr int T = KP / 32;                       // 32x32 Gram sub-tiles per side
};

// coefficient tiles of R^-1 needed (kt*32 < (nt+1)*64), in order; index -> slot
template <int KP>
__device__ __forceinline__ int tile_slot(int kt, int nt) {
  int slot = 0;
  for (int n = 0; n < nt; ++n) slot += min(FusedCfg<KP>::NKT, 2 * (n + 1));
  return slot + kt;
}
template <int KP>
__host__ __device__ constexpr int n_tiles_needed() {
  int s = 0;
  for (int n = 0; n < FusedCfg<KP>::NNT; ++n) s += (FusedCfg<KP>::NKT < 2 * (n + 1)) ? FusedCfg<KP>::NKT : 2 * (n + 1);
  return s;
}

template <int KP>
__host__ __device__ constexpr size_t fused_smem_doubles() {
  return ((size_t)n_tiles_needed<KP>() * CT_TILE + 2 * FusedCfg<KP>::STAGE) > (size_t)KP * KP
             ? (size_t)n_tiles_needed<KP>() * CT_TILE + 2 * FusedCfg<KP>::STAGE
             : (size_t)KP * KP;
}

// Gram work of warp w: (sub-tile i, j, diag, k4 start, k4 stride)
template <int KP>
__device__ __forceinline__ void gram_role(int w, int& si, int& sj, int& k0, int& kst) {
  if constexpr (KP == 128) {
    // 6 off-diagonal sub-tiles (warps 0-5), 4 diagonal ones in pairs (warps 6, 7)
    // off sub-tiles (1,0) (2,0) (3,0) (2,1) (3,1) (3,2) for warps 0..5
    if (w < 6) {
      si = (w < 3) ? w + 1 : (w < 5 ? w - 1 : 3);
      sj = (w < 3) ? 0 : (w < 5 ? 1 : 2);
    } else {
      si = sj = (w - 6) * 2;   // and si + 1
    }
    k0 = 0; kst = 1;
  } else if constexpr (KP == 64) {
    // off (1,0) over warps 0-3 (k4 mod 4), diag (0,0) over 4-5, diag (1,1) over 6-7 (k4 mod 2)
    if (w < 4) { si = 1; sj = 0; k0 = w; kst = 4; }
    else if (w < 6) { si = sj = 0; k0 = w - 4; kst = 2; }
    else { si = sj = 1; k0 = w - 6; kst = 2; }
  } else {
    si = sj = 0; k0 = w; kst = 8;
  }
}

template <int KP>
__global__ void __launch_bounds__(FU_THREADS, 1) apply_gram_fused_kernel(const double* X, int64_t ldx,
                                                                          int k, const double* __restrict__ Rt,
                                                                          double* Q, int64_t ldq, int64_t rows,
                                                                          double* __restrict__ ws) {
  using C = FusedCfg<KP>;
  extern __shared__ __align__(128) double smem[];
  double* rt_s = smem;                                        // R^-1 tiles
  double* stg = rt_s + n_tiles_needed<KP>() * CT_TILE;        // 2 x STAGE
  double* red = smem;   // KP x KP partial Gram (column-major), reuses tiles + stages after the loop
  __shared__ __align__(8) uint64_t bars[6];
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  uint64_t* rbar = bars + 4;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t npan = ceil_div(rows, C::BR);

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  (void)lane;

  // bulk-copy issue (thread 0): R^-1 tiles once, X panels one ahead
  auto issue_panel = [&](int64_t p, int st) {
    const int64_t r0 = p * C::BR;
    const int nq = (int)imin64(C::BR, rows - r0) >> 2;
    double* dst = stg + st * C::STAGE;
    mbar_arrive_expect_tx(&full[st], (uint32_t)nq * k * 32);
    const double* src = X + (r0 >> 2) * 4 * ldx;
    if (ldx == KP && k == KP) {
      bulk_g2s(dst, src, (uint32_t)nq * KP * 32, &full[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s(dst + q * 4 * KP, src + q * 4 * ldx, (uint32_t)k * 32, &full[st]);
    }
  };
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(rbar, n_tiles_needed<KP>() * CT_TILE * 8);
    for (int nt = 0; nt < C::NNT; ++nt)
      for (int kt = 0; kt < min(C::NKT, 2 * (nt + 1)); ++kt)
        bulk_g2s(rt_s + tile_slot<KP>(kt, nt) * CT_TILE, Rt + ((int64_t)nt * C::NKT + kt) * CT_TILE, CT_TILE * 8,
                 rbar);
    if (blockIdx.x < npan) issue_panel(blockIdx.x, 0);
  }

  // ---------------- consumers
  // TRMM role: row blocks [rg*RB, rg*RB + RB), column blocks cA = pair, cB = NC-1-pair
  const int pair = warp % C::PAIRS, rg = warp / C::PAIRS;
  const int cA = pair, cB = C::NC - 1 - pair;
  int si, sj, k0, kst;
  gram_role<KP>(warp, si, sj, k0, kst);
  const bool dg = (si == sj);

  constexpr int NX = (KP == 128) ? 2 : 1;   // KP = 128: the diagonal warps own two sub-tiles
  double gacc[NX][4][4][2];
#pragma unroll
  for (int x = 0; x < NX; ++x)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) { gacc[x][i][j][0] = 0.0; gacc[x][i][j][1] = 0.0; }

  mbar_wait(rbar, 0);
  int it = 0;
  for (int64_t p = blockIdx.x; p < npan; p += gridDim.x, ++it) {
    const int s = it & 1;
    if (threadIdx.x == 0 && p + gridDim.x < npan) {
      // stage s^1 held panel it-1: wait until every warp released it, then refill
      if (it >= 1) mbar_wait(&empty[s ^ 1], ((it - 1) >> 1) & 1);
      issue_panel(p + gridDim.x, s ^ 1);
    }
    mbar_wait(&full[s], (it >> 1) & 1);
    const int64_t r0 = p * C::BR;
    const int nrows = (int)imin64(C::BR, rows - r0);
    double* P = stg + s * C::STAGE;

    // ---- 1. TRMM: qacc[rb][cb] for rb < RB, cb in {cA, cB}
    double qacc[C::RB][2][2];
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb)
#pragma unroll
      for (int c = 0; c < 2; ++c) { qacc[rb][c][0] = 0.0; qacc[rb][c][1] = 0.0; }
    // K loop over k4 steps; column block c needs K < 8(c+1)
    const int kmaxB = min(2 * (cB + 1), (k + 3) / 4);
    const int kmaxA = min(2 * (cA + 1), (k + 3) / 4);
    for (int ks = 0; ks < kmaxB; ++ks) {
      const int kc = 4 * ks + t;   // X column of this lane's A fragment
      double a[C::RB];
#pragma unroll
      for (int rb = 0; rb < C::RB; ++rb) {
        const int row = 8 * (rg * C::RB + rb) + g;
        a[rb] = (kc < k) ? P[(row >> 2) * 4 * KP + 4 * kc + (row & 3)] : 0.0;
      }
      // B fragment: R^-1(kc, 8 cb + g) from tile (kc/32, (8cb+g)/64)
      const int nB = 8 * cB + g;
      const double bB = rt_s[tile_slot<KP>(kc >> 5, nB >> 6) * CT_TILE + (nB & 63) * CT_LD + (kc & 31)];
#pragma unroll
      for (int rb = 0; rb < C::RB; ++rb) dmma(qacc[rb][1], a[rb], bB);
      if (ks < kmaxA) {
        const int nA = 8 * cA + g;
        const double bA = rt_s[tile_slot<KP>(kc >> 5, nA >> 6) * CT_TILE + (nA & 63) * CT_LD + (kc & 31)];
#pragma unroll
        for (int rb = 0; rb < C::RB; ++rb) dmma(qacc[rb][0], a[rb], bA);
      }
    }
    // store Q to HBM (QI) straight from registers
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) {
      const int row = 8 * (rg * C::RB + rb) + g;
      if (row < nrows) {
        double* qrow = Q + ((r0 + row) >> 2) * 4 * ldq + (row & 3);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * (c ? cB : cA) + 2 * t + e;
            if (col < k) qrow[4 * (int64_t)col] = qacc[rb][c][e];
          }
      }
    }
    // ---- 2. overwrite the staged X with Q, then the Gram
    asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
    for (int rb = 0; rb < C::RB; ++rb) {
      const int row = 8 * (rg * C::RB + rb) + g;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * (c ? cB : cA) + 2 * t + e;
          P[(row >> 2) * 4 * KP + 4 * col + (row & 3)] = (row < nrows && col < k) ? qacc[rb][c][e] : 0.0;
        }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    {
      const int nk4 = nrows >> 2;
      const double* base = P + 4 * g + t;   // (column g, row t) inside quad 0
      for (int ks = k0; ks < nk4; ks += kst) {
        const double* qd = base + ks * 4 * KP;
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = qd[4 * (32 * si + 8 * i)];
        if (dg) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) dmma(gacc[0][i][j], a[i], a[j]);
          if constexpr (NX == 2) {
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = qd[4 * (32 * (si + 1) + 8 * i)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j <= i; ++j) dmma(gacc[NX - 1][i][j], b[i], b[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = qd[4 * (32 * sj + 8 * j)];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(gacc[0][i][j], a[i], b[j]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- CTA reduction of the Gram partials into red (KP x KP column-major), fixed warp order
  asm volatile("bar.sync 1, 256;" ::: "memory");   // every warp is done with the tiles and stages
  for (int e = threadIdx.x; e < KP * KP; e += 256) red[e] = 0.0;
  asm volatile("bar.sync 1, 256;" ::: "memory");
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int x = 0; x < NX; ++x) {
        if (x == 1 && !dg) break;
        const int ti = si + x, tj = sj + x;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = 32 * ti + 8 * i + g, c = 32 * tj + 8 * j + 2 * t + e;
              if (!dg || i >= j) red[c * KP + r] += gacc[x][i][j][e];
            }
      }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
  double* out = ws + (int64_t)blockIdx.x * KP * KP;
  for (int e = threadIdx.x; e < KP * KP; e += 256) out[e] = red[e];
}

// fixed-order sum over CTAs of the per-CTA KP x KP partials; lower triangle, mirrored
__global__ void gram_fused_reduce(const double* __restrict__ ws, int nparts, int KP, int k, double* G, int ldg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), c = (int)(e / k);
    if (r < c) continue;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += ws[(int64_t)p * KP * KP + c * KP + r];
    G[(int64_t)c * ldg + r] = s;
    G[(int64_t)r * ldg + c] = s;
  }
}

static int fused_kp(int k) {
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  if (k > 96 && k <= 128) return 128;
  return 0;   // 65..96: unfused path
}

// Off by default: measured slower than TRMM + Gram on B200 in round 1 (two CTA
// barriers per panel keep the 8 warps in lockstep).  Enabled
// with cqr_set_fused(1) (tests exercise it).
static int g_fused_enabled = 0;
void set_fused(int on) { g_fused_enabled = on ? 1 : 0; }
bool apply_gram_fused_supported(int k) { return g_fused_enabled && k >= 1 && fused_kp(k) != 0; }

static int fused_ctas(int64_t rows, int kp) {
  const int br = (kp >= 128) ? 32 : 64;
  int64_t n = ceil_div(rows, br);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

size_t apply_gram_fused_ws_bytes(int64_t rows, int k) {
  const int kp = fused_kp(k);
  if (!kp) return 0;
  return (size_t)fused_ctas(rows, kp) * kp * kp * sizeof(double) + 256;
}

template <int KP>
static cudaError_t launch_fused(const double* X, int64_t ldx, int k, const double* Rt, double* Q, int64_t ldq,
                                int64_t rows, double* G, int ldg, double* ws, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = fused_smem_doubles<KP>() * sizeof(double);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(apply_gram_fused_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ctas = fused_ctas(rows, KP);
  apply_gram_fused_kernel<KP><<<ctas, FU_THREADS, smem, s>>>(X, ldx, k, Rt, Q, ldq, rows, ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t nel = (int64_t)k * k;
  int blocks = (int)imin64(ceil_div(nel, 256), 2 * num_sms());
  gram_fused_reduce<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(ws, ctas, KP, k, G, ldg);
  return cudaGetLastError();
}

cudaError_t apply_gram_fused_launch(const double* X, int64_t ldx, int k, const double* Rinv_tiles, double* Q,
                                    int64_t ldq, int64_t rows, double* G, int ldg, double* ws, size_t ws_bytes,
                                    cudaStream_t stream) {
  (void)ws_bytes;
  switch (fused_kp(k)) {
    case 32: return launch_fused<32>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream);
    case 64: return launch_fused<64>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream);
    case 128: return launch_fused<128>(X, ldx, k, Rinv_tiles, Q, ldq, rows, G, ldg, ws, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace cqr
