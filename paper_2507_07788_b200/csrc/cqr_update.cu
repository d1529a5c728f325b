// K3: fused block-update pass (Alg. 2 inner loop), p <= 16 new columns.
//
// Replaces one outer iteration of `chol_qr_update` (reference
// algorithms.py:442-450):
//     proj = Q_in Bt; Q -= proj; Q = Q R^-1      (lincomb, axpy, lincomb)
//     Bt'  = Q_in^T Q; G' = Q^T Q                 (gramian(other), gramian)
// in one sweep over the rows, and (mode `initial`) the pass before the loop
// (algorithms.py:430-431): Bt = Q_in^T Q, G = Q^T Q.
//
// The reference streams Q_in three times per iteration (projection, cross
// Gram, and the copy of the basis); here Q_in is read from HBM once.  The
// rows are cut into 16-row sub-panels; a sub-panel of Q_in (4 quads x q
// columns, one bulk copy per quad) and of the block go through a 2-stage
// ring, and everything the iteration needs from those rows is done before
// the stage is released (work split per sub-panel: see the kernel).  CTA =
// 8 warps, persistent over sub-panels; thread 0 issues the bulk copies.
// Per-CTA partials [Bt'(q x 16) | G'(16 x 16)] are summed by a fixed-order
// reduce kernel.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int UP_THREADS = 256;
constexpr int UP_SR = 16;                 // rows per sub-panel (4 quads)
constexpr int UP_MAXQ = 512;
constexpr int UP_PB = 16;                 // padded block width
constexpr int UP_BLD = UP_MAXQ + 4;       // Bt staging: [16][516] (516 = 4 mod 16)
constexpr int UP_QIN = UP_SR * UP_MAXQ;   // doubles per staged Q_in sub-panel (64 KB)
constexpr int UP_QB = UP_SR * UP_PB;      // doubles per staged block sub-panel
constexpr int UP_STAGE = UP_QIN + UP_QB;
constexpr int UP_MAXCB = UP_MAXQ / 8 / 8; // column blocks of Bt' per warp (8)

struct UpdateArgs {
  const double* Qin; int64_t ldqin; int q;
  double* Qb; int64_t ldqb; int p;        // block (updated in place unless initial)
  int64_t rows;
  const double* Bt; int ldbt;             // q x p column-major (iteration mode)
  const double* Rinv;                     // p x p coefficient tiles (iteration mode)
  int initial;
  double* ws;                             // [ctas][(q_pad + 16) * 16]
};

static size_t update_smem_bytes() {
  return ((size_t)2 * UP_STAGE + UP_PB * UP_BLD + UP_PB * CT_LD + 8 * 256 + 2 * UP_QB) * sizeof(double) + 64;
}

// Per 16-row sub-panel (Q_in rows: 4 quads x q columns, staged with one bulk
// copy per quad; block rows: 4 quads x p):
//   proj = Q_in Bt          K = q split over the 8 warps, fixed-order reduce
//   t    = Q - proj         (iteration mode)
//   Q'   = t R^-1           warps 0..3 (2 x 2 blocks, K = 16) -> HBM + smem
//   Bt' += Q_in^T Q'        warp w owns Bt' row blocks w, w+8, ... (registers)
//   G   += Q'^T Q'          warps 0..2 (lower blocks)
// Q_in is read from HBM once per pass.
__global__ void __launch_bounds__(UP_THREADS, 1) update_pass_kernel(UpdateArgs a) {
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;                                   // 2 stages: [Q_in sub-panel | block sub-panel]
  double* bts = ring + 2 * UP_STAGE;                     // Bt as [n][k] (ld UP_BLD)
  double* ris = bts + UP_PB * UP_BLD;                    // R^-1 as [n][k] (ld 36)
  double* red = ris + UP_PB * CT_LD;                     // 8 warps x 256 projection partials
  double* tq = red + 8 * 256;                            // t (16 x 16, QI)
  double* qn = tq + UP_QB;                               // Q' (16 x 16, QI)
  __shared__ __align__(8) uint64_t full[2], empty[2];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int q = a.q, p = a.p;
  const int qs = (q + 3) & ~3;                           // staged column stride (quad = 4 qs doubles)
  const int nk4 = (q + 3) / 4;
  const int ncb = (q + 7) / 8;                           // Bt' row blocks
  const int64_t nsp = ceil_div(a.rows, UP_SR);
  const bool init = a.initial != 0;

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  if (!init) {
    for (int e = tid; e < UP_PB * UP_BLD; e += UP_THREADS) {
      const int n = e / UP_BLD, kk = e % UP_BLD;
      bts[e] = (n < p && kk < q) ? a.Bt[(int64_t)n * a.ldbt + kk] : 0.0;
    }
    for (int e = tid; e < UP_PB * CT_LD; e += UP_THREADS) {
      const int n = e / CT_LD, kk = e % CT_LD;
      ris[e] = (n < p && kk < p) ? a.Rinv[coeff_off(kk, n, p)] : 0.0;
    }
  }
  __syncthreads();

  auto issue = [&](int64_t sp, int st) {
    const int64_t r0 = sp * UP_SR;
    const int nq = (int)imin64(UP_SR, a.rows - r0) >> 2;
    double* dq = ring + st * UP_STAGE;
    double* db = dq + UP_QIN;
    mbar_arrive_expect_tx(&full[st], (uint32_t)nq * (q + p) * 32);
    const double* sq = a.Qin + (r0 >> 2) * 4 * a.ldqin;
    const double* sb = a.Qb + (r0 >> 2) * 4 * a.ldqb;
    for (int qq = 0; qq < nq; ++qq) {
      bulk_g2s(dq + qq * 4 * qs, sq + qq * 4 * a.ldqin, (uint32_t)q * 32, &full[st]);
      bulk_g2s(db + qq * 4 * UP_PB, sb + qq * 4 * a.ldqb, (uint32_t)p * 32, &full[st]);
    }
  };
  if (tid == 0 && blockIdx.x < nsp) issue(blockIdx.x, 0);

  double ct[UP_MAXCB][2][2];
#pragma unroll
  for (int i = 0; i < UP_MAXCB; ++i)
#pragma unroll
    for (int n = 0; n < 2; ++n) { ct[i][n][0] = 0.0; ct[i][n][1] = 0.0; }
  double gq[2] = {0.0, 0.0};

  int it = 0;
  for (int64_t sp = blockIdx.x; sp < nsp; sp += gridDim.x, ++it) {
    const int s = it & 1;
    if (tid == 0 && sp + gridDim.x < nsp) {
      if (it >= 1) mbar_wait(&empty[s ^ 1], ((it - 1) >> 1) & 1);
      issue(sp + gridDim.x, s ^ 1);
    }
    mbar_wait(&full[s], (it >> 1) & 1);
    const int64_t r0 = sp * UP_SR;
    const int nrows = (int)imin64(UP_SR, a.rows - r0);
    const double* Qs = ring + s * UP_STAGE;   // [quad][qs][4]
    const double* Bs = Qs + UP_QIN;           // [quad][16][4], columns >= p stale
    const double* src;                        // Q' (or Q in initial mode) as [quad][16][4]
    if (!init) {
      // ---- proj partial: warp w takes k4 steps [w*c, (w+1)*c)
      const int chunk = (nk4 + 7) / 8;
      const int ks0 = warp * chunk, ks1 = min(nk4, ks0 + chunk);
      double pr[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
      for (int ks = ks0; ks < ks1; ++ks) {
        const int kc = 4 * ks + t;
        double av[2];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int row = 8 * rb + g;
          av[rb] = (kc < q) ? Qs[(row >> 2) * 4 * qs + 4 * kc + (row & 3)] : 0.0;
        }
        const double b0 = bts[g * UP_BLD + kc], b1 = bts[(8 + g) * UP_BLD + kc];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          dmma(pr[rb][0], av[rb], b0);
          dmma(pr[rb][1], av[rb], b1);
        }
      }
      // partials -> red[w][(col)*16 + row]
#pragma unroll
      for (int rb = 0; rb < 2; ++rb)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e) red[warp * 256 + (8 * nb + 2 * t + e) * 16 + 8 * rb + g] = pr[rb][nb][e];
      __syncthreads();
      {
        // thread e: proj(row, col) = sum over warps (fixed order); t = Q - proj
        const int row = tid & 15, col = tid >> 4;
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += red[w * 256 + col * 16 + row];
        const bool v = row < nrows && col < p;
        const double x = v ? Bs[(row >> 2) * 4 * UP_PB + 4 * col + (row & 3)] : 0.0;
        tq[(row >> 2) * 4 * UP_PB + 4 * col + (row & 3)] = v ? x - sum : 0.0;
      }
      __syncthreads();
      // ---- Q' = t R^-1: warps 0..3, block (rb = w >> 1, nb = w & 1)
      if (warp < 4) {
        const int rb = warp >> 1, nb = warp & 1;
        const int row = 8 * rb + g;
        double c2[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < UP_PB / 4; ++ks) {
          const int kc = 4 * ks + t;
          dmma(c2, tq[(row >> 2) * 4 * UP_PB + 4 * kc + (row & 3)], ris[(8 * nb + g) * CT_LD + kc]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * nb + 2 * t + e;
          const bool v = row < nrows && col < p;
          qn[(row >> 2) * 4 * UP_PB + 4 * col + (row & 3)] = v ? c2[e] : 0.0;
          if (v) a.Qb[((r0 + row) >> 2) * 4 * a.ldqb + 4 * col + (row & 3)] = c2[e];
        }
      }
      __syncthreads();
      src = qn;
    } else {
      // initial mode: Q' = Q; zero its stale padding columns / rows in a copy
      {
        const int row = tid & 15, col = tid >> 4;
        const bool v = row < nrows && col < p;
        qn[(row >> 2) * 4 * UP_PB + 4 * col + (row & 3)] = v ? Bs[(row >> 2) * 4 * UP_PB + 4 * col + (row & 3)] : 0.0;
      }
      __syncthreads();
      src = qn;
    }
    // ---- Bt' += Q_in^T Q' (K = 16 rows); warp w: Bt' row blocks cb = w + 8 i
    {
      const double* bq = src + 4 * g + t;   // (column g, row t) of quad 0
      const int nq = nrows >> 2;
#pragma unroll
      for (int i = 0; i < UP_MAXCB; ++i) {
        const int cb = warp + 8 * i;
        if (cb < ncb) {
          const double* xa = Qs + 4 * (8 * cb + g) + t;
          for (int ks = 0; ks < nq; ++ks) {
            const double av = xa[ks * 4 * qs];
            dmma(ct[i][0], av, bq[ks * 4 * UP_PB]);
            dmma(ct[i][1], av, bq[ks * 4 * UP_PB + 32]);
          }
        }
      }
      if (warp < 3) {
        const int bi = (warp == 0) ? 0 : 1, bj = (warp == 2) ? 1 : 0;
        for (int ks = 0; ks < nq; ++ks) dmma(gq, bq[ks * 4 * UP_PB + 32 * bi], bq[ks * 4 * UP_PB + 32 * bj]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    __syncthreads();   // qn / tq / red are rewritten by the next sub-panel
  }

  // ---- per-CTA partials: [Bt'(q_pad x 16) | G (16 x 16)] column-major with ld = q_pad + 16
  const int qp = (int)round_up(q, 64);
  const int ld = qp + UP_PB;
  double* out = a.ws + (int64_t)blockIdx.x * ld * UP_PB;
#pragma unroll
  for (int i = 0; i < UP_MAXCB; ++i) {
    const int cb = warp + 8 * i;
    if (cb >= ncb) continue;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) out[(int64_t)(8 * n + 2 * t + e) * ld + 8 * cb + g] = ct[i][n][e];
  }
  if (warp < 3) {
    const int bi = (warp == 0) ? 0 : 1, bj = (warp == 2) ? 1 : 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) out[(int64_t)(8 * bj + 2 * t + e) * ld + qp + 8 * bi + g] = gq[e];
  }
}

// fixed-order sum over CTAs; Bt' (q x p, ld ldbt) and G (p x p, lower mirrored, ld ldg)
__global__ void update_reduce_kernel(const double* __restrict__ ws, int nparts, int q, int p, int qp,
                                     double* Bt, int ldbt, double* G, int ldg) {
  const int ld = qp + UP_PB;
  const int64_t nbt = (int64_t)q * p, ng = (int64_t)p * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nbt + ng;
       e += (int64_t)gridDim.x * blockDim.x) {
    int r, c;
    int64_t off;
    if (e < nbt) { r = (int)(e % q); c = (int)(e / q); off = (int64_t)c * ld + r; }
    else {
      const int64_t f = e - nbt;
      r = (int)(f % p); c = (int)(f / p);
      if (r < c) continue;
      off = (int64_t)c * ld + qp + r;
    }
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += ws[(int64_t)i * ld * UP_PB + off];
    if (e < nbt) Bt[(int64_t)c * ldbt + r] = s;
    else { G[(int64_t)c * ldg + r] = s; G[(int64_t)r * ldg + c] = s; }
  }
}

static int update_ctas(int64_t rows) {
  int64_t n = ceil_div(rows, UP_SR);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

bool update_pass_supported(int q, int p) { return q >= 1 && q <= UP_MAXQ && p >= 1 && p <= UP_PB; }

size_t update_pass_ws_bytes(int64_t rows, int q) {
  const int qp = (int)round_up(q, 64);
  return (size_t)update_ctas(rows) * (qp + UP_PB) * UP_PB * sizeof(double) + 256;
}

cudaError_t update_pass_launch(const double* Qin, int64_t ldqin, int q, double* Qb, int64_t ldqb, int p,
                               int64_t rows, const double* Bt, int ldbt, const double* Rinv_tiles, int initial,
                               double* Bt_next, double* G, int ldg, double* ws, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = update_smem_bytes();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(update_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  UpdateArgs a{};
  a.Qin = Qin; a.ldqin = ldqin; a.q = q;
  a.Qb = Qb; a.ldqb = ldqb; a.p = p;
  a.rows = rows;
  a.Bt = Bt; a.ldbt = ldbt; a.Rinv = Rinv_tiles;
  a.initial = initial;
  a.ws = ws;
  const int ctas = update_ctas(rows);
  update_pass_kernel<<<ctas, UP_THREADS, smem, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int qp = (int)round_up(q, 64);
  const int64_t nel = (int64_t)q * p + (int64_t)p * p;
  int blocks = (int)imin64(ceil_div(nel, 256), 2 * num_sms());
  update_reduce_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(ws, ctas, q, p, qp, Bt_next, q, G, ldg);
  return cudaGetLastError();
}

}  // namespace cqr
