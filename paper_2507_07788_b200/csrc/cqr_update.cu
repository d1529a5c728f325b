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
// Gram, and the copy of the basis); here Q_in is read from HBM once: per row
// panel (64 rows) its 64-column chunks go through a 3-stage bulk-copy ring
// for the projection, and again (now hitting L2) for the cross Gram against
// the updated block.  CTA = 8 warps; thread 0 issues the bulk copies.
//   projection : warp w owns row block w (8 rows) x 2 column blocks
//   R^-1 apply : the same, K = p
//   cross Gram : warp w owns column block w of every 64-column chunk of
//                Q_in (2 N blocks each), accumulated over the CTA's panels
//   block Gram : warps 0..2 own the 3 lower 8x8 blocks of the 16x16 G
// Per-CTA partials [Bt'(q x 16) | G'(16 x 16)] are summed by a fixed-order
// reduce kernel.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int UP_THREADS = 256;
constexpr int UP_BR = 64;                 // rows per panel (16 quads)
constexpr int UP_CH = 64;                 // Q_in columns per chunk
constexpr int UP_MAXQ = 512;
constexpr int UP_MAXCH = UP_MAXQ / UP_CH; // 8
constexpr int UP_STAGES = 3;
constexpr int UP_CHUNK = UP_BR * UP_CH;   // doubles per staged chunk (4096 = 32 KB)
constexpr int UP_PB = 16;                 // padded block width
constexpr int UP_BLD = UP_MAXQ + 4;       // Bt staging: [16][516] (516 = 4 mod 16)

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
  return ((size_t)UP_STAGES * UP_CHUNK + UP_BR * UP_PB + UP_PB * UP_BLD + UP_PB * CT_LD) * sizeof(double) + 64;
}

__global__ void __launch_bounds__(UP_THREADS, 1) update_pass_kernel(UpdateArgs a) {
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;                                   // UP_STAGES x [16 quads][64][4]
  double* blk = ring + UP_STAGES * UP_CHUNK;             // block panel [16 quads][16][4]
  double* bts = blk + UP_BR * UP_PB;                     // Bt as [n][k] (ld UP_BLD)
  double* ris = bts + UP_PB * UP_BLD;                    // R^-1 as [n][k] (ld 36)
  __shared__ __align__(8) uint64_t full[UP_STAGES], empty[UP_STAGES], bbar;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int q = a.q, p = a.p;
  const int nch = (q + UP_CH - 1) / UP_CH;
  const int64_t npan = ceil_div(a.rows, UP_BR);
  const bool init = a.initial != 0;

  if (tid == 0) {
    for (int s = 0; s < UP_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    mbar_init(&bbar, 1);
    fence_mbar_init();
  }
  // stage Bt (q x p) and R^-1 (p x p) once, zero padded to 16 columns
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

  // ring producer state (thread 0): sequence of (panel, pass, chunk) loads
  // pass 0 = projection stream (skipped in initial mode), pass 1 = cross Gram stream
  const int npass = init ? 1 : 2;
  const int per_panel = npass * nch;
  int64_t my_panels = 0;
  for (int64_t pp = blockIdx.x; pp < npan; pp += gridDim.x) ++my_panels;
  const int64_t total_loads = my_panels * per_panel;
  int64_t issued = 0;
  auto issue = [&](int64_t idx) {
    const int s = (int)(idx % UP_STAGES);
    const int64_t use = idx / UP_STAGES;
    if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
    const int64_t pl = idx / per_panel;
    const int ch = (int)(idx % per_panel) % nch;
    const int64_t pn = blockIdx.x + pl * gridDim.x;
    const int64_t r0 = pn * UP_BR;
    const int nq = (int)imin64(UP_BR, a.rows - r0) >> 2;
    const int c0 = ch * UP_CH, ncol = min(UP_CH, q - c0);
    double* dst = ring + s * UP_CHUNK;
    mbar_arrive_expect_tx(&full[s], (uint32_t)nq * ncol * 32);
    const double* src = a.Qin + (r0 >> 2) * 4 * a.ldqin + 4 * (int64_t)c0;
    for (int qq = 0; qq < nq; ++qq) bulk_g2s(dst + qq * UP_CH * 4, src + qq * 4 * a.ldqin, (uint32_t)ncol * 32, &full[s]);
  };
  if (tid == 0) {
    while (issued < total_loads && issued < UP_STAGES - 1) issue(issued++);
  }

  // accumulators
  double ct[UP_MAXCH][2][2];                // cross Gram: chunk c, column block w, N blocks 0/1
#pragma unroll
  for (int c = 0; c < UP_MAXCH; ++c)
#pragma unroll
    for (int n = 0; n < 2; ++n) { ct[c][n][0] = 0.0; ct[c][n][1] = 0.0; }
  double gq[2] = {0.0, 0.0};                // block Gram: warps 0..2

  int64_t consumed = 0;
  int bph = 0;
  for (int64_t pn = blockIdx.x; pn < npan; pn += gridDim.x) {
    const int64_t r0 = pn * UP_BR;
    const int nrows = (int)imin64(UP_BR, a.rows - r0);
    const int nq = nrows >> 2;
    // ---- block panel (64 x p) -> blk [quad][16][4], zero padded
    if (tid == 0) {
      mbar_arrive_expect_tx(&bbar, (uint32_t)nq * p * 32);
      const double* src = a.Qb + (r0 >> 2) * 4 * a.ldqb;
      for (int qq = 0; qq < nq; ++qq) bulk_g2s(blk + qq * UP_PB * 4, src + qq * 4 * a.ldqb, (uint32_t)p * 32, &bbar);
    }
    mbar_wait(&bbar, (uint32_t)(bph & 1));
    ++bph;
    // columns p..15 / rows >= nrows of blk hold stale data: mask at use
    double proj[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int row = 8 * warp + g;               // projection / TRMM row of this lane
    if (!init) {
      // ---- pass 0: proj(row block w) = Q_in(rows, :) Bt
      for (int ch = 0; ch < nch; ++ch, ++consumed) {
        if (tid == 0 && issued < total_loads) issue(issued++);
        const int s = (int)(consumed % UP_STAGES);
        mbar_wait(&full[s], (uint32_t)((consumed / UP_STAGES) & 1));
        const double* ck = ring + s * UP_CHUNK;
        const int c0 = ch * UP_CH, ncol = min(UP_CH, q - c0);
        const double* xa = ck + (row >> 2) * UP_CH * 4 + (row & 3);
        for (int ks = 0; ks < (ncol + 3) / 4; ++ks) {
          const int kc = 4 * ks + t;
          const double av = (kc < ncol) ? xa[4 * kc] : 0.0;
          const double b0 = bts[g * UP_BLD + c0 + kc];
          const double b1 = bts[(8 + g) * UP_BLD + c0 + kc];
          dmma(proj[0], av, b0);
          dmma(proj[1], av, b1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // ---- t = Q - proj, then Q' = t R^-1 (K = 16), written to HBM and to blk
      __syncthreads();   // every warp has read blk (none yet) -- keep ordering simple
      double tv[2][2];
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * n + 2 * t + e;
          const double x = (col < p && row < nrows) ? blk[(row >> 2) * UP_PB * 4 + 4 * col + (row & 3)] : 0.0;
          tv[n][e] = (col < p && row < nrows) ? x - proj[n][e] : 0.0;
        }
      __syncthreads();
      // stage t into blk for the A fragments of the R^-1 apply
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) blk[(row >> 2) * UP_PB * 4 + 4 * (8 * n + 2 * t + e) + (row & 3)] = tv[n][e];
      __syncthreads();
      double qn[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const double* ta = blk + (row >> 2) * UP_PB * 4 + (row & 3);
#pragma unroll
      for (int ks = 0; ks < UP_PB / 4; ++ks) {
        const int kc = 4 * ks + t;
        const double av = ta[4 * kc];
        dmma(qn[0], av, ris[g * CT_LD + kc]);
        dmma(qn[1], av, ris[(8 + g) * CT_LD + kc]);
      }
      __syncthreads();
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * n + 2 * t + e;
          const double v = (col < p && row < nrows) ? qn[n][e] : 0.0;
          blk[(row >> 2) * UP_PB * 4 + 4 * col + (row & 3)] = v;
          if (col < p && row < nrows) a.Qb[((r0 + row) >> 2) * 4 * a.ldqb + 4 * col + (row & 3)] = v;
        }
      __syncthreads();
    } else {
      // initial mode: zero the padding columns / rows of the staged block
      for (int e = tid; e < UP_BR * UP_PB; e += UP_THREADS) {
        const int qq = e / (UP_PB * 4), col = (e / 4) % UP_PB, rr = 4 * qq + (e & 3);
        if (col >= p || rr >= nrows) blk[e] = 0.0;
      }
      __syncthreads();
    }
    // ---- pass 1: cross Gram ct[ch] += Q_in(:, chunk)^T Q' and the block Gram
    const double* bq = blk + 4 * g + t;     // (column g, row t) of quad 0
    for (int ch = 0; ch < nch; ++ch, ++consumed) {
      if (tid == 0 && issued < total_loads) issue(issued++);
      const int s = (int)(consumed % UP_STAGES);
      mbar_wait(&full[s], (uint32_t)((consumed / UP_STAGES) & 1));
      const double* ck = ring + s * UP_CHUNK + 4 * (8 * warp + g) + t;   // (column 8w+g, row t)
      const int c0 = ch * UP_CH;
      const bool live = c0 + 8 * warp < q;
#pragma unroll
      for (int cc = 0; cc < UP_MAXCH; ++cc) {
        if (cc != ch) continue;
        if (live) {
          for (int ks = 0; ks < nq; ++ks) {
            const double av = ck[ks * UP_CH * 4];
            const double b0 = bq[ks * UP_PB * 4];
            const double b1 = bq[ks * UP_PB * 4 + 32];
            dmma(ct[cc][0], av, b0);
            dmma(ct[cc][1], av, b1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (warp < 3) {
      // lower blocks of G: (0,0), (1,0), (1,1)
      const int bi = (warp == 0) ? 0 : 1, bj = (warp == 2) ? 1 : 0;
      for (int ks = 0; ks < nq; ++ks) {
        const double av = bq[ks * UP_PB * 4 + 32 * bi];
        const double bv = bq[ks * UP_PB * 4 + 32 * bj];
        dmma(gq, av, bv);
      }
    }
    __syncthreads();   // blk is rewritten for the next panel
  }

  // ---- per-CTA partials: [Bt'(q_pad x 16) | G (16 x 16)] column-major with ld = q_pad + 16
  const int qp = nch * UP_CH;
  const int ld = qp + UP_PB;
  double* out = a.ws + (int64_t)blockIdx.x * ld * UP_PB;
#pragma unroll
  for (int cc = 0; cc < UP_MAXCH; ++cc) {
    if (cc >= nch) break;
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = cc * UP_CH + 8 * warp + g, c = 8 * n + 2 * t + e;
        out[(int64_t)c * ld + r] = ct[cc][n][e];
      }
  }
  if (warp < 3) {
    const int bi = (warp == 0) ? 0 : 1, bj = (warp == 2) ? 1 : 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) out[(int64_t)(8 * bj + 2 * t + e) * ld + qp + 8 * bi + g] = gq[e];
  } else if (warp == 3) {
    // upper block (0,1) of G is the mirror of (1,0): written by the reduce
#pragma unroll
    for (int e = 0; e < 2; ++e) out[(int64_t)(8 + 2 * t + e) * ld + qp + g] = 0.0;
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
  int64_t n = ceil_div(rows, UP_BR);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

bool update_pass_supported(int q, int p) { return q >= 1 && q <= UP_MAXQ && p >= 1 && p <= UP_PB; }

size_t update_pass_ws_bytes(int64_t rows, int q) {
  const int qp = (int)round_up(q, UP_CH);
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
  const int qp = (int)round_up(q, UP_CH);
  const int64_t nel = (int64_t)q * p + (int64_t)p * p;
  int blocks = (int)imin64(ceil_div(nel, 256), 2 * num_sms());
  update_reduce_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(ws, ctas, q, p, qp, Bt_next, q, G, ldg);
  return cudaGetLastError();
}

}  // namespace cqr
