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
// Gram, and the copy of the basis); here Q_in is read from HBM once.  Rows go
// in 16-row sub-panels through a TMA ring (Q_in: 4 quads x q columns, block:
// 4 quads x p), one CTA per SM, persistent.  The CTA is warp-specialised:
//   * 8 projection warps: warp w owns the column slices [64c + 8w, +8) of
//     Q_in (its Bt rows live in registers): proj partial = Q_in Bt over its
//     slices, fixed-order sum of the 8 partials in shared memory, t = Q - proj,
//     Q' = t R^-1 (warps 0-3, one 8x8 block each), Q' -> HBM (in place) and
//     into a 2-slot ring of Q' sub-panels;
//   * 8 cross-Gram warps: warp w owns the same slices as rows of Bt':
//     Bt' += Q_in^T Q' in registers over the sweep, G += Q'^T Q' (warps 8-10);
//     they release the stage, and the last one's lane 0 refills it.
// Both groups issue q/8 DMMA per warp per 16 rows; the width enters as the
// template parameter NQ = ceil(q/64) so no DMMA is predicated off.  Bases up to
// 144 columns use 32-row sub-panels (half the per-row synchronisation).  Groups hand
// over through mbarriers; the projection group syncs on a named barrier.
// Per-CTA partials [Bt'(q_pad x 16) | G'(16 x 16)] are written once per CTA
// and summed by a fixed-order reduce kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int UP_MAXQ = 512;
constexpr int UP_PB = 16;                 // padded block width
constexpr int UP_THREADS = 512;           // 8 projection + 8 cross-Gram warps
constexpr int UP_YS = 4;                  // Q' ring slots
constexpr int UP_MAXNS = 8;               // TMA ring stages (at most)

// SR = rows per sub-panel (16 or 32): 32 halves the per-row cost of the
// projection group's barriers and reduction, used where the stage still
// leaves room for a deep ring (narrow bases).
// (the narrow path -- bases up to 64 columns -- has no projection partials;
// the two-team path has two t buffers)
__host__ __device__ constexpr int up_fixed(int SR, bool narrow = false, bool teams = false) {   // doubles before the ring
  return UP_PB * CT_LD + (narrow ? 0 : 8 * SR * UP_PB) + (teams ? 2 : 1) * SR * UP_PB + UP_YS * SR * UP_PB;
}

// A sub-panel of a QI array with column capacity ldk is SR/4 runs of 4q
// doubles, 32*ldk bytes apart.  As separate cp.async.bulk copies these are
// small (512 B per row quad at q = 16) and a copy costs ~110 cycles of issue on
// one SM (profiles/r01_bulk_pieces.jsonl: 512-B pieces stream at 1.4 TB/s,
// 8 KB pieces at 6.5 TB/s), so narrow passes stage through a 3-D TMA tensor
// map instead -- dims {4 (row in quad), ldk, quads}, box {4, qs, SR/4}: ONE
// cp.async.bulk.tensor per sub-panel, landing exactly in the padded stage
// layout (columns past the capacity and quads past the end are zero-filled).
struct alignas(64) UpdateArgs {
  CUtensorMap tm_qin;                     // valid when use_tm_qin
  CUtensorMap tm_qb;                      // valid when use_tm_qb
  int use_tm_qin, use_tm_qb;
  const double* Qin; int64_t ldqin; int q;
  const double* Qb; int64_t ldqb; int p;  // block read by the pass
  double* Qo; int64_t ldqo;               // where Q' goes (iteration mode; may be Qb)
  int64_t rows;                           // multiple of 16
  const double* Bt; int ldbt;             // p x q as [n][k] (iteration mode)
  const double* Rinv;                     // p x p coefficient tiles (iteration mode)
  int initial;
  double* ws;                             // [ctas][(q_pad + 16) * 16]
  int qs;                                 // staged column stride (= 4 mod 8)
  int ns;                                 // ring stages
  const int* gate;                        // no-op unless *gate == CQR_FACTORED
  int lag;                                // cross-Gram group one sub-panel behind the projection DMMAs (see kernel)
  int direct;                             // initial mode: the cross-Gram warps read the block from the stage (see kernel)
};

static int up_qs(int q) { return (int)round_up(q, 8) + 4; }
// 64-row sub-panels for bases up to 64 columns: the narrow pass is bound by the
// per-sub-panel chain (projection -> t -> R^-1 -> hand-over), so twice the rows
// per chain halve its cost per row (q = 16 at 8M rows: 1.45 -> see DESIGN)
static int g_sr16_from = 145;   // cqr_debug_update_sr16_from: bases from this width use 16-row sub-panels
static int up_sr(int q) { return q <= 64 ? 64 : (q < g_sr16_from ? 32 : 16); }
static bool up_narrow(int q) { return q <= 64; }
static int up_stage(int q, int sr) { return sr * up_qs(q) + sr * UP_PB; }
static int up_stages_with(int q, int sr, bool teams) {
  const int64_t avail = 227 * 1024 - 512 - (int64_t)up_fixed(sr, up_narrow(q), teams) * 8;
  int64_t ns = avail / ((int64_t)up_stage(q, sr) * 8);
  if (ns > UP_MAXNS) ns = UP_MAXNS;
  // Two projection teams take alternate sub-panels, so each must see every
  // phase of the stages it waits on: an even stage count keeps each stage with
  // one team (with an odd count a team would skip a phase of a stage and read
  // it a phase early through the parity wait).
  if (teams) ns &= ~int64_t(1);
  return (int)ns;
}
// Two projection teams where they fit with four stages (65 <= q <= 144 at 32-row
// sub-panels): with two stages the teams starve (q = 160: 3.63 -> 4.58 ms).
static int g_narrow_teams = 1;   // cqr_debug_update_narrow_teams
static bool up_teams_q(int q, int sr) {
  const int nq = (q + 63) / 64;
  if (sr == 64 && nq == 1) return g_narrow_teams && up_stages_with(q, sr, true) >= 4;   // the narrow path
  return sr == 32 && (nq == 2 || nq == 3) && up_stages_with(q, sr, true) >= 4;
}
static int up_stages(int q, int sr) { return up_stages_with(q, sr, up_teams_q(q, sr)); }
static size_t update_smem_bytes(int q, int sr) {
  return ((size_t)up_fixed(sr, up_narrow(q), up_teams_q(q, sr)) + (size_t)up_stages(q, sr) * up_stage(q, sr)) * 8;
}

// PART: the last 64-column block is partial (q % 64 != 0, NQ >= 2): its work
// is split by k4 step (projection) and by output block (cross Gram) so that it
// spreads over the four SM sub-partitions and the part past q is skipped.
template <int NQ, int SR, bool PART, bool TEAMS>
__global__ void __launch_bounds__(UP_THREADS, 1) update_pass_kernel(const __grid_constant__ UpdateArgs a) {
  if (a.gate != nullptr && *a.gate != 0) return;   // gated off
  constexpr int RB = SR / 8;        // 8-row blocks per sub-panel
  constexpr int Q4 = SR / 4;        // quads (k4 steps of the cross Gram) per sub-panel
  constexpr int TE = SR * UP_PB;    // elements of a 16-wide sub-panel
  extern __shared__ __align__(128) double smem[];
  const int q = a.q, p = a.p, qs = a.qs, ns = a.ns;
  const int STG = SR * qs + SR * UP_PB;
  constexpr bool NARROW = NQ == 1 && SR >= 32;   // bases up to 64 columns
  // 65 <= q <= 144: two independent projection teams of 4 warps take alternate
  // sub-panels, so one team's reduction / R^-1 / hand-over overlaps the other
  // team's DMMAs (one team of 8 left the cross-Gram warps waiting on Q')
  double* ris = smem;                      // R^-1 as [n][k] (ld 36)
  double* red = ris + UP_PB * CT_LD;       // 8 projection partials (QI, SR x 16); none on the narrow path
  double* tq = red + (NARROW ? 0 : 8 * TE);   // t = Q - proj (QI, SR x 16), one per team
  double* yring = tq + (TEAMS ? 2 : 1) * TE;  // UP_YS x Q' (QI, SR x 16)
  double* stg = yring + UP_YS * TE;        // ns x [Q_in sub-panel (Q4 quads x qs x 4) | block (Q4 quads x 16 x 4)]
  __shared__ __align__(8) uint64_t full[UP_MAXNS], empty[UP_MAXNS], yfull[UP_YS], yempty[UP_YS], pdone[UP_YS];
  // Lag (single projection group, iteration mode): the cross-Gram group starts
  // sub-panel j only once the projection DMMAs of j+1 are issued (pdone), so
  // its DMMAs run during the projection group's serial tail (partials ->
  // fixed-order sum -> R^-1 -> hand-over), when the FP64 pipe is otherwise
  // idle (ncu at q = 320: the cross-Gram warps waited on Q' for 23% of their
  // samples).  Timing only: the same operations in the same order per element.
  const bool lag = a.lag != 0 && !TEAMS && a.initial == 0;
  // Direct (initial mode, full 16-column blocks, rows a multiple of SR): Q' is the
  // staged block itself, so the cross-Gram warps wait for the stage and read it in
  // place; the projection group's copy into the Q' ring and its hand-over (a
  // latency chain per sub-panel that bounds the narrow initial passes) are skipped.
  const bool direct = a.direct != 0 && a.initial != 0;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool init = a.initial != 0;
  const int64_t nsp = ceil_div(a.rows, SR);
  const int64_t mine = (nsp > blockIdx.x) ? ceil_div(nsp - blockIdx.x, gridDim.x) : 0;

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    for (int s = 0; s < UP_YS; ++s) {
      mbar_init(&yfull[s], TEAMS ? 128 : 256); mbar_init(&yempty[s], 8); mbar_init(&pdone[s], 8);
    }
    fence_mbar_init();
  }
  if (!init) {
    for (int e = tid; e < UP_PB * CT_LD; e += UP_THREADS) {
      const int n = e / CT_LD, kk = e % CT_LD;
      ris[e] = (n < p && kk < p) ? a.Rinv[coeff_off(kk, n, p)] : 0.0;
    }
  }
  __syncthreads();

  auto issue = [&](int64_t j, int st) {
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * SR;
    const int nq = (int)imin64(SR, a.rows - r0) >> 2;
    double* dq = stg + st * STG;
    double* db = dq + SR * qs;
    // a tensor copy always delivers the whole box (zero-filled out of bounds)
    const uint32_t bq = a.use_tm_qin ? (uint32_t)(SR / 4) * qs * 32 : (uint32_t)nq * q * 32;
    const uint32_t bb = a.use_tm_qb ? (uint32_t)(SR / 4) * UP_PB * 32 : (uint32_t)nq * p * 32;
    mbar_arrive_expect_tx(&full[st], bq + bb);
    const double* sq = a.Qin + (r0 >> 2) * 4 * a.ldqin;
    const double* sb = a.Qb + (r0 >> 2) * 4 * a.ldqb;
    if (a.use_tm_qin) {
      tma_load_3d_stream(dq, &a.tm_qin, 0, 0, (int)(r0 >> 2), &full[st]);
    } else {
      for (int qq = 0; qq < nq; ++qq) bulk_g2s_stream(dq + qq * 4 * qs, sq + qq * 4 * a.ldqin, (uint32_t)q * 32, &full[st]);
    }
    if (a.use_tm_qb) {
      tma_load_3d_stream(db, &a.tm_qb, 0, 0, (int)(r0 >> 2), &full[st]);
    } else if (a.ldqb == UP_PB && p == UP_PB) {
      bulk_g2s_stream(db, sb, (uint32_t)nq * UP_PB * 32, &full[st]);
    } else {
      for (int qq = 0; qq < nq; ++qq) bulk_g2s_stream(db + qq * 4 * UP_PB, sb + qq * 4 * a.ldqb, (uint32_t)p * 32, &full[st]);
    }
  };
  if (tid == 0)
    for (int j = 0; j < ns && j < mine; ++j) issue(j, j);

  int s = 0, ys = 0;
  uint32_t ph = 0, yph = 0;
  if (TEAMS && warp < 8) {
    // ================= projection group, two teams of 4 warps (alternate sub-panels)
    const int team = warp >> 2, wt = warp & 3, tt = tid & 127;
    // warp wt of a team owns the 16 columns [64c + 16wt, +16) of every full block
    // (k4 steps h = 0..3); a partial last block is split by k4 step, step wt + 4h,
    // so its valid steps land evenly on the four sub-partitions.
    auto kcolt = [&](int c, int h) {
      return (PART && c == NQ - 1) ? 64 * c + 4 * (wt + 4 * h) : 64 * c + 16 * wt + 4 * h;
    };
    double btt[NQ][4][2];
#pragma unroll
    for (int c = 0; c < NQ; ++c)
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          const int kk = kcolt(c, h) + t, n = 8 * nb + g;
          btt[c][h][nb] = (!init && kk < q && n < p) ? a.Bt[(int64_t)n * a.ldbt + kk] : 0.0;
        }
    // narrow (q <= 64): warp wt owns the output blocks (row block (wt >> 1) + 2u,
    // column block wt & 1) of proj over the full width, Bt in registers -- the
    // 8-warp narrow mapping given to a 4-warp team, the same per-element chains
    double btn[NARROW ? 16 : 1];
    if constexpr (NARROW) {
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const int kk = 4 * ks + t, n = 8 * (wt & 1) + g;
        btn[ks] = (!init && kk < q && n < p) ? a.Bt[(int64_t)n * a.ldbt + kk] : 0.0;
      }
    }
    double* tqt = tq + team * TE;
    const int bar = 2 + team;
    for (int64_t j = team; j < (direct ? 0 : mine); j += 2) {
      const int sj = (int)(j % ns), ysj = (int)(j % UP_YS);
      const uint32_t phj = (uint32_t)((j / ns) & 1), yphj = (uint32_t)((j / UP_YS) & 1);
      const int64_t r0 = (blockIdx.x + j * gridDim.x) * SR;
      const int nrows = (int)imin64(SR, a.rows - r0);
      mbar_wait(&full[sj], phj);
      const double* Qs = stg + sj * STG;
      const double* Ys = Qs + SR * qs;
      double* yd = yring + ysj * TE;
      if (nrows < SR) {
        double* Qz = stg + sj * STG + nrows * qs;
        for (int e = tt; e < (SR - nrows) * qs; e += 128) Qz[e] = 0.0;
      }
      if (!init) {
       if constexpr (NARROW) {
        constexpr int NU2 = NARROW ? RB / 2 : 1;
        const int nbw = wt & 1;
        double acc[NU2][4][2] = {};   // k4 steps round-robin over four accumulator chains per block
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          if (4 * ks < q) {   // warp-uniform
#pragma unroll
            for (int u = 0; u < NU2; ++u) {
              const int rbw = (wt >> 1) + 2 * u;
              const double* xa = Qs + (2 * rbw + (g >> 2)) * 4 * qs + (g & 3) + 4 * t;
              const double av = (4 * ks + t < q) ? xa[16 * ks] : 0.0;
              dmma(acc[u][ks & 3], av, btn[ks]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NU2; ++u) {
          const int row = 8 * ((wt >> 1) + 2 * u) + g;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * nbw + 2 * t + e;
            const int off = (row >> 2) * 4 * UP_PB + 4 * col + (row & 3);
            tqt[off] = (col < p && row < nrows)
                           ? Ys[off] - ((acc[u][0][e] + acc[u][1][e]) + (acc[u][2][e] + acc[u][3][e])) : 0.0;
          }
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
       } else {
        double pr[RB][2][2];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) { pr[rb][nb][0] = 0.0; pr[rb][nb][1] = 0.0; }
        const double* xa = Qs + (g >> 2) * 4 * qs + (g & 3) + 4 * t;   // row g, column t
#pragma unroll
        for (int c = 0; c < NQ; ++c)
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int kc = kcolt(c, h);
            if (PART && c == NQ - 1 && kc >= q) continue;   // warp-uniform
            const bool kv = kc + t < q;
            double av[RB];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) av[rb] = kv ? xa[4 * kc + rb * 8 * qs] : 0.0;
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
              dmma(pr[rb][0], av[rb], btt[c][h][0]);
              dmma(pr[rb][1], av[rb], btt[c][h][1]);
            }
          }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              red[warp * TE + (2 * rb + (g >> 2)) * 4 * UP_PB + 4 * (8 * nb + 2 * t + e) + (g & 3)] = pr[rb][nb][e];
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
        for (int e = tt; e < TE; e += 128) {
          const int row = 4 * (e >> 6) + (e & 3), col = (e >> 2) & 15;
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < 4; ++w) sum += red[(4 * team + w) * TE + e];
          tqt[e] = (col < p && row < nrows) ? Ys[e] - sum : 0.0;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
       }
        if (j >= UP_YS) mbar_wait(&yempty[ysj], yphj ^ 1);
        for (int qb = wt; qb < 2 * RB; qb += 4) {
          const int rb = qb >> 1, nb = qb & 1;
          const int r = 8 * rb + g;
          const double* tp = tqt + (r >> 2) * 4 * UP_PB + (r & 3) + 4 * t;
          const double* rp = ris + (8 * nb + g) * CT_LD + t;
          double c2[2] = {0.0, 0.0};
          if (nb == 0) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) dmma(c2, tp[16 * ks], rp[4 * ks]);
          } else {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) dmma(c2, tp[16 * ks], rp[4 * ks]);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = 8 * nb + 2 * t + e;
            const bool v = cc < p;
            yd[(r >> 2) * 4 * UP_PB + 4 * cc + (r & 3)] = v ? c2[e] : 0.0;
            if (v && r < nrows) st_stream(a.Qo + ((r0 + r) >> 2) * 4 * a.ldqo + 4 * cc + (r & 3), c2[e]);
          }
        }
      } else {
        if (j >= UP_YS) mbar_wait(&yempty[ysj], yphj ^ 1);
        for (int e = tt; e < TE; e += 128) {
          const int row = 4 * (e >> 6) + (e & 3), col = (e >> 2) & 15;
          yd[e] = (col < p && row < nrows) ? Ys[e] : 0.0;
        }
      }
      mbar_arrive(&yfull[ysj]);   // every thread of the team: its own stores are released
    }
  } else if (warp < 8) {
    // ================= projection group
    // Bases up to 64 columns ("narrow", 32-row sub-panels): warp wa owns the
    // output block (rows 8(wa/2).., columns 8(wa%2)..) of proj = Q_in Bt over
    // the FULL width, its Bt column block in registers, so there are no
    // per-warp partials to reduce through shared memory: t = Q - proj goes
    // straight from the accumulators to the t buffer (one barrier per
    // sub-panel instead of two, 1 KB of t stores instead of 8 x 4 KB of
    // partials plus their 8-way sum).  Wider bases split the width over the
    // warps (Bt rows in registers) and sum the 8 partials in a fixed order.
    const int wa = warp;
    double btn[NARROW ? 16 * NQ : 1];   // narrow: Bt(4ks + t, 8(wa%2) + g)
    if constexpr (NARROW) {
#pragma unroll
      for (int ks = 0; ks < 16 * NQ; ++ks) {
        const int kk = 4 * ks + t, n = 8 * (wa & 1) + g;
        btn[ks] = (!init && kk < q && n < p) ? a.Bt[(int64_t)n * a.ldbt + kk] : 0.0;
      }
    }
    // Bt(kc(c, h) + t, 8nb + g).  Full 64-column blocks: warp wa owns the 8
    // columns [64c + 8wa, +8).  The last block (only q - 64(NQ-1) columns
    // valid) is split by k4 step instead: warp wa takes steps s + 4j + 8h
    // (s = wa % 4 = its SM sub-partition, j = wa / 4), so the valid steps of a
    // partial block land evenly on the four sub-partitions, and the steps past
    // q are skipped whole (warp-uniform), not multiplied by zero.
    const int kap = (wa & 3) + 4 * (wa >> 2);
    auto kcol = [&](int c, int h) {
      return (PART && c == NQ - 1) ? 64 * c + 4 * (kap + 8 * h) : 64 * c + 8 * wa + 4 * h;
    };
    double btr[NARROW ? 1 : NQ][2][2];
    if constexpr (!NARROW) {
#pragma unroll
    for (int c = 0; c < NQ; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          const int kk = kcol(c, h) + t, n = 8 * nb + g;
          btr[c][h][nb] = (!init && kk < q && n < p) ? a.Bt[(int64_t)n * a.ldbt + kk] : 0.0;
        }
    }
    for (int64_t j = 0; j < (direct ? 0 : mine); ++j) {
      const int64_t r0 = (blockIdx.x + j * gridDim.x) * SR;
      const int nrows = (int)imin64(SR, a.rows - r0);
      mbar_wait(&full[s], ph);
      const double* Qs = stg + s * STG;
      const double* Ys = Qs + SR * qs;
      double* yd = yring + ys * TE;
      if (SR > 16 && nrows < SR) {
        // ragged last sub-panel: the stage's rows >= nrows are stale; zero them
        // for the cross-Gram group (it multiplies them by Q' rows that are 0)
        double* Qz = stg + s * STG + nrows * qs;
        for (int e = tid; e < (SR - nrows) * qs; e += 256) Qz[e] = 0.0;
      }
      if (NARROW && !init) {
        // warp wa owns the output blocks (row block (wa / 2) + 4u, column block wa % 2), u < NU
        constexpr int NU = NARROW ? RB / 4 : 1;
        const int nbw = wa & 1;
        double acc[NU][4][2] = {};   // k4 steps round-robin over four accumulator chains per block
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          if (4 * ks < q) {   // warp-uniform
#pragma unroll
            for (int u = 0; u < NU; ++u) {
              // A fragments Q_in(row 8 rbw + g, column 4 ks + t): conflict-free (qs = 4 mod 8)
              const int rbw = (wa >> 1) + 4 * u;
              const double* xa = Qs + (2 * rbw + (g >> 2)) * 4 * qs + (g & 3) + 4 * t;
              const double av = (4 * ks + t < q) ? xa[16 * ks] : 0.0;
              dmma(acc[u][ks & 3], av, btn[ks]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const int row = 8 * ((wa >> 1) + 4 * u) + g;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * nbw + 2 * t + e;
            const int off = (row >> 2) * 4 * UP_PB + 4 * col + (row & 3);
            tq[off] = (col < p && row < nrows)
                          ? Ys[off] - ((acc[u][0][e] + acc[u][1][e]) + (acc[u][2][e] + acc[u][3][e])) : 0.0;
          }
        }
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
      if (!NARROW && !init) {
        double pr[RB][2][2];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) { pr[rb][nb][0] = 0.0; pr[rb][nb][1] = 0.0; }
        const double* xa = Qs + (g >> 2) * 4 * qs + (g & 3) + 4 * t;   // row g, column t
#pragma unroll
        for (int c = 0; c < NQ; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kc = kcol(c, h);                // + t
            if (PART && c == NQ - 1 && kc >= q) continue;   // a whole k4 step past q: skipped (warp-uniform)
            const bool kv = kc + t < q;               // columns >= q of the stage are stale
            double av[RB];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) av[rb] = kv ? xa[4 * kc + rb * 8 * qs] : 0.0;   // row 8 rb + g
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) {
              dmma(pr[rb][0], av[rb], btr[c][h][0]);
              dmma(pr[rb][1], av[rb], btr[c][h][1]);
            }
          }
        if (lag) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&pdone[ys]);   // this warp's projection DMMAs of sub-panel j are issued
        }
        // partials in the QI layout of the sub-panel (as tq, yd and the stage)
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              red[wa * TE + (2 * rb + (g >> 2)) * 4 * UP_PB + 4 * (8 * nb + 2 * t + e) + (g & 3)] = pr[rb][nb][e];
        asm volatile("bar.sync 2, 256;" ::: "memory");
        for (int e = tid; e < TE; e += 256) {
          // e is the QI offset itself: a warp touches 32 consecutive doubles
          const int row = 4 * (e >> 6) + (e & 3), col = (e >> 2) & 15;
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < 8; ++w) sum += red[w * TE + e];
          tq[e] = (col < p && row < nrows) ? Ys[e] - sum : 0.0;
        }
        asm volatile("bar.sync 2, 256;" ::: "memory");
      }
      if (!init) {
        if (j >= UP_YS) mbar_wait(&yempty[ys], yph ^ 1);
        for (int qb = wa; qb < 2 * RB; qb += 8) {
          // Q' block (rb, nb) = t(rows 8rb.., :) R^-1(:, cols 8nb..); R^-1 upper: K < 8(nb+1)
          const int rb = qb >> 1, nb = qb & 1;
          const int r = 8 * rb + g;
          const double* tp = tq + (r >> 2) * 4 * UP_PB + (r & 3) + 4 * t;
          const double* rp = ris + (8 * nb + g) * CT_LD + t;
          double c2[2] = {0.0, 0.0};
          if (nb == 0) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) dmma(c2, tp[16 * ks], rp[4 * ks]);
          } else {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) dmma(c2, tp[16 * ks], rp[4 * ks]);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = 8 * nb + 2 * t + e;
            const bool v = cc < p;
            yd[(r >> 2) * 4 * UP_PB + 4 * cc + (r & 3)] = v ? c2[e] : 0.0;
            if (v && r < nrows) st_stream(a.Qo + ((r0 + r) >> 2) * 4 * a.ldqo + 4 * cc + (r & 3), c2[e]);
          }
        }
      } else {
        // initial mode: Q' = Q (stale padding columns / rows zeroed)
        if (j >= UP_YS) mbar_wait(&yempty[ys], yph ^ 1);
        for (int e = tid; e < TE; e += 256) {
          const int row = 4 * (e >> 6) + (e & 3), col = (e >> 2) & 15;
          yd[e] = (col < p && row < nrows) ? Ys[e] : 0.0;
        }
      }
      mbar_arrive(&yfull[ys]);   // every projection thread: its own stores are released
      if (++s == ns) { s = 0; ph ^= 1; }
      if (++ys == UP_YS) { ys = 0; yph ^= 1; }
    }
  } else {
    // ================= cross-Gram group
    const int wb = warp - 8;
    double ct[NQ][2][2];
#pragma unroll
    for (int c = 0; c < NQ; ++c)
#pragma unroll
      for (int n = 0; n < 2; ++n) { ct[c][n][0] = 0.0; ct[c][n][1] = 0.0; }
    double gq[2] = {0.0, 0.0};
    const int bi = (wb == 0) ? 0 : 1, bj = (wb == 2) ? 1 : 0;
    // Full blocks c < NQ - 1: warp wb owns the Bt' rows [64c + 8wb, +8) (both
    // 8-column halves of p).  The last block is split by output 8 x 8 block
    // instead: chain i = wb + 8 h2 is block (rows 64(NQ-1) + 8(i / 2), columns
    // 8(i % 2)), kept in ct[NQ-1][h2]; the chains of a partial block spread
    // over the sub-partitions and the blocks past q are skipped whole.
    const int cl0 = 64 * (NQ - 1);
    for (int64_t j = 0; j < mine; ++j) {
      if (lag && j + 1 < mine) {
        const int yn = (ys + 1 == UP_YS) ? 0 : ys + 1;
        mbar_wait(&pdone[yn], (ys + 1 == UP_YS) ? (yph ^ 1) : yph);
      }
      const double* Qs = stg + s * STG;
      const double* yd;
      if (direct) {
        mbar_wait(&full[s], ph);
        yd = Qs + SR * qs;
      } else {
        mbar_wait(&yfull[ys], yph);
        yd = yring + ys * TE;
      }
      const double* xa = Qs + 4 * (8 * wb + g) + t;   // Q_in(row t, column 8wb + g)
#pragma unroll
      for (int ks = 0; ks < Q4; ++ks) {
        const double b0 = yd[ks * 64 + 4 * g + t], b1 = yd[ks * 64 + 32 + 4 * g + t];
#pragma unroll
        for (int c = 0; c < (PART ? NQ - 1 : NQ); ++c) {
          // a warp whose Bt' rows all lie past q (q < 64: NQ = 1 covers 64 columns)
          // skips its chain, warp-uniformly: at q = 16 six of the eight warps
          // issued DMMAs on zero operands in a pass throttled by the FP64 pipe
          if constexpr (NQ == 1) {
            if (8 * wb >= q) continue;
          }
          const bool v = PART || 64 * c + 8 * wb + g < q;
          const double av = v ? xa[ks * 4 * qs + 256 * c] : 0.0;
          dmma(ct[c][0], av, b0);
          dmma(ct[c][1], av, b1);
        }
        if (PART) {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int i = wb + 8 * h2, ob = i >> 1;
            if (cl0 + 8 * ob >= q) continue;             // warp-uniform: block past q
            const bool v = cl0 + 8 * ob + g < q;
            const double av = v ? Qs[4 * (cl0 + 8 * ob + g) + t + ks * 4 * qs] : 0.0;
            dmma(ct[NQ - 1][h2], av, (i & 1) ? b1 : b0);
          }
        }
      }
      if (wb < 3) {
#pragma unroll
        for (int ks = 0; ks < Q4; ++ks) dmma(gq, yd[ks * 64 + 32 * bi + 4 * g + t], yd[ks * 64 + 32 * bj + 4 * g + t]);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        if (!direct) mbar_arrive(&yempty[ys]);
        if (wb == 7 && j + ns < mine) {
          mbar_wait(&empty[s], ph);   // all 8 cross-Gram warps are done with the stage
          issue(j + ns, s);
        }
      }
      __syncwarp();
      if (++s == ns) { s = 0; ph ^= 1; }
      if (++ys == UP_YS) { ys = 0; yph ^= 1; }
    }
    // ---- per-CTA partials: [Bt'(q_pad x 16) | G (16 x 16)] column-major with ld = q_pad + 16
    const int qp = (int)round_up(q, 64);
    const int ld = qp + UP_PB;
    double* out = a.ws + (int64_t)blockIdx.x * ld * UP_PB;
#pragma unroll
    for (int c = 0; c < (PART ? NQ - 1 : NQ); ++c)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) out[(int64_t)(8 * n + 2 * t + e) * ld + 64 * c + 8 * wb + g] = ct[c][n][e];
    if (PART) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int i = wb + 8 * h2, ob = i >> 1, n = i & 1;   // chains past q hold zeros (never accumulated)
#pragma unroll
        for (int e = 0; e < 2; ++e) out[(int64_t)(8 * n + 2 * t + e) * ld + cl0 + 8 * ob + g] = ct[NQ - 1][h2][e];
      }
    }
    if (wb < 3) {
#pragma unroll
      for (int e = 0; e < 2; ++e) out[(int64_t)(8 * bj + 2 * t + e) * ld + qp + 8 * bi + g] = gq[e];
    }
  }
}

// fixed-order sum over CTAs; Bt' (q x p, ld ldbt) and G (p x p, lower mirrored, ld ldg).
// One thread per element adds the partials in CTA order (bitwise the order of
// every earlier version), loading them in batches of 32 ahead of the adds.
__global__ void update_reduce_kernel(const double* __restrict__ ws, int nparts, int q, int p, int qp,
                                     double* Bt, int ldbt, double* G, int ldg, const int* gate) {
  if (gate != nullptr && *gate != 0) return;
  const int ld = qp + UP_PB;
  const int64_t nbt = (int64_t)q * p, ng = (int64_t)p * p;
  const int64_t ps = (int64_t)ld * UP_PB;
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
    int i = 0;
    for (; i + 32 <= nparts; i += 32) {
      double v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ws[(i + j) * ps + off];
#pragma unroll
      for (int j = 0; j < 32; ++j) s += v[j];
    }
    if (i < nparts) {   // the remainder as one masked batch (one L2 round trip, not one per partial)
      double v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = (i + j < nparts) ? ws[(i + j) * ps + off] : 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (i + j < nparts) s += v[j];
    }
    if (e < nbt) Bt[(int64_t)c * ldbt + r] = s;
    else { G[(int64_t)c * ldg + r] = s; G[(int64_t)r * ldg + c] = s; }
  }
}

static int update_ctas(int64_t rows) {
  int64_t n = ceil_div(rows, 16);
  int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

// ---- 3-D tensor maps of QI arrays (driver entry point through the runtime: no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}
static int g_update_tma = 1;   // cqr_debug_update_tma: 0 = per-quad bulk copies only (comparisons)
void set_update_tma(int on) { g_update_tma = on ? 1 : 0; }

// box {4, boxc, sr/4} over the first `cols` columns of a QI array (rows a
// multiple of 16, column capacity ld).  The column extent is `cols`, not the
// capacity: `base` may be a column block inside the buffer (the update path's
// tail block), and a box reaching past its last column must be zero-filled by
// the TMA unit, never read from past the allocation.
static bool encode_qi_map(CUtensorMap* tm, const double* base, int64_t ld, int cols, int64_t rows, int boxc, int sr) {
  auto enc = tensor_map_encoder();
  if (!g_update_tma || enc == nullptr || boxc > 256 || ((uintptr_t)base & 15) != 0) return false;
  const cuuint64_t dims[3] = {4, (cuuint64_t)cols, (cuuint64_t)(rows / 4)};
  const cuuint64_t strides[2] = {32, (cuuint64_t)ld * 32};
  const cuuint32_t box[3] = {4, (cuuint32_t)boxc, (cuuint32_t)(sr / 4)};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool update_pass_supported(int q, int p) {
  return q >= 1 && q <= UP_MAXQ && p >= 1 && p <= UP_PB && up_stages(q, up_sr(q)) >= 2;
}

size_t update_pass_ws_bytes(int64_t rows, int q) {
  const int qp = (int)round_up(q, 64);
  return (size_t)update_ctas(rows) * (qp + UP_PB) * UP_PB * sizeof(double) + 256;
}

template <int NQ, int SR, bool TEAMS>
static cudaError_t launch_up_t(const UpdateArgs& a, int ctas, size_t smem, cudaStream_t s) {
  const bool part = NQ >= 2 && (a.q % 64) != 0;
  const void* fn = part ? (const void*)update_pass_kernel<NQ, SR, (NQ >= 2), TEAMS>
                        : (const void*)update_pass_kernel<NQ, SR, false, TEAMS>;
  cudaError_t e = smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  if (part)
    update_pass_kernel<NQ, SR, (NQ >= 2), TEAMS><<<ctas, UP_THREADS, smem, s>>>(a);
  else
    update_pass_kernel<NQ, SR, false, TEAMS><<<ctas, UP_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NQ, int SR>
static cudaError_t launch_up(const UpdateArgs& a, int ctas, size_t smem, cudaStream_t s) {
  if constexpr ((SR == 32 && (NQ == 2 || NQ == 3)) || (SR == 64 && NQ == 1)) {
    if (up_teams_q(a.q, SR)) return launch_up_t<NQ, SR, true>(a, ctas, smem, s);
  }
  return launch_up_t<NQ, SR, false>(a, ctas, smem, s);
}

int update_set_narrow_teams(int on) {
  g_narrow_teams = on ? 1 : 0;
  return 0;
}
int update_set_sr16_from(int q) {
  if (q < 145 || q > 193) return -1;   // 65..144 run the two-team schedule on 32-row sub-panels
  g_sr16_from = q;
  return 0;
}
// 0 = never, 1 = always (wide single-group passes), 2 (default) = where it was
// measured to pay: 16-row sub-panels with a 4- or 5-stage ring (q = 256..368)
static int g_update_direct = 1;   // cqr_debug_update_direct
int update_set_direct(int on) {
  g_update_direct = on ? 1 : 0;
  return 0;
}
static int g_update_lag = 2;   // cqr_debug_update_lag
int update_set_lag(int mode) {
  g_update_lag = mode;
  return 0;
}

cudaError_t update_pass_launch(const double* Qin, int64_t ldqin, int q, const double* Qb, int64_t ldqb, double* Qo,
                               int64_t ldqo, int p, int64_t rows, const double* Bt, int ldbt, const double* Rinv_tiles,
                               int initial, double* Bt_next, double* G, int ldg, double* ws, cudaStream_t s,
                               const int* gate) {
  if (rows % 16) return cudaErrorInvalidValue;
  UpdateArgs a{};
  a.Qin = Qin; a.ldqin = ldqin; a.q = q;
  a.Qb = Qb; a.ldqb = ldqb; a.p = p;
  a.Qo = Qo; a.ldqo = ldqo;
  a.rows = rows;
  a.Bt = Bt; a.ldbt = ldbt; a.Rinv = Rinv_tiles;
  a.initial = initial;
  a.ws = ws;
  a.gate = gate;
  a.qs = up_qs(q);
  const int sr = up_sr(q);
  a.direct = (g_update_direct && initial && p == UP_PB && rows % sr == 0) ? 1 : 0;
  {
    const int nst = up_stages(q, sr);
    a.lag = g_update_lag == 1 || (g_update_lag == 2 && sr == 16 && (nst == 4 || nst == 5));
  }
  // one tensor copy per sub-panel where the per-quad runs would be small
  a.use_tm_qin = (q * 32 < 8192) && encode_qi_map(&a.tm_qin, Qin, ldqin, q, rows, a.qs, sr) ? 1 : 0;
  a.use_tm_qb = !(ldqb == UP_PB && p == UP_PB) && encode_qi_map(&a.tm_qb, Qb, ldqb, p, rows, UP_PB, sr) ? 1 : 0;
  a.ns = up_stages(q, sr);
  const size_t smem = update_smem_bytes(q, sr);
  const int ctas = update_ctas(rows);
  cudaError_t e;
  switch ((q + 63) / 64) {
    case 1: e = launch_up<1, 64>(a, ctas, smem, s); break;
    case 2: e = launch_up<2, 32>(a, ctas, smem, s); break;
    case 3: e = (sr == 32) ? launch_up<3, 32>(a, ctas, smem, s) : launch_up<3, 16>(a, ctas, smem, s); break;
    case 4: e = launch_up<4, 16>(a, ctas, smem, s); break;
    case 5: e = launch_up<5, 16>(a, ctas, smem, s); break;
    case 6: e = launch_up<6, 16>(a, ctas, smem, s); break;
    case 7: e = launch_up<7, 16>(a, ctas, smem, s); break;
    case 8: e = launch_up<8, 16>(a, ctas, smem, s); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  const int qp = (int)round_up(q, 64);
  const int64_t nel = (int64_t)q * p + (int64_t)p * p;
  update_reduce_kernel<<<(int)ceil_div(nel, 256), 256, 0, s>>>(ws, ctas, q, p, qp, Bt_next, q, G, ldg, gate);
  return cudaGetLastError();
}

}  // namespace cqr
