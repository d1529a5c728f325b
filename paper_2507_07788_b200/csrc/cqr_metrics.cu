// K5: streaming quality measures (reference metrics.py:53-71).
//
// reconstruction_residual(a, q, r) forms D = A - Q R as a fresh tall array
// (a.copy(), q.lincomb(r), axpy) and then its Gramian; at BASELINE config 5
// (128M x 64, 65.5 GB per array) that is two more arrays than one B200 holds
// next to A and Q.  This kernel makes one sweep over the rows of Q and A and
// never materialises Q R or D:
//   * per 64-row panel (8 warps x 8 rows, the register-resident scheme of
//     cqr_fused.cu), a warp computes (Q R)^T for its 8 rows by DMMA with
//     A = R^T from coefficient tiles (R upper triangular: column block j
//     only sees k4 steps < 8(j+1)) and B = Q from the staged panel, so lane
//     (g, t) holds (Q R)[r0 + 2t + e][8j + g];
//   * it loads A at exactly those positions straight from HBM (two
//     consecutive doubles of the QI layout per lane and column block, a fully
//     coalesced 256-byte run per warp instruction), issued before the TRMM so
//     the loads are in flight while the DMMAs run;
//   * D = A - Q R in registers; D^T D accumulates from the same registers
//     (the accumulator layout of the TRMM is the operand layout of the Gram
//     DMMA over the 4 rows {r0 + 2t + e}), and sum A^2 in one scalar per lane.
// Per-CTA partials (the lower triangle of D^T D, and sum A^2) are summed over
// CTAs in a fixed order: the result is reproducible bit for bit.
// Reads Q and A once (16 k bytes per row), writes nothing tall; FP64 work
// k(k+1) (TRMM) + k(k+1) (SYRK) flops per row.  k <= 64.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

constexpr int RS_ROWS = 64;   // rows per staged Q panel (8 warps x 8 rows)

template <int KP>
struct RsCfg {
  static constexpr int NB = KP / 8;
  static constexpr int NKS = KP / 4;
  static constexpr int NKT = KP > CT_K ? KP / CT_K : 1;
  static constexpr int NG = NB * (NB + 1) / 2;
  static constexpr int STAGE = RS_ROWS * KP;
  static constexpr int STAGES = KP >= 64 ? 5 : 8;
  static constexpr int THREADS = 256;
};
template <int KP>
__host__ __device__ constexpr size_t rs_smem_doubles() {
  return (size_t)RsCfg<KP>::NKT * CT_TILE + (size_t)RsCfg<KP>::STAGES * RsCfg<KP>::STAGE;
}

__device__ __forceinline__ void ld_global_nc_v2(const double* p, double& a, double& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}

template <int KP, bool KFULL>
__global__ void __launch_bounds__(RsCfg<KP>::THREADS, 1)
    resid_gram_kernel(const double* Q, int64_t ldq, const double* A, int64_t lda, int k,
                      const double* __restrict__ Rt, int64_t rows, double* __restrict__ ws) {
  using C = RsCfg<KP>;
  constexpr int NB = C::NB, NKS = C::NKS, ST = C::STAGES;
  constexpr int LAG = 2, D = ST - LAG;
  extern __shared__ __align__(128) double smem[];
  double* rt_s = smem;
  double* qst = smem + C::NKT * CT_TILE;
  __shared__ __align__(8) uint64_t bars[2 * ST + 1];
  __shared__ double xred[C::THREADS];
  uint64_t* full = bars;
  uint64_t* empty = bars + ST;
  uint64_t* rbar = bars + 2 * ST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t npan = ceil_div(rows, RS_ROWS);
  const int64_t mine = (npan > blockIdx.x) ? ceil_div(npan - blockIdx.x, gridDim.x) : 0;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t j, int st) {
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * RS_ROWS;
    const int nq = (int)imin64(RS_ROWS, rows - r0) >> 2;
    double* dst = qst + st * C::STAGE;
    const double* src = Q + (r0 >> 2) * 4 * ldq;
    mbar_arrive_expect_tx(&full[st], (uint32_t)nq * k * 32);
    if (ldq == KP && KFULL) {
      bulk_g2s_stream(dst, src, (uint32_t)nq * KP * 32, &full[st]);
    } else {
      for (int q = 0; q < nq; ++q) bulk_g2s_stream(dst + q * 4 * KP, src + q * 4 * ldq, (uint32_t)k * 32, &full[st]);
    }
  };
  if (tid == 0) {
    mbar_arrive_expect_tx(rbar, C::NKT * CT_TILE * 8);
    for (int kt = 0; kt < C::NKT; ++kt) bulk_g2s(rt_s + kt * CT_TILE, Rt + (int64_t)kt * CT_TILE, CT_TILE * 8, rbar);
    for (int j = 0; j < D && j < mine; ++j) issue(j, j);
  }

  double gacc[C::NG][2];
#pragma unroll
  for (int b = 0; b < C::NG; ++b) { gacc[b][0] = 0.0; gacc[b][1] = 0.0; }
  double asq = 0.0;
  const double* rp = rt_s + g * CT_LD + t;
  mbar_wait(rbar, 0);
  int s = 0;
  uint32_t ph = 0;
  for (int64_t j = 0; j < mine; ++j) {
    if (tid == 0 && j + D < mine) {
      const int64_t j2 = j + D;
      const int s2 = (int)(j2 % ST);
      if (j2 >= ST) mbar_wait(&empty[s2], (uint32_t)((j2 / ST) - 1) & 1);
      issue(j2, s2);
    }
    const int64_t r0 = (blockIdx.x + j * gridDim.x) * RS_ROWS + 8 * warp;
    const bool valid = r0 < rows;   // rows is a multiple of 16
    // A at the accumulator positions: rows r0 + 2t + e (one quad, consecutive), column 8b + g
    double av[NB][2];
    if (valid) {
      const double* ap = A + ((r0 >> 2) + (t >> 1)) * 4 * lda + 4 * g + 2 * (t & 1);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (KFULL || 8 * b + g < k) ld_global_nc_v2(ap + 32 * b, av[b][0], av[b][1]);
        else { av[b][0] = 0.0; av[b][1] = 0.0; }
      }
    }
    mbar_wait(&full[s], ph);
    double qt[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) { qt[b][0] = 0.0; qt[b][1] = 0.0; }
    if (valid) {
      const double* xp = qst + s * C::STAGE + (2 * warp + (g >> 2)) * 4 * KP + 4 * t + (g & 3);
      double xb[2];
      xb[0] = (KFULL || t < k) ? xp[0] : 0.0;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int cur = ks & 1;
        if (ks + 1 < NKS) xb[cur ^ 1] = (KFULL || 4 * (ks + 1) + t < k) ? xp[16 * (ks + 1)] : 0.0;
#pragma unroll
        for (int b = ks / 2; b < NB; ++b) {
          const double ra = rp[(ks / 8) * CT_TILE + 8 * b * CT_LD + 4 * (ks % 8)];
          dmma(qt[b], ra, xb[cur]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == ST) { s = 0; ph ^= 1; }
    if (!valid) continue;
    // D = A - Q R (columns >= k: both zero), sum A^2
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      asq = fma(av[b][0], av[b][0], asq);
      asq = fma(av[b][1], av[b][1], asq);
      if (KFULL || 8 * b + g < k) {
        qt[b][0] = av[b][0] - qt[b][0];
        qt[b][1] = av[b][1] - qt[b][1];
      } else {
        qt[b][0] = 0.0;
        qt[b][1] = 0.0;
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c) dmma(gacc[i * (i + 1) / 2 + c], qt[i][e], qt[c][e]);
    }
  }

  // ---- per-CTA partials: D^T D (KP x KP column-major, lower triangle, warps in
  // fixed order) and sum A^2 (threads in fixed order)
  double* red = smem;
  __syncthreads();
  xred[tid] = asq;
  for (int e = tid; e < KP * KP; e += 256) red[e] = 0.0;
  __syncthreads();
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int c = 0; c <= i; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) red[(8 * c + 2 * t + e) * KP + 8 * i + g] += gacc[i * (i + 1) / 2 + c][e];
    }
    __syncthreads();
  }
  double* out = ws + (int64_t)blockIdx.x * (KP * KP + 1);
  for (int e = tid; e < KP * KP; e += 256) out[e] = red[e];
  if (tid == 0) {
    double sacc = 0.0;
    for (int i = 0; i < C::THREADS; ++i) sacc += xred[i];
    out[KP * KP] = sacc;
  }
}

// Fixed-order sum over CTAs: DtD (k x k, lower triangle computed and mirrored)
// and out_asq[0] = sum A^2.
__global__ void __launch_bounds__(256) resid_reduce_kernel(const double* __restrict__ ws, int nparts, int KP, int k,
                                                           double* DtD, int ldd, double* out_asq) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ps = (int64_t)KP * KP + 1;
  if (e == (int64_t)k * k) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += ws[p * ps + (int64_t)KP * KP];
    out_asq[0] = s;
    return;
  }
  if (e > (int64_t)k * k) return;
  const int r = (int)(e % k), c = (int)(e / k);
  if (r < c) return;
  const double* src = ws + (int64_t)c * KP + r;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += src[p * ps];
  DtD[(int64_t)c * ldd + r] = s;
  DtD[(int64_t)r * ldd + c] = s;
}

static int rs_kp(int k) {
  if (k < 1) return 0;
  if (k <= 16) return 16;
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  return 0;
}
static int rs_ctas(int64_t rows) {
  const int64_t n = ceil_div(rows, RS_ROWS);
  const int64_t c = num_sms();
  return (int)(n < c ? (n < 1 ? 1 : n) : c);
}

bool resid_gram_supported(int k) { return rs_kp(k) != 0; }
size_t resid_gram_ws_bytes(int64_t rows, int k) {
  const int kp = rs_kp(k);
  return kp ? (size_t)rs_ctas(rows) * ((size_t)kp * kp + 1) * sizeof(double) + 256 : 0;
}

template <int KP>
static cudaError_t launch_rs(const double* Q, int64_t ldq, const double* A, int64_t lda, int k, const double* Rt,
                             int64_t rows, double* DtD, int ldd, double* asq, double* ws, cudaStream_t s) {
  const size_t smem = rs_smem_doubles<KP>() * sizeof(double);
  cudaError_t e = smem_attr((const void*)resid_gram_kernel<KP, true>, smem);
  if (e == cudaSuccess) e = smem_attr((const void*)resid_gram_kernel<KP, false>, smem);
  if (e != cudaSuccess) return e;
  const int ctas = rs_ctas(rows);
  if (k == KP)
    resid_gram_kernel<KP, true><<<ctas, RsCfg<KP>::THREADS, smem, s>>>(Q, ldq, A, lda, k, Rt, rows, ws);
  else
    resid_gram_kernel<KP, false><<<ctas, RsCfg<KP>::THREADS, smem, s>>>(Q, ldq, A, lda, k, Rt, rows, ws);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t nel = (int64_t)k * k + 1;
  resid_reduce_kernel<<<(int)ceil_div(nel, 256), 256, 0, s>>>(ws, ctas, KP, k, DtD, ldd, asq);
  return cudaGetLastError();
}

cudaError_t resid_gram_launch(const double* Q, int64_t ldq, const double* A, int64_t lda, int k,
                              const double* R_tiles, int64_t rows, double* DtD, int ldd, double* asq, double* ws,
                              cudaStream_t s) {
  switch (rs_kp(k)) {
    case 16: return launch_rs<16>(Q, ldq, A, lda, k, R_tiles, rows, DtD, ldd, asq, ws, s);
    case 32: return launch_rs<32>(Q, ldq, A, lda, k, R_tiles, rows, DtD, ldd, asq, ws, s);
    case 64: return launch_rs<64>(Q, ldq, A, lda, k, R_tiles, rows, DtD, ldd, asq, ws, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace cqr
