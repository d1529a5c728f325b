// Block-row pair helpers shared by the self-Gram kernels (cqr_gram_pairs.cu,
// cqr_fused.cu).  The lower triangle of the NB x NB grid of 8x8 blocks is cut
// into the NB/2 block-row pairs (i, NB-1-i), each exactly NB+1 blocks.  A
// staged panel is QI with ldk = KP: fp points at (column g, row t) of quad 0.
#pragma once
#include "cqr_common.cuh"

namespace cqr {

// one pair (i, NB-1-i): acc[0..i] = row i (cols 0..i), acc[i+1..NB] = row NB-1-i (cols 0..NB-1-i)
template <int NB, int I>
__device__ __forceinline__ void pair_load(double (&f)[NB - I], const double* fp, int ks) {
  const double* q = fp + ks * (NB * 32);   // quad ks of a [quad][KP][4] panel
#pragma unroll
  for (int c = 0; c < NB - I; ++c) f[c] = q[32 * c];
}
template <int NB, int I>
__device__ __forceinline__ void pair_mma(double (&acc)[NB + 1][2], const double (&f)[NB - I]) {
  constexpr int J = NB - 1 - I;
#pragma unroll
  for (int c = 0; c <= I; ++c) dmma(acc[c], f[I], f[c]);
#pragma unroll
  for (int c = 0; c <= J; ++c) dmma(acc[I + 1 + c], f[J], f[c]);
}
// NS k4 steps ks0, ks0 + kst, ... fully unrolled (full panels: no loop overhead)
template <int NB, int I, int NS>
__device__ __forceinline__ void pair_steps_fixed(double (&acc)[NB + 1][2], const double* fp, int ks0, int kst) {
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    double f[NB - I];
    pair_load<NB, I>(f, fp, ks0 + j * kst);
    pair_mma<NB, I>(acc, f);
  }
}

// lean variant for wide panels: only the two row fragments stay live, column
// fragments stream one at a time (fits the 168-register cap of a 9-warp CTA)
template <int NB, int I>
__device__ __forceinline__ void pair_step_lean(double (&acc)[NB + 1][2], const double* q) {
  constexpr int J = NB - 1 - I;
  const double fI = q[32 * I], fJ = q[32 * J];
#pragma unroll
  for (int c = 0; c <= J; ++c) {
    const double fc = q[32 * c];
    if (c <= I) dmma(acc[c], fI, fc);
    dmma(acc[I + 1 + c], fJ, fc);
  }
}
template <int NB, int I>
__device__ __forceinline__ void pair_steps_lean(double (&acc)[NB + 1][2], const double* fp, int ks0, int ks1,
                                                int kst) {
  for (int ks = ks0; ks < ks1; ks += kst) pair_step_lean<NB, I>(acc, fp + ks * (NB * 32));
}

// k4 steps ks0, ks0 + kst, ... < ks1.  PF: the fragments of the next step are
// loaded before this step's DMMAs issue (needs twice the fragment registers).
template <int NB, int I, bool PF>
__device__ __forceinline__ void pair_steps(double (&acc)[NB + 1][2], const double* fp, int ks0, int ks1, int kst) {
  if constexpr (!PF) {
    for (int ks = ks0; ks < ks1; ks += kst) {
      double f[NB - I];
      pair_load<NB, I>(f, fp, ks);
      pair_mma<NB, I>(acc, f);
    }
  } else {
    if (ks0 >= ks1) return;
    double f0[NB - I], f1[NB - I];
    pair_load<NB, I>(f0, fp, ks0);
    for (int ks = ks0; ks < ks1; ks += 2 * kst) {
      const bool has1 = ks + kst < ks1;
      if (has1) pair_load<NB, I>(f1, fp, ks + kst);
      pair_mma<NB, I>(acc, f0);
      if (!has1) break;
      if (ks + 2 * kst < ks1) pair_load<NB, I>(f0, fp, ks + 2 * kst);
      pair_mma<NB, I>(acc, f1);
    }
  }
}

template <int NB, int I>
__device__ __forceinline__ void pair_store(const double (&acc)[NB + 1][2], double* out, int g, int t) {
  constexpr int J = NB - 1 - I;
  constexpr int KP = 8 * NB;
  // out: KP x KP column-major partial
#pragma unroll
  for (int c = 0; c <= I; ++c)
#pragma unroll
    for (int e = 0; e < 2; ++e) out[(8 * c + 2 * t + e) * KP + 8 * I + g] += acc[c][e];
#pragma unroll
  for (int c = 0; c <= J; ++c)
#pragma unroll
    for (int e = 0; e < 2; ++e) out[(8 * c + 2 * t + e) * KP + 8 * J + g] += acc[I + 1 + c][e];
}

template <int NB, int I>
struct PairDispatch {
  template <bool PF = false>
  __device__ static void run(int pair, double (&acc)[NB + 1][2], const double* fp, int ks0, int ks1, int kst) {
    if (pair == I) pair_steps<NB, I, PF>(acc, fp, ks0, ks1, kst);
    else PairDispatch<NB, I + 1>::template run<PF>(pair, acc, fp, ks0, ks1, kst);
  }
  template <int NS>
  __device__ static void run_fixed(int pair, double (&acc)[NB + 1][2], const double* fp, int ks0, int kst) {
    if (pair == I) pair_steps_fixed<NB, I, NS>(acc, fp, ks0, kst);
    else PairDispatch<NB, I + 1>::template run_fixed<NS>(pair, acc, fp, ks0, kst);
  }
  __device__ static void run_lean(int pair, double (&acc)[NB + 1][2], const double* fp, int ks0, int ks1, int kst) {
    if (pair == I) pair_steps_lean<NB, I>(acc, fp, ks0, ks1, kst);
    else PairDispatch<NB, I + 1>::run_lean(pair, acc, fp, ks0, ks1, kst);
  }
  __device__ static void store(int pair, const double (&acc)[NB + 1][2], double* out, int g, int t) {
    if (pair == I) pair_store<NB, I>(acc, out, g, t);
    else PairDispatch<NB, I + 1>::store(pair, acc, out, g, t);
  }
};
template <int NB>
struct PairDispatch<NB, NB / 2> {
  template <bool PF = false>
  __device__ static void run(int, double (&)[NB + 1][2], const double*, int, int, int) {}
  template <int NS>
  __device__ static void run_fixed(int, double (&)[NB + 1][2], const double*, int, int) {}
  __device__ static void run_lean(int, double (&)[NB + 1][2], const double*, int, int, int) {}
  __device__ static void store(int, const double (&)[NB + 1][2], double*, int, int) {}
};

// Fixed-order sum of the per-CTA KP x KP partial triangles into G (k x k,
// lower triangle mirrored): one thread per element adds the partials in CTA
// order, p = 0, 1, 2, ... (the order every earlier version used, so results
// are bitwise unchanged).  The partials are loaded in batches of 32 before the
// adds: the first version issued one load per add and was latency bound at
// 30-50 us per call at k = 64 (profiles/r01_launches_config5.csv).  64-thread
// blocks: the call is bound by each SM's L2 load throughput, so the k^2
// elements are spread over as many SMs as possible (256-thread blocks put
// k = 64 on 16 SMs: 14.4 us per call, 3 of them in config 1's 0.54 ms).
constexpr int PR_BATCH = 32;
constexpr int PR_THREADS = 64;
static __global__ void __launch_bounds__(PR_THREADS) gram_partials_reduce(const double* __restrict__ ws, int nparts, int KP,
                                                                   int k, double* G, int ldg, const int* gate) {
  if (gate != nullptr && *gate != 0) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)k * k) return;
  const int r = (int)(e % k), c = (int)(e / k);
  if (r < c) return;
  const double* src = ws + (int64_t)c * KP + r;
  const int64_t ps = (int64_t)KP * KP;
  double s = 0.0;
  int p = 0;
  for (; p + PR_BATCH <= nparts; p += PR_BATCH) {
    double v[PR_BATCH];
#pragma unroll
    for (int j = 0; j < PR_BATCH; ++j) v[j] = src[(p + j) * ps];
#pragma unroll
    for (int j = 0; j < PR_BATCH; ++j) s += v[j];
  }
  if (p < nparts) {
    // the remainder as one masked batch (a scalar loop here was one L2 round
    // trip per partial: ~7 us of the call at 148 partials)
    double v[PR_BATCH];
#pragma unroll
    for (int j = 0; j < PR_BATCH; ++j) v[j] = (p + j < nparts) ? src[(p + j) * ps] : 0.0;
#pragma unroll
    for (int j = 0; j < PR_BATCH; ++j)
      if (p + j < nparts) s += v[j];
  }
  G[(int64_t)c * ldg + r] = s;
  G[(int64_t)r * ldg + c] = s;
}
inline int gram_partials_reduce_blocks(int k) { return (int)(((int64_t)k * k + PR_THREADS - 1) / PR_THREADS); }

}  // namespace cqr
