// Shared device helpers for the fp64 Cholesky-QR kernels (sm_100a).
//
// FP64 tensor work uses warp-level mma.sync .f64 (SASS DMMA.8x8x4): on
// sm_100a tcgen05 has no f64 kind, and the measured DMMA peak (37.2 TF/s on
// this pool's B200s, profiles/r01_fp64_peak.json) equals the DFMA peak, so the
// 8x8x4 DMMA is the fp64 tensor path.  Row panels are staged in shared memory
// by cp.async.bulk (the TMA bulk-copy engine, SASS UBLKCP) against mbarriers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cqr {

// ---------------------------------------------------------------- DMMA 8x8x4
// C[8x8] += A[8x4] * B[4x8].  Fragment ownership (lane = 4*g + t):
//   a = A[g][t], b = B[t][g], c[e] = C[g][2t+e].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy (TMA engine), completion counted on an mbarrier.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global bulk copy (TMA engine); tracked with bulk async-groups.
// 3-D TMA tensor copy (box of a CUtensorMap in param / const / global space) -> shared memory
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_stream(void* dst, const void* src, uint32_t bytes) {
#if CQR_L2_HINTS
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(l2_evict_first())
               : "memory");
#else
  bulk_s2g(dst, src, bytes);
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Streaming tall operands (X, Q panels: read or written once per pass) carry
// an L2 evict-first hint, so a pass that streams gigabytes through the 126 MB
// L2 does not evict what the next kernels reuse: the k x k stage's code (the
// factor kernel is ~1 MB of SASS; fetched cold from HBM it ran 16-37 us
// slower per call after a tall pass, tools/diag/factor_cold.py), its Gram and
// the coefficient tiles.  CQR_L2_HINTS=0 at build time turns the hints off.
#ifndef CQR_L2_HINTS
#define CQR_L2_HINTS 1
#endif
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#if CQR_L2_HINTS
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first())
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}
__device__ __forceinline__ void tma_load_3d_stream(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
#if CQR_L2_HINTS
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(l2_evict_first())
      : "memory");
#else
  tma_load_3d(dst, tmap, c0, c1, c2, bar);
#endif
}
// one streamed fp64 store (st.global.cs: evict-first in L2)
__device__ __forceinline__ void st_stream(double* p, double v) {
#if CQR_L2_HINTS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// make generic-proxy shared-memory writes visible to the async (bulk) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- misc
__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ constexpr int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------- layouts (include/cqr.h)
// QI tall layout: element (r, c) of an array with column capacity ldk
__host__ __device__ __forceinline__ int64_t qi_off(int64_t r, int64_t c, int64_t ldk) {
  return (r >> 2) * 4 * ldk + 4 * c + (r & 3);
}
// coefficient tiles: 32 (k) x 64 (n) tiles, each [64][36] (4 padding doubles per
// column keep the DMMA B-fragment loads bank-conflict free)
constexpr int CT_K = 32, CT_N = 64, CT_LD = 36, CT_TILE = CT_N * CT_LD;
__host__ __device__ constexpr int64_t coeff_tiles_doubles(int k, int n) {
  return ceil_div(k, CT_K) * ceil_div(n, CT_N) * CT_TILE;
}
__host__ __device__ __forceinline__ int64_t coeff_off(int kk, int nn, int k) {
  const int64_t nkt = ceil_div(k, CT_K);
  return ((nn / CT_N) * nkt + kk / CT_K) * CT_TILE + (nn % CT_N) * CT_LD + kk % CT_K;
}

// Python's max(a, b): returns b only when b > a, so a NaN first argument wins
// (kernels.py:194, algorithms.py:317,396 rely on this for NaN propagation).
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }

}  // namespace cqr
