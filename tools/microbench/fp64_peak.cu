// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64 -> DMMA.8x8x4),
// DFMA, and both interleaved, plus an HBM read / copy bandwidth probe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NCH>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// even warps DMMA, odd warps DFMA (same per-warp iteration counts scaled so
// both finish at about the same time if the pipes are independent)
__global__ void mixed_loop(double* out, int iters, int fma_iters, double seed) {
  int w = threadIdx.x / 32;
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double s = 0;
  if ((w & 1) == 0) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    double bb = 1.0 - 1e-12;
    for (int it = 0; it < fma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], bb, a);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(in + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}
__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ o, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(o + i, __ldcs(in + i));
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int threads = 256;
  // DMMA
  for (int bpsm : {1, 2, 4}) {
    int iters = 20000, blocks = sms * bpsm;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    printf(", \"dmma_tflops_bpsm%d\": %.2f", bpsm, flops / (ms * 1e-3) / 1e12);
  }
  // DFMA
  for (int bpsm : {2, 4, 8}) {
    int iters = 20000, blocks = sms * bpsm;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf(", \"dfma_tflops_bpsm%d\": %.2f", bpsm, flops / (ms * 1e-3) / 1e12);
  }
  // mixed: DMMA warp does 8*256 FMA/iter, DFMA warp 8*32 FMA/iter
  for (int ratio : {4, 8}) {
    int iters = 10000, blocks = sms * 2;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      mixed_loop<<<blocks, threads>>>(out, iters, iters * ratio, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double warps = (threads / 32) * blocks / 2.0;
    double flops = warps * 2.0 * (256.0 * 8 * iters + 32.0 * 8 * iters * ratio);
    printf(", \"mixed_tflops_ratio%d\": %.2f", ratio, flops / (ms * 1e-3) / 1e12);
  }
  // HBM
  size_t bytes = (size_t)4 << 30; size_t n2 = bytes / 16;
  double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); read_kernel<<<sms * 8, 512>>>(a, n2, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"hbm_read_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
  best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"hbm_copy_gbs\": %.1f}\n", 2.0 * bytes / (best * 1e-3) / 1e9);
  return 0;
}
