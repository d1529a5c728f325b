// DMMA.8x8x4 latency / per-SMSP throughput vs independent accumulator chains
// and warps per SM sub-partition (B200, sm_100a).  One CTA on one SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_latency dmma_latency.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int NACC>
__global__ void chains(double* out, long long* cycles, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cycles = t1 - t0;
}

template <int NACC>
void run(double* out, long long* dcyc, int warps) {
  const int iters = 4096;
  chains<NACC><<<1, 32 * warps>>>(out, dcyc, iters, 1.0);
  chains<NACC><<<1, 32 * warps>>>(out, dcyc, iters, 1.0);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double per_smsp = (double)iters * NACC * ((warps + 3) / 4);   // DMMAs issued on the busiest SMSP
  printf("{\"warps\": %d, \"chains_per_warp\": %d, \"cycles_per_dmma_per_smsp\": %.2f, \"cycles_per_chain_step\": %.1f}\n",
         warps, NACC, cyc / per_smsp, (double)cyc / iters);
}

int main() {
  double* out;
  long long* dcyc;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&dcyc, sizeof(long long));
  for (int w : {1, 4, 8, 12, 16}) {
    run<1>(out, dcyc, w);
    run<2>(out, dcyc, w);
    run<4>(out, dcyc, w);
    run<8>(out, dcyc, w);
    run<16>(out, dcyc, w);
  }
  return 0;
}
