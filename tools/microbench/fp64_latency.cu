// Dependent-chain latency (cycles) of scalar FP64 ops and 64-bit shuffles for
// one warp on B200 (sm_100a).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, int n, double seed) {
  double x = seed + threadIdx.x, y = 1.0 - 1e-13;
  long long t[8];
  t[0] = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);                 // DFMA chain
  t[1] = clock64();
  for (int i = 0; i < n; ++i) x = x * y;                           // DMUL chain
  t[2] = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);   // SHFL x2 (64-bit)
  t[3] = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x * x + 1.0);              // rsqrt chain (+ DFMA)
  t[4] = clock64();
  float f = (float)x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.999f, 1e-6f);          // FFMA chain
  t[5] = clock64();
  for (int i = 0; i < n; ++i) f = __shfl_sync(0xffffffffu, f, (threadIdx.x + 1) & 31);  // SHFL 32-bit
  t[6] = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) cyc[k] = (t[k + 1] - t[k]) / n;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8 * 8);
  chain<<<1, 32>>>(out, cyc, 4096, 1.0);
  chain<<<1, 32>>>(out, cyc, 4096, 1.0);
  cudaDeviceSynchronize();
  long long c[6]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("{\"dfma\": %lld, \"dmul\": %lld, \"shfl64\": %lld, \"rsqrt64_plus_dfma\": %lld, \"ffma\": %lld, \"shfl32\": %lld}\n",
         c[0], c[1], c[2], c[3], c[4], c[5]);
  return 0;
}
