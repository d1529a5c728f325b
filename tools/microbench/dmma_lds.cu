// DMMA.8x8x4 throughput when operands stream from shared memory: per k4
// step a warp loads NA A-fragments and NB B-fragments (LDS.64 each, conflict
// free) and issues NA*NB DMMAs into NA*NB accumulators.  8 warps on one SM
// (2 per SM sub-partition), as in the tall kernels.  Reports cycles per DMMA
// per SMSP (16.0 = the measured pipe peak).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lds dmma_lds.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NA, int NB>
__global__ void lds_dmma(double* out, long long* cycles, int iters) {
  __shared__ double sm[NA + NB][4 * 32];   // fragments for 4 k4 steps (shared by the warps)
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (NA + NB) * 128; i += blockDim.x) (&sm[0][0])[i] = 1.0 + 1e-9 * i;
  double c[NA][NB][2];
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) { c[i][j][0] = 0; c[i][j][1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int ks = it & 3;
    double a[NA], b[NB];
#pragma unroll
    for (int i = 0; i < NA; ++i) a[i] = sm[i][ks * 32 + lane];
#pragma unroll
    for (int j = 0; j < NB; ++j) b[j] = sm[NA + j][ks * 32 + lane];
#pragma unroll
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.678) out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cycles = t1 - t0;
}

template <int NA, int NB>
void run(double* out, long long* dc, int warps) {
  const int iters = 8192;
  lds_dmma<NA, NB><<<1, 32 * warps>>>(out, dc, iters);
  lds_dmma<NA, NB><<<1, 32 * warps>>>(out, dc, iters);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double per_smsp = (double)iters * NA * NB * (warps / 4);
  printf("{\"warps\": %d, \"a_frags\": %d, \"b_frags\": %d, \"lds_per_dmma\": %.3f, \"cycles_per_dmma_per_smsp\": %.2f}\n",
         warps, NA, NB, (double)(NA + NB) / (NA * NB), cyc / per_smsp);
}

int main() {
  double* out;
  long long* dc;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&dc, sizeof(long long));
  for (int w : {4, 8}) {
    run<4, 1>(out, dc, w);
    run<4, 2>(out, dc, w);
    run<4, 4>(out, dc, w);
    run<2, 4>(out, dc, w);
    run<1, 8>(out, dc, w);
    run<1, 16>(out, dc, w);
    run<4, 8>(out, dc, w);
  }
  return 0;
}
