// Cycle cost of one warp factoring an 8x8 SPD block held in registers (lane c
// owns column c), as in cqr_factor.cu's diag_block_warp, and of its pieces:
// the double rsqrt chain and the shuffle chain.  B200 sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o diag_block diag_block.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void factor8(double (&d)[8], int c, double* inv, int variant) {
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const double s = __shfl_sync(0xffffffffu, d[jj], jj);
    double aji[8];
#pragma unroll
    for (int ii = jj + 1; ii < 8; ++ii) aji[ii] = __shfl_sync(0xffffffffu, d[jj], ii);
    double r;
    if (variant == 0) r = rsqrt(s);
    else if (variant == 1) r = 1.0 / sqrt(s);
    else {   // hardware approximation + one Newton step (not exact: timing only)
      float rf = rsqrtf((float)s);
      r = (double)rf;
      r = r * (1.5 - 0.5 * s * r * r);
      r = r * (1.5 - 0.5 * s * r * r);
    }
    const double ajc = d[jj] * (r * r);
#pragma unroll
    for (int ii = jj + 1; ii < 8; ++ii)
      if (c >= ii) d[ii] -= aji[ii] * ajc;
    if (c > jj) d[jj] *= r;
    if (c == jj) d[jj] = s * r;
    if (c == 0) inv[jj] = r;
  }
}

// one thread: the 36 upper entries in registers, no shuffles
__device__ __forceinline__ constexpr int pk8(int i, int c) { return c * (c + 1) / 2 + i; }
__device__ __forceinline__ void factor8_thread(double (&a)[36], double* inv) {
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const double s = a[pk8(jj, jj)];
    const double r = rsqrt(s);
    a[pk8(jj, jj)] = s * r;
    inv[jj] = r;
#pragma unroll
    for (int c = jj + 1; c < 8; ++c) a[pk8(jj, c)] *= r;
#pragma unroll
    for (int c = jj + 1; c < 8; ++c)
#pragma unroll
      for (int i = jj + 1; i <= c; ++i) a[pk8(i, c)] -= a[pk8(jj, i)] * a[pk8(jj, c)];
  }
}

__global__ void bench_thread(double* out, long long* cyc, int reps) {
  __shared__ double blk[64], inv[8];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < 64; e += 32) { int r = e & 7, cc = e >> 3; blk[e] = (r == cc) ? 8.0 : 0.5; }
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (lane == 0) {
      double a[36];
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int i = 0; i <= c; ++i) a[pk8(i, c)] = blk[c * 8 + i];
      factor8_thread(a, inv);
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int i = 0; i <= c; ++i) blk[c * 8 + i] = (i == c) ? 8.0 : 0.5 + 1e-20 * a[pk8(i, c)];
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = (t1 - t0) / reps; out[0] = inv[3]; }
}

__global__ void bench(double* out, long long* cyc, int reps, int variant) {
  __shared__ double blk[64], inv[8];
  const int lane = threadIdx.x & 31, c = lane & 7;
  for (int e = lane; e < 64; e += 32) { int r = e & 7, cc = e >> 3; blk[e] = (r == cc) ? 8.0 : 0.5; }
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    double d[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) d[r] = blk[c * 8 + r];
    factor8(d, c, inv, variant);
    if (lane < 8) {
#pragma unroll
      for (int r = 0; r < 8; ++r) blk[c * 8 + r] = (r == c) ? 8.0 : (r < c ? 0.5 + 1e-20 * d[r] : 0.5);
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { *cyc = (t1 - t0) / reps; out[0] = inv[3]; }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
  for (int v = 0; v < 3; ++v) {
    bench<<<1, 32>>>(out, cyc, 1000, v);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"cycles_per_8x8_block\": %lld}\n",
           v == 0 ? "rsqrt(double)" : v == 1 ? "1/sqrt(double)" : "rsqrtf + 2 Newton (fp64)", c);
  }
  bench_thread<<<1, 32>>>(out, cyc, 1000);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"single thread, registers\", \"cycles_per_8x8_block\": %lld}\n", c);
  return 0;
}
