// Global <-> shared traffic of ONE CTA (384 threads, ~200 KB shared memory,
// i.e. one CTA on one SM, as in the single-CTA k x k factorization) with data
// resident in L2: plain loads / stores against cp.async.bulk copies.
//   mode 0: ld.global.nc, coalesced, 8 loads in flight per thread -> smem
//   mode 1: generic-pointer loads (LD.E), same pattern
//   mode 2: generic loads, 64-byte runs (an 8-row block column per 8 lanes)
//   mode 3: cp.async.bulk global -> shared, 16 KB per copy, all issued at once
//   mode 4: coalesced plain stores shared -> global
//   mode 5: cp.async.bulk shared -> global, 16 KB per copy
//   mode 6: shared -> shared copy through generic pointers (LD.E / ST.E)
//   mode 7: the same through shared-window pointers (LDS / STS)
//   mode 8: coherent ld.global (LDG without .nc), as mode 0
// Prints cycles and bytes per cycle for each.  B200, sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o single_sm_io single_sm_io.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(384, 1) io(double* g, int n, int mode, const double* volatile* gp,
                                             unsigned long long* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(s32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long t0 = clock64();
  if (mode == 0) {
    const double* __restrict__ src = g;
    for (int base = tid; base < n; base += 8 * 384) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int e = base + u * 384; v[u] = e < n ? __ldg(src + e) : 0.0; }
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int e = base + u * 384; if (e < n) sm[e] = v[u]; }
    }
  } else if (mode == 1 || mode == 2) {
    const double* src = *gp;   // opaque: the compiler cannot tell global from shared
    for (int base = tid; base < n; base += 8 * 384) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * 384;
        // mode 2: runs of 8 doubles, successive runs 2 KB apart
        const int a = mode == 1 ? e : ((e >> 3) % 32) * 256 + ((e >> 8) * 8) + (e & 7);
        v[u] = e < n ? src[a % n] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int e = base + u * 384; if (e < n) sm[e] = v[u]; }
    }
  } else if (mode == 3) {
    const int bytes = n * 8, chunk = 16384;
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bytes) : "memory");
      for (int o = 0; o < bytes; o += chunk) {
        const int c = min(chunk, bytes - o);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s32(reinterpret_cast<char*>(sm) + o)), "l"(reinterpret_cast<char*>(g) + o), "r"(c),
                     "r"(s32(&bar)) : "memory");
      }
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(s32(&bar)), "r"(0) : "memory");
  } else if (mode == 4) {
    for (int e = tid; e < n; e += 384) g[e] = sm[e];
  } else if (mode == 5) {
    const int bytes = n * 8, chunk = 16384;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      for (int o = 0; o < bytes; o += chunk) {
        const int c = min(chunk, bytes - o);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(reinterpret_cast<char*>(g) + o), "r"(s32(reinterpret_cast<char*>(sm) + o)), "r"(c)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (mode == 8) {
    for (int base = tid; base < n; base += 8 * 384) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int e = base + u * 384; v[u] = e < n ? g[e] : 0.0; }
#pragma unroll
      for (int u = 0; u < 8; ++u) { const int e = base + u * 384; if (e < n) sm[e] = v[u]; }
    }
  } else if (mode == 6 || mode == 7) {
    // copy the first half of the shared buffer onto the second half, 8 in flight
    const int h = n / 2;
    double* gsrc = (mode == 6 && *gp == nullptr) ? g : sm;   // opaque when mode 6
    for (int base = tid; base < h; base += 8 * 384) {
      double v[8];
      if (mode == 6) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = base + u * 384; v[u] = e < h ? gsrc[e] : 0.0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = base + u * 384; if (e < h) gsrc[h + e] = v[u]; }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = base + u * 384; v[u] = e < h ? sm[e] : 0.0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = base + u * 384; if (e < h) sm[h + e] = v[u]; }
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (tid == 0) out[0] = (unsigned long long)(t1 - t0);
  if ((mode < 4 || mode == 8) && sm[tid] == 1234.5) g[0] = 0.0;
}

int main() {
  const int ns[] = {8192, 18432, 25600};
  double* g;
  const double** gp;
  unsigned long long* out;
  cudaMalloc(&g, 32 << 20);
  cudaMalloc(&gp, sizeof(double*));
  cudaMemcpy(gp, &g, sizeof(double*), cudaMemcpyHostToDevice);
  cudaMallocManaged(&out, 8);
  cudaMemset(g, 0, 32 << 20);
  const int smem = 205 * 1024;
  cudaFuncSetAttribute(io, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"ldg", "generic_ld", "generic_ld_runs64", "bulk_g2s", "stg", "bulk_s2g", "generic_smem_copy", "lds_sts_copy", "ldg_coherent"};
  for (int n : ns)
    for (int mode = 0; mode < 9; ++mode) {
      unsigned long long best = ~0ull;
      for (int r = 0; r < 5; ++r) {
        io<<<1, 384, smem>>>(g, n, mode, (const double* volatile*)gp, out);
        cudaDeviceSynchronize();
        if (out[0] < best) best = out[0];
      }
      printf("{\"mode\": \"%s\", \"bytes\": %d, \"cycles\": %llu, \"bytes_per_cycle\": %.1f}\n", names[mode], n * 8,
             best, n * 8.0 / best);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
