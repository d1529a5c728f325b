// HBM -> shared-memory streaming rate of a cp.async.bulk ring (no compute):
// one thread per CTA issues STAGE-byte bulk copies into an NST-deep ring,
// consumers (all warps) just wait on the full barrier and release the stage.
// Sweeps stage size, ring depth and CTAs per SM.  B200, sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_stream bulk_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(s32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(s32(d)), "l"(s), "r"(n), "r"(s32(b)) : "memory");
}

__global__ void stream(const char* x, int64_t bytes, int stage, int nst, int lag, double* out) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nst * stage);
  uint64_t* empty = full + nst;
  const int warps = blockDim.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], warps); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t npan = bytes / stage;
  const int64_t p0 = npan * blockIdx.x / gridDim.x, p1 = npan * (blockIdx.x + 1) / gridDim.x;
  const int D = nst - lag;
  if (threadIdx.x == 0)
    for (int j = 0; j < D && p0 + j < p1; ++j) { expect_tx(&full[j], stage); g2s(sm + j * stage, x + (p0 + j) * stage, stage, &full[j]); }
  double acc = 0;
  int it = 0;
  for (int64_t p = p0; p < p1; ++p, ++it) {
    const int s = it % nst;
    if (threadIdx.x == 0 && p + D < p1) {
      const int it2 = it + D, s2 = it2 % nst;
      if (it2 >= nst) mbar_wait(&empty[s2], ((it2 / nst) - 1) & 1);
      expect_tx(&full[s2], stage);
      g2s(sm + s2 * stage, x + (p + D) * stage, stage, &full[s2]);
    }
    mbar_wait(&full[s], (it / nst) & 1);
    acc += reinterpret_cast<const double*>(sm + s * stage)[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 16LL << 30;
  char* x;
  double* out;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 0, bytes);
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int stage, nst, lag, ctas_per_sm, threads; };
  Cfg cfgs[] = {{16384, 3, 1, 1, 256}, {16384, 6, 1, 1, 256}, {16384, 8, 2, 1, 256}, {16384, 12, 2, 1, 256},
                {32768, 3, 1, 1, 256}, {32768, 6, 2, 1, 256}, {65536, 3, 1, 1, 256}, {8192, 12, 2, 1, 256},
                {16384, 6, 1, 2, 256}, {16384, 4, 1, 2, 128}, {4096, 24, 2, 1, 256}};
  for (auto c : cfgs) {
    size_t smem = (size_t)c.nst * c.stage + 2 * c.nst * 8;
    dim3 grid(sms * c.ctas_per_sm);
    stream<<<grid, c.threads, smem>>>(x, bytes, c.stage, c.nst, c.lag, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) stream<<<grid, c.threads, smem>>>(x, bytes, c.stage, c.nst, c.lag, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("{\"stage\": %d, \"stages\": %d, \"lag\": %d, \"ctas_per_sm\": %d, \"in_flight_kb_per_sm\": %d, \"gbs\": %.0f, \"err\": \"%s\"}\n",
           c.stage, c.nst, c.lag, c.ctas_per_sm, (c.nst - c.lag) * c.stage * c.ctas_per_sm / 1024,
           3.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
  }
  return 0;
}
