// HBM -> shared-memory streaming rate when each ring stage arrives as P
// separate cp.async.bulk copies (row-quad runs of a wider matrix, as the update
// pass stages Q_in) instead of one: is the cost per copy or per byte?
// One thread per CTA issues; consumers wait on the full barrier and release.
// Variants: pieces contiguous in global or strided (one piece per STRIDE
// bytes), issued by one lane or spread over the lanes of the producer warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_pieces bulk_pieces.cu
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

// stage = pieces * piece bytes; piece i of panel p comes from x + (p * pieces + i) * stride
__global__ void stream(const char* x, int64_t npanels_total, int piece, int pieces, int64_t stride, int nst,
                       int lanes, double* out) {
  extern __shared__ __align__(128) char sm[];
  const int stage = piece * pieces;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nst * stage);
  uint64_t* empty = full + nst;
  const int cw = blockDim.x / 32 - 1;   // consumer warps; the last warp produces
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cw); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t p0 = npanels_total * blockIdx.x / gridDim.x, p1 = npanels_total * (blockIdx.x + 1) / gridDim.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == cw) {
    int it = 0;
    for (int64_t p = p0; p < p1; ++p, ++it) {
      const int s = it % nst;
      if (it >= nst && lane == 0) mbar_wait(&empty[s], ((it / nst) - 1) & 1);
      __syncwarp();
      if (lane == 0) expect_tx(&full[s], stage);
      __syncwarp();
      for (int i = lane; i < pieces && lane < lanes; i += lanes)
        g2s(sm + (size_t)s * stage + (size_t)i * piece, x + (p * pieces + i) * stride, piece, &full[s]);
    }
    return;
  }
  double acc = 0;
  int it = 0;
  for (int64_t p = p0; p < p1; ++p, ++it) {
    const int s = it % nst;
    mbar_wait(&full[s], (it / nst) & 1);
    acc += reinterpret_cast<const double*>(sm + (size_t)s * stage)[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
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
  struct Cfg { int piece, pieces, strided, nst, lanes; };
  Cfg cfgs[] = {{16384, 1, 0, 8, 1}, {4096, 4, 0, 8, 1}, {2048, 8, 0, 8, 1}, {1024, 16, 0, 8, 1}, {512, 32, 0, 8, 1},
                {512, 32, 1, 8, 1}, {512, 32, 1, 8, 32}, {2048, 8, 1, 8, 1}, {2048, 8, 1, 8, 8},
                {512, 16, 1, 16, 1}, {512, 16, 1, 16, 16}, {8192, 4, 1, 6, 1}};
  for (auto c : cfgs) {
    const int stage = c.piece * c.pieces;
    // strided: one piece per 16 KB of the source (as one 512-column row quad), same total bytes read
    const int64_t stride = c.strided ? 16384 : c.piece;
    const int64_t npan = (bytes / (c.strided ? 16384 : c.piece)) / c.pieces;
    size_t smem = (size_t)c.nst * stage + 2 * c.nst * 8;
    dim3 grid(sms);
    stream<<<grid, 288, smem>>>(x, npan, c.piece, c.pieces, stride, c.nst, c.lanes, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r) stream<<<grid, 288, smem>>>(x, npan, c.piece, c.pieces, stride, c.nst, c.lanes, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const double moved = 3.0 * npan * stage;
    printf("{\"piece\": %d, \"pieces\": %d, \"strided\": %d, \"stages\": %d, \"issue_lanes\": %d, \"gbs\": %.0f, "
           "\"copies_per_us_per_sm\": %.2f, \"err\": \"%s\"}\n",
           c.piece, c.pieces, c.strided, c.nst, c.lanes, moved / (ms * 1e-3) / 1e9,
           3.0 * npan * c.pieces / (ms * 1e3) / sms, cudaGetErrorString(err));
  }
  return 0;
}
