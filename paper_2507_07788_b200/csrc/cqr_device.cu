// Per-device host state of libcqr: the SM count and the one-time kernel
// attributes (dynamic shared-memory opt-in).  Both are kept per device
// ordinal, so one process may drive several GPUs (a single-process multi-GPU
// host, or a rank that switches devices) without a stale cache.
#include <mutex>
#include <unordered_map>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

namespace {
constexpr int MAX_DEV = 64;
std::mutex g_mu;
int g_sms[MAX_DEV] = {};
std::unordered_map<const void*, size_t> g_attr[MAX_DEV];

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < MAX_DEV) ? dev : 0;
}
}  // namespace

int num_sms() {
  const int dev = current_device();
  int n = g_sms[dev];
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    g_sms[dev] = n;
  }
  return n;
}

cudaError_t smem_attr(const void* fn, size_t bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_attr[dev].find(fn);
  if (it != g_attr[dev].end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) g_attr[dev][fn] = bytes;
  return e;
}

}  // namespace cqr
