// Native enqueue of the fixed schedules (chol_qr, chol_qr2, s_chol_qr3;
// reference algorithms.py:201-244) and their CUDA-graph replay.
//
// The fixed schedules take no host decision between passes, so the whole run
// -- Racc reset, Gram, then per pass the k x k stage and the TRMM (+ next
// Gram), then R's download -- is enqueued by ONE ABI call through the same
// entry points the per-call API uses (bitwise the same kernels and
// arguments).  With use_graph the run is captured once per plan (every plan
// and factor-config field is the key) and replayed with cudaGraphLaunch:
// config 1 (200k x 64) spends more host time launching ~10 kernels through
// Python than the GPU spends on several of them.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace {

constexpr size_t kStatusBytes = 96;   // sizeof(cqr_factor_status) rounded to 16 (shifts follow)
constexpr size_t kMaxGraphs = 32;

struct GraphEntry {
  int dev;
  std::vector<unsigned char> key;
  cudaGraphExec_t exec;
  unsigned long long last;
};

std::mutex g_mu;
std::vector<GraphEntry> g_graphs;
unsigned long long g_tick = 0;
cudaStream_t g_capture[64] = {};

int enqueue(const cqr_fixed_plan& p, cudaStream_t s) {
  const int k = p.k;
  const size_t racc_bytes = (size_t)k * p.ldr * sizeof(double);
  if (p.Racc0 != p.Racc) {
    cudaError_t e = cudaMemcpyAsync(p.Racc, p.Racc0, racc_bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cqr::set_error(CQR_ECUDA, std::string("cqr_fixed_schedule: Racc reset: ") +
                                                               cudaGetErrorString(e));
  }
  int rc = cqr_gram(p.X, p.ldx, p.m, k, p.G, k, p.ws, p.ws_bytes, s);
  if (rc) return rc;
  const double* src = p.X;
  int64_t lds = p.ldx;
  for (int i = 0; i < p.passes; ++i) {
    char* base = static_cast<char*>(p.status[i]);
    rc = cqr_factor(p.fcfg[i], k, p.G, k, nullptr, 1, 0, p.Rk, p.Rinv, p.ldr, p.Racc, nullptr, 1,
                    reinterpret_cast<double*>(base + kStatusBytes), reinterpret_cast<cqr_factor_status*>(base),
                    p.fws, p.fws_bytes, s);
    if (rc) return rc;
    if (i + 1 < p.passes)
      rc = cqr_apply_gram(src, lds, p.m, k, p.Rinv, p.dst[i], p.lddst[i], p.G, k, p.ws, p.ws_bytes, s);
    else
      rc = cqr_lincomb(src, lds, p.m, k, p.Rinv, k, 1, p.dst[i], p.lddst[i], s);
    if (rc) return rc;
    src = p.dst[i];
    lds = p.lddst[i];
  }
  if (p.R_host != nullptr) return cqr_store_to_host(p.Racc, (int64_t)k * p.ldr, p.R_host, s);
  return CQR_OK;
}

std::vector<unsigned char> plan_key(const cqr_fixed_plan& p, int dev) {
  std::vector<unsigned char> key(sizeof(int) + sizeof(p) + p.passes * sizeof(cqr_factor_config));
  unsigned char* w = key.data();
  std::memcpy(w, &dev, sizeof(int));
  w += sizeof(int);
  std::memcpy(w, &p, sizeof(p));
  w += sizeof(p);
  for (int i = 0; i < p.passes; ++i, w += sizeof(cqr_factor_config))
    std::memcpy(w, p.fcfg[i], sizeof(cqr_factor_config));
  return key;
}

}  // namespace

extern "C" {

int cqr_fixed_graphs(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int)g_graphs.size();
}

int cqr_fixed_schedule(const cqr_fixed_plan* plan, void* stream) {
  if (plan == nullptr) return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: null plan");
  cqr_fixed_plan p;
  std::memcpy(&p, plan, sizeof(p));   // the key covers padding bytes too: start from the caller's bytes
  if (p.passes < 1 || p.passes > CQR_FIXED_MAX_PASSES)
    return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: passes must be 1..3");
  if (p.k < 1 || p.m < 1) return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: empty shape");
  if (p.Racc == nullptr || p.Racc0 == nullptr || p.G == nullptr || p.ldr < p.k)
    return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: bad k x k buffers");
  for (int i = 0; i < p.passes; ++i) {
    if (p.fcfg[i] == nullptr || p.status[i] == nullptr || p.dst[i] == nullptr)
      return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: pass without config / status / destination");
    if (p.fcfg[i]->policy != CQR_POLICY_PLAIN && p.fcfg[i]->policy != CQR_POLICY_SHIFT_ONCE &&
        p.fcfg[i]->policy != CQR_POLICY_FIXED_SHIFT)
      return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: only the fixed policies (plain, shift-once, fixed shift)");
    if (p.fcfg[i]->gate != nullptr) return cqr::set_error(CQR_EINVAL, "cqr_fixed_schedule: gated factor calls");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!p.use_graph) return enqueue(p, s);

  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return enqueue(p, s);
  }
  std::vector<unsigned char> key = plan_key(p, dev);
  std::lock_guard<std::mutex> lk(g_mu);
  for (GraphEntry& g : g_graphs) {
    if (g.dev == dev && g.key == key) {
      g.last = ++g_tick;
      cudaError_t e = cudaGraphLaunch(g.exec, s);
      if (e != cudaSuccess)
        return cqr::set_error(CQR_ECUDA, std::string("cqr_fixed_schedule: graph launch: ") + cudaGetErrorString(e));
      return CQR_OK;
    }
  }
  // capture on a private stream (the caller's may be the legacy default stream,
  // which cannot be captured); the graph is then launched on the caller's
  if (g_capture[dev] == nullptr && cudaStreamCreateWithFlags(&g_capture[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    g_capture[dev] = nullptr;
    return enqueue(p, s);
  }
  cudaStream_t cs = g_capture[dev];
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    return enqueue(p, s);
  }
  const int rc = enqueue(p, cs);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(cs, &graph);
  if (rc != CQR_OK) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return rc;   // argument errors: nothing was enqueued on the caller's stream
  }
  cudaGraphExec_t exec = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return enqueue(p, s);   // not capturable here: run the same schedule directly
  }
  if (g_graphs.size() >= kMaxGraphs) {
    size_t lru = 0;
    for (size_t i = 1; i < g_graphs.size(); ++i)
      if (g_graphs[i].last < g_graphs[lru].last) lru = i;
    // a launched graph may still be running: let it finish before its exec goes
    cudaDeviceSynchronize();
    cudaGraphExecDestroy(g_graphs[lru].exec);
    g_graphs.erase(g_graphs.begin() + (long)lru);
  }
  g_graphs.push_back(GraphEntry{dev, std::move(key), exec, ++g_tick});
  e = cudaGraphLaunch(exec, s);
  if (e != cudaSuccess)
    return cqr::set_error(CQR_ECUDA, std::string("cqr_fixed_schedule: graph launch: ") + cudaGetErrorString(e));
  return CQR_OK;
}

}  // extern "C"
