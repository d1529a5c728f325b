// Fused TRMM + Gram pass (K2) -- placeholder until the fused kernel lands;
// cqr_apply_gram falls back to the row-panel GEMM followed by the Gram kernel.
#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace cqr {

bool apply_gram_fused_supported(int) { return false; }
size_t apply_gram_fused_ws_bytes(int64_t, int) { return 0; }
cudaError_t apply_gram_fused_launch(const double*, int64_t, int, const double*, double*, int64_t, int64_t,
                                    double*, int, double*, size_t, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace cqr
