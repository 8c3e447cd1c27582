// topk_safe.cu -- safe softmax fused with top-K (reference
// safe_softmax_fused_topk_kernel, kernels.hpp:87-104): 3 passes, selection on
// the on-the-fly probability.
#include "topk_impl.cuh"

namespace osmx_host {
cudaError_t launch_topk_safe(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                             long long* idx, void* ws, cudaStream_t st, bool split) {
  return dispatch_mode<kModeSafe>(x, ldx, rows, V, k, vals, idx, ws, st, split, 0, nullptr);
}
}  // namespace osmx_host
