// topk_of.cu -- top-K of arbitrary values (reference topk_kernel / topk_of,
// kernels.hpp:72-83, topk.cpp:20-28): second stage of the unfused pipelines.
#include "topk_impl.cuh"

namespace osmx_host {
cudaError_t launch_topk_of(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                           long long* idx, void* ws, cudaStream_t st, bool split) {
  return dispatch_mode<kModeTopkOf>(x, ldx, rows, V, k, vals, idx, ws, st, split, 0, nullptr);
}
}  // namespace osmx_host
