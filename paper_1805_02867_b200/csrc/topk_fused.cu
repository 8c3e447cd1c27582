// topk_fused.cu -- Alg. 4, fused online softmax + top-K (reference
// online_softmax_topk_kernel, kernels.hpp:108-125): one access per element.
#include "topk_impl.cuh"

namespace osmx_host {
cudaError_t launch_topk_fused(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                              long long* idx, void* ws, cudaStream_t st, bool split, long long col0,
                              char* out_rec) {
  return dispatch_mode<kModeFused>(x, ldx, rows, V, k, vals, idx, ws, st, split, col0, out_rec);
}
}  // namespace osmx_host
