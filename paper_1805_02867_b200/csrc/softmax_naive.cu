// softmax_naive.cu -- Alg. 1 (reference naive_softmax_kernel, kernels.hpp:39-46).
#include "softmax_impl.cuh"

namespace osmx_host {
cudaError_t launch_softmax_naive(const float* x, long long ldx, float* y, long long ldy, long long rows,
                                 long long V, void* ws, cudaStream_t st) {
  return launch_alg<kNaive>(x, ldx, y, ldy, rows, V, ws, st);
}
}  // namespace osmx_host
