// softmax_online.cu -- Alg. 3 (reference online_softmax_kernel,
// kernels.hpp:61-69) and the batched normalizer (normalizer.hpp:61-85).
#include "softmax_impl.cuh"

namespace osmx_host {
cudaError_t launch_softmax_online(const float* x, long long ldx, float* y, long long ldy, long long rows,
                                  long long V, void* ws, cudaStream_t st) {
  return launch_alg<kOnline>(x, ldx, y, ldy, rows, V, ws, st);
}

cudaError_t launch_normalizer_f32_tree(const float* x, long long ldx, long long rows, long long V, float* m,
                                       float* d, void* ws, cudaStream_t st) {
  const long long grid = std::min<long long>(rows, 1LL << 30);
  k_normalizer<256, 4><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, m, d, ws);
  count_launch();
  return cudaGetLastError();
}
}  // namespace osmx_host
