// softmax_safe.cu -- Alg. 2 (reference safe_softmax_kernel, kernels.hpp:49-58),
// plus the safe split statistics used by the safe fused top-K.
#include "softmax_impl.cuh"

namespace osmx_host {
cudaError_t launch_softmax_safe(const float* x, long long ldx, float* y, long long ldy, long long rows,
                                long long V, void* ws, cudaStream_t st) {
  return launch_alg<kSafe>(x, ldx, y, ldy, rows, V, ws, st);
}

cudaError_t launch_safe_split_stats(const float* x, long long ldx, long long rows, long long V,
                                    long long chunk, void* srec, cudaStream_t st) {
  const long long S = (V + chunk - 1) / chunk;
  dim3 grid((unsigned)S, (unsigned)rows);
  SRec* rec = static_cast<SRec*>(srec);
  k_softmax_split_part<kSplitBlock, kSplitU, kSafe, 0><<<grid, kSplitBlock, 0, st>>>(x, ldx, V, chunk, rec);
  k_softmax_split_part<kSplitBlock, kSplitU, kSafe, 2><<<grid, kSplitBlock, 0, st>>>(x, ldx, V, chunk, rec);
  count_launch(2);
  return cudaGetLastError();
}
}  // namespace osmx_host
