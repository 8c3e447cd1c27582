// softmax.cu -- dispatch of the batched softmax family (kernels in
// softmax_impl.cuh; one translation unit per algorithm so they build in
// parallel: softmax_naive.cu, softmax_safe.cu, softmax_online.cu).
#include "softmax_impl.cuh"

namespace osmx_host {

cudaError_t launch_softmax_naive(const float*, long long, float*, long long, long long, long long, void*, cudaStream_t);
cudaError_t launch_softmax_safe(const float*, long long, float*, long long, long long, long long, void*, cudaStream_t);
cudaError_t launch_softmax_online(const float*, long long, float*, long long, long long, long long, void*, cudaStream_t);

size_t softmax_split_ws(long long rows, long long V) {
  const long long ch = split_chunk(rows, V);
  const long long S = (V + ch - 1) / ch;
  return (size_t)(rows * S) * sizeof(SRec);
}

int resident_limit(bool vec) {
  // Rows that are not 16-byte aligned go to the staged ring earlier (its
  // phase-offset slots keep them vectorised): 4000 rows, V = 1778: staged
  // 0.0156 ms vs resident 0.0188; V = 1023: resident 0.0132 vs 0.0147.
  const int r = tuning().resident_max_v;
  return vec ? r : std::min(r, 1536);
}

// Conservative (workspace sizing does not know the pointers' alignment).
bool softmax_uses_split(long long rows, long long V) {
  const auto& tn = tuning();
  if (tn.shape == kShapeSplit) return rows <= 65535;
  if (tn.shape != kShapeAuto) return false;
  return V > std::max<long long>(resident_limit(false), kStagedMaxV) && rows < 2LL * num_sms();
}

cudaError_t launch_softmax(int alg, const float* x, long long ldx, float* y, long long ldy,
                           long long rows, long long V, void* ws, size_t, cudaStream_t st) {
  switch (alg) {
    case kNaive: return launch_softmax_naive(x, ldx, y, ldy, rows, V, ws, st);
    case kSafe: return launch_softmax_safe(x, ldx, y, ldy, rows, V, ws, st);
    case kOnline: return launch_softmax_online(x, ldx, y, ldy, rows, V, ws, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace osmx_host
