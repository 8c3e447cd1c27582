// topk.cu -- dispatch of the batched top-K family and the record (V-split)
// entry points.  Kernels live in topk_impl.cuh; one translation unit per
// selection mode (topk_fused.cu, topk_of.cu, topk_safe.cu) so they build in
// parallel.
#include "topk_impl.cuh"

namespace osmx_host {

cudaError_t launch_topk_fused(const float*, long long, long long, long long, int, float*, long long*, void*,
                              cudaStream_t, bool, long long, char*);
cudaError_t launch_topk_of(const float*, long long, long long, long long, int, float*, long long*, void*,
                           cudaStream_t, bool);
cudaError_t launch_topk_safe(const float*, long long, long long, long long, int, float*, long long*, void*,
                             cudaStream_t, bool);

size_t record_bytes(int k) { return rec_bytes_(k); }

size_t topk_split_ws(int alg, long long rows, long long V, int k) {
  const long long ch = topk_split_chunk(rows, V);
  const long long S = (V + ch - 1) / ch;
  const long long pc = topk_piece_chunk(rows, V);
  const long long R = (V + pc - 1) / pc;  // warp-per-piece records (fused / topk_of)
  // + the first-level records of the two-level combine (R >= 1024).  The
  // TMA-ring pieces (split_cta = 2) are never more: >= 16K elements over at
  // most 28 resident CTAs per SM.
  size_t b = (size_t)(rows * std::max(S, R + (R + 255) / 256)) * rec_bytes_(k);
  // one-launch wide rows: rows x (resident CTAs / rows) records
  if (topk_wide_ok(rows, V)) b = std::max(b, (size_t)std::max(topk_wide_slots(k), rows) * rec_bytes_(k));
  if (alg == kSafeFusedTopk) b += ((size_t)(rows * S) * sizeof(SRecView) + 255) / 256 * 256;
  return b;
}
bool topk_split(long long rows, long long V) { return topk_uses_split(rows, V); }

cudaError_t launch_topk_tma(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                            float* vals, long long* idx, void* ws, cudaStream_t st);

bool topk_uses_tma(int mode, long long rows, long long V) {
  const auto& tn = tuning();
  if (mode == kModeSafe || tn.tma == 0) return false;
  if (tn.shape == kShapeSplit || tn.shape == kShapeResident) return false;
  if (tn.tma == 2) return true;
  return V >= 8192 && rows >= num_sms() && !topk_uses_split(rows, V);
}

cudaError_t launch_topk_mode(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                             float* vals, long long* idx, void* ws, cudaStream_t st) {
  if (k > kMaxK)
    return launch_topk_large(mode, x, ldx, rows, V, k, vals, idx, ws, static_cast<char*>(ws) + kWsHeader, st);
  const bool split = topk_uses_split(rows, V);
  if (topk_uses_tma(mode, rows, V)) return launch_topk_tma(mode, x, ldx, rows, V, k, vals, idx, ws, st);
  switch (mode) {
    case kModeFused: return launch_topk_fused(x, ldx, rows, V, k, vals, idx, ws, st, split, 0, nullptr);
    case kModeTopkOf: return launch_topk_of(x, ldx, rows, V, k, vals, idx, ws, st, split);
    case kModeSafe: return launch_topk_safe(x, ldx, rows, V, k, vals, idx, ws, st, split);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_slice_record(const float* x, long long V, long long col0, int k, void* record,
                                void* ws, size_t, cudaStream_t st) {
  // Always the split path: chunk records, then one combined record.
  const int kk = k > 0 ? k : 1;
  return launch_topk_fused(x, V, 1, V, kk, nullptr, nullptr, ws, st, true, col0, static_cast<char*>(record));
}

cudaError_t launch_records_combine(const void* records, int n, int k, void* out_record, float* vals,
                                   long long* idx, void* ws, cudaStream_t st) {
  const int kk = k > 0 ? k : 1;
  if (k == 0) vals = nullptr, idx = nullptr;
  if (kk <= 1) return combine_kc<1>(records, n, kk, out_record, vals, idx, ws, st);
  if (kk <= 5) return combine_kc<5>(records, n, kk, out_record, vals, idx, ws, st);
  if (kk <= 8) return combine_kc<8>(records, n, kk, out_record, vals, idx, ws, st);
  if (kk <= 16) return combine_kc<16>(records, n, kk, out_record, vals, idx, ws, st);
  return combine_kc<32>(records, n, kk, out_record, vals, idx, ws, st);
}

}  // namespace osmx_host

// ------------------------------------------------- scale against record --
namespace {
template <int BLOCK, int U>
__global__ void __launch_bounds__(BLOCK)
    k_scale_with_record(const float* __restrict__ x, long long V, const RecHdr* __restrict__ rec,
                        float* __restrict__ y) {
  const RecHdr h = *rec;
  const float M = h.m;
  const Recip R = recip_of((double)h.d);
  const long long per = (V + gridDim.x - 1) / gridDim.x;
  const long long chunk = (per + 15) / 16 * 16;
  const long long c0 = (long long)blockIdx.x * chunk;
  if (c0 >= V) return;
  const long long n = std::min(chunk, V - c0);
  const Seg s = make_seg(x + c0, n);
  map_seg<BLOCK, U>(s, y + c0, threadIdx.x, [&](float v) { return out_md(v, M, R); });
}
}  // namespace

namespace osmx_host {
cudaError_t launch_scale_with_record(const float* x, long long V, const void* record, float* y,
                                     cudaStream_t st) {
  const long long want = (V + 32767) / 32768;
  const long long grid = std::max<long long>(1, std::min<long long>(want, 8LL * num_sms()));
  k_scale_with_record<512, 4><<<(unsigned)grid, 512, 0, st>>>(x, V, static_cast<const RecHdr*>(record), y);
  count_launch();
  return cudaGetLastError();
}
}  // namespace osmx_host

// ------------------------------------------------- diagnostic read probe --
namespace {
__global__ void __launch_bounds__(256) k_read_probe(const float4* __restrict__ p, size_t n, float* sink) {
  constexpr int U = 16;
  float m = kNegInf;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_f4(reinterpret_cast<const float*>(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
  }
  for (; i < n; i += stride) m = fmaxf(m, p[i].x);
  if (m == 12345.678f) *sink = m;  // never true: keeps the loads
}
}  // namespace

namespace osmx_host {
cudaError_t launch_read_probe(const void* x, size_t bytes, float* sink, cudaStream_t st) {
  k_read_probe<<<(unsigned)(4 * num_sms()), 256, 0, st>>>(static_cast<const float4*>(x), bytes / 16, sink);
  count_launch();
  return cudaGetLastError();
}
}  // namespace osmx_host
