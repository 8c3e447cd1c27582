// include/osmx/topk.hpp -- the reference's top-K API (proj/include/osmx/
// topk.hpp:14-68) on the B200.  topk_of / safe_softmax_then_topk /
// safe_softmax_fused_topk / online_softmax_topk run the sm_100a kernels
// through osmx_softmax_topk_host_multi / osmx_topk_host_multi; indices are
// bit-identical to the reference's (ties to the smaller index).
#pragma once

#include <cstddef>
#include <cstdint>
#include <limits>
#include <span>
#include <vector>

#include "b200_runtime.hpp"

namespace osmx {

// topk.hpp:14-17: values non-increasing, int64 positions, equal values by
// smaller index first.
struct topk_result {
  std::vector<float> values;
  std::vector<std::int64_t> indices;
};

// topk.hpp:19-50: the streaming selection buffer, kept for callers that use
// it directly (host scalar code; the device kernels hold the same list in
// registers, csrc/common.cuh TopList).  An offered value enters only if it
// beats the current k-th (strictly) or the buffer is not yet full, and then
// moves up past strictly smaller values only -- so an equal value never
// overtakes an earlier one.
class topk_buffer {
 public:
  explicit topk_buffer(std::size_t k)
      : v_(k + 1, -std::numeric_limits<float>::infinity()), i_(k + 1, -1), k_(k) {}
  std::size_t k() const { return k_; }
  float value(std::size_t rank) const { return v_[rank]; }
  std::int64_t index(std::size_t rank) const { return i_[rank]; }
  void offer(float value, std::int64_t index) {
    const bool full = i_[k_ - 1] >= 0;
    if (full && !(value > v_[k_ - 1])) return;
    std::size_t s = k_;
    while (s > 0 && v_[s - 1] < value) {  // strict: ties stay behind
      v_[s] = v_[s - 1];
      i_[s] = i_[s - 1];
      --s;
    }
    v_[s] = value;
    i_[s] = index;
  }

 private:
  std::vector<float> v_;
  std::vector<std::int64_t> i_;
  std::size_t k_;
};

namespace b200 {

constexpr int kTopkOf = -1;  // osmx_topk_host_multi

inline topk_result topk_rows(int alg, std::span<const float> x, std::size_t rows, std::size_t k,
                             const std::vector<int>& devs) {
  topk_result r;
  if (rows == 0) return r;
  const std::size_t V = x.size() / rows;
  if (V == 0) throw empty_input_error();
  if (k == 0 || k > V) throw invalid_k_error();
  r.values.resize(rows * k);
  r.indices.resize(rows * k);
  const osmx_status s =
      alg == kTopkOf
          ? osmx_topk_host_multi(x.data(), (int64_t)rows, (int64_t)V, (int32_t)k, r.values.data(),
                                 r.indices.data(), devs.data(), (int32_t)devs.size(), nullptr)
          : osmx_softmax_topk_host_multi(alg, x.data(), (int64_t)rows, (int64_t)V, (int32_t)k, r.values.data(),
                                         r.indices.data(), devs.data(), (int32_t)devs.size(), nullptr);
  throw_status(s);
  return r;
}

}  // namespace b200

// topk.hpp:54 / :58 / :63 / :68
inline topk_result topk_of(std::span<const float> values, std::size_t k) {
  return b200::topk_rows(b200::kTopkOf, values, 1, k, b200::devices());
}
inline topk_result safe_softmax_then_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_UNFUSED_TOPK, x, 1, k, b200::devices());
}
inline topk_result safe_softmax_fused_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_FUSED_TOPK, x, 1, k, b200::devices());
}
inline topk_result online_softmax_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_ONLINE_SOFTMAX_FUSED_TOPK, x, 1, k, b200::devices());
}

// Batched (rows x V row-major in, rows x k row-major out), rows sharded over
// `devs` (default: osmx::b200::devices()).
namespace batched {
inline topk_result topk_of(std::span<const float> x, std::size_t rows, std::size_t k,
                           const std::vector<int>& devs = b200::devices()) {
  return b200::topk_rows(b200::kTopkOf, x, rows, k, devs);
}
inline topk_result safe_softmax_then_topk(std::span<const float> x, std::size_t rows, std::size_t k,
                                          const std::vector<int>& devs = b200::devices()) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_UNFUSED_TOPK, x, rows, k, devs);
}
inline topk_result safe_softmax_fused_topk(std::span<const float> x, std::size_t rows, std::size_t k,
                                           const std::vector<int>& devs = b200::devices()) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_FUSED_TOPK, x, rows, k, devs);
}
inline topk_result online_softmax_topk(std::span<const float> x, std::size_t rows, std::size_t k,
                                       const std::vector<int>& devs = b200::devices()) {
  return b200::topk_rows(OSMX_ONLINE_SOFTMAX_FUSED_TOPK, x, rows, k, devs);
}
inline topk_result online_softmax_then_topk(std::span<const float> x, std::size_t rows, std::size_t k,
                                            const std::vector<int>& devs = b200::devices()) {
  return b200::topk_rows(OSMX_ONLINE_SOFTMAX_UNFUSED_TOPK, x, rows, k, devs);
}
}  // namespace batched

}  // namespace osmx
