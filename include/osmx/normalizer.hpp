// include/osmx/normalizer.hpp -- the reference's normalizer API (proj/
// include/osmx/normalizer.hpp:24-85) on the B200.
//
//   norm_state<T>, merge      host scalar types with the reference's exact
//                             arithmetic (absorb: :32-41, merge: :53-58) --
//                             the paper's Eq. 4/5 operator, kept on the host
//                             for callers that fold states themselves
//   run_normalizer<T>         the (max, sum e^(x - max)) of a vector, on the
//   run_normalizer_chunked<T> GPU (osmx_normalizer_host): T = float keeps an
//                             fp32 state, T = double a double one like the
//                             reference's kernels (kernels.hpp:65); chunked
//                             = one state per contiguous chunk, merged left
//                             to right (:77-83); one chunk == unchunked, bit
//                             for bit
//   batched::run_normalizer*  rows x V at once, rows sharded over devices
#pragma once

#include <algorithm>
#include <cmath>
#include <concepts>
#include <cstddef>
#include <limits>
#include <span>
#include <vector>

#include "b200_runtime.hpp"

namespace osmx {

template <std::floating_point T>
struct norm_state {
  T max = -std::numeric_limits<T>::infinity();  // exact running maximum
  T sum = T(0);                                 // sum of e^(x - max)

  // One element (normalizer.hpp:32-41); non-finite input throws.
  void add(T x) {
    if (!std::isfinite(x)) throw non_finite_error();
    if (!(x > max)) {
      sum += std::exp(x - max);
      return;
    }
    sum = sum * std::exp(max - x) + T(1);  // exp(-inf) = 0: the first element gives (x, 1)
    max = x;
  }
  bool is_identity() const { return max < T(0) && std::isinf(max); }
  friend bool operator==(const norm_state&, const norm_state&) = default;
};

// Eq. 4/5 merge; identity operands pass the other operand through untouched
// (normalizer.hpp:53-58).
template <std::floating_point T>
norm_state<T> merge(const norm_state<T>& a, const norm_state<T>& b) {
  if (b.is_identity()) return a;
  if (a.is_identity()) return b;
  const T top = a.max < b.max ? b.max : a.max;
  return norm_state<T>{top, a.sum * std::exp(a.max - top) + b.sum * std::exp(b.max - top)};
}

namespace b200 {

template <class T>
constexpr int precision_of() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                "the device normalizer keeps a float or a double state");
  return std::is_same_v<T, double> ? 64 : 32;
}

// chunk 0 = unchunked.
template <class T>
std::vector<norm_state<T>> normalizer_rows(std::span<const float> x, std::size_t rows, std::size_t chunk,
                                           const std::vector<int>& devs) {
  if (rows == 0) return {};
  const std::size_t V = x.size() / rows;
  if (V == 0) throw empty_input_error();
  std::vector<T> m(rows), d(rows);
  throw_status(osmx_normalizer_host(x.data(), (int64_t)rows, (int64_t)V, (int64_t)chunk, precision_of<T>(),
                                    m.data(), d.data(), devs.data(), (int32_t)devs.size(), nullptr));
  std::vector<norm_state<T>> out(rows);
  for (std::size_t r = 0; r < rows; ++r) out[r] = norm_state<T>{m[r], d[r]};
  return out;
}

}  // namespace b200

// normalizer.hpp:61-67
template <std::floating_point T>
norm_state<T> run_normalizer(std::span<const float> x) {
  if (x.empty()) throw empty_input_error();
  return b200::normalizer_rows<T>(x, 1, 0, b200::devices())[0];
}

// normalizer.hpp:73-85: validation order empty -> chunk, as the reference.
template <std::floating_point T>
norm_state<T> run_normalizer_chunked(std::span<const float> x, std::size_t chunk_len) {
  if (x.empty()) throw empty_input_error();
  if (chunk_len == 0) throw invalid_chunk_error();
  return b200::normalizer_rows<T>(x, 1, chunk_len, b200::devices())[0];
}

namespace batched {
template <std::floating_point T>
std::vector<norm_state<T>> run_normalizer(std::span<const float> x, std::size_t rows,
                                          const std::vector<int>& devs = b200::devices()) {
  return b200::normalizer_rows<T>(x, rows, 0, devs);
}
template <std::floating_point T>
std::vector<norm_state<T>> run_normalizer_chunked(std::span<const float> x, std::size_t rows, std::size_t chunk_len,
                                                  const std::vector<int>& devs = b200::devices()) {
  if (chunk_len == 0) throw invalid_chunk_error();
  return b200::normalizer_rows<T>(x, rows, chunk_len, devs);
}
}  // namespace batched

}  // namespace osmx
