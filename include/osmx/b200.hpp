// include/osmx/b200.hpp -- the reference's C++ API (proj/include/osmx/*.hpp)
// re-exposed over the B200 C-ABI (include/osmx_b200.h).
//
// Same namespace, names, argument meaning, return types and exception types
// as the reference, so a caller of
//     osmx::online_softmax(std::span<const float>)          softmax.hpp:28
//     osmx::online_softmax_topk(std::span<const float>, k)  topk.hpp:68
// switches by including this header and linking libosmx_b200.so instead of
// the reference's libosmx.a.  Every call runs on the GPU (device 0 unless
// osmx::b200::set_device is called); there is no CPU path.
//
// Batched overloads take a row-major batch (rows x V) and return a row-major
// result, the form the reference's bench harness drives row by row
// (bench.cpp:34-96).
#pragma once

#include <cstddef>
#include <cstdint>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../osmx_b200.h"

namespace osmx {

// error.hpp:8-25 -- identical types and messages.
struct empty_input_error : std::invalid_argument {
  empty_input_error() : std::invalid_argument("empty input vector") {}
};
struct non_finite_error : std::invalid_argument {
  non_finite_error() : std::invalid_argument("non-finite input element") {}
};
struct invalid_k_error : std::invalid_argument {
  invalid_k_error() : std::invalid_argument("k must satisfy 1 <= k <= input size") {}
};
struct invalid_chunk_error : std::invalid_argument {
  invalid_chunk_error() : std::invalid_argument("chunk length must be >= 1") {}
};
// Device-side failures the reference cannot have.
struct device_error : std::runtime_error {
  explicit device_error(const std::string& m) : std::runtime_error(m) {}
};

// topk.hpp:14-17
struct topk_result {
  std::vector<float> values;
  std::vector<std::int64_t> indices;
};

namespace b200 {

inline int& device_ref() {
  static int d = 0;
  return d;
}
inline void set_device(int d) { device_ref() = d; }

inline void throw_status(osmx_status s) {
  switch (s) {
    case OSMX_OK: return;
    case OSMX_ERR_EMPTY: throw empty_input_error();
    case OSMX_ERR_NON_FINITE: throw non_finite_error();
    case OSMX_ERR_INVALID_K: throw invalid_k_error();
    case OSMX_ERR_INVALID_CHUNK: throw invalid_chunk_error();
    case OSMX_ERR_CUDA: throw device_error(std::string("CUDA: ") + osmx_last_cuda_error());
    default: throw device_error(osmx_status_string(s));
  }
}

inline std::vector<float> softmax_rows(int alg, std::span<const float> x, std::size_t rows) {
  if (rows == 0) return {};
  const std::size_t V = x.size() / rows;
  if (V == 0) throw empty_input_error();
  std::vector<float> y(x.size());
  throw_status(osmx_softmax_host(alg, x.data(), (int64_t)rows, (int64_t)V, y.data(), device_ref(), nullptr));
  return y;
}

inline topk_result topk_rows(int alg, std::span<const float> x, std::size_t rows, std::size_t k) {
  topk_result r;
  if (rows == 0) return r;
  const std::size_t V = x.size() / rows;
  if (V == 0) throw empty_input_error();
  if (k == 0 || k > V) throw invalid_k_error();
  r.values.resize(rows * k);
  r.indices.resize(rows * k);
  osmx_status s = alg < 0 ? osmx_topk_host(x.data(), (int64_t)rows, (int64_t)V, (int32_t)k, r.values.data(),
                                           r.indices.data(), device_ref(), nullptr)
                          : osmx_softmax_topk_host(alg, x.data(), (int64_t)rows, (int64_t)V, (int32_t)k,
                                                   r.values.data(), r.indices.data(), device_ref(), nullptr);
  throw_status(s);
  return r;
}

}  // namespace b200

// softmax.hpp:17-28 -- single vector in, fresh vector out.
inline std::vector<float> naive_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_NAIVE_SOFTMAX, x, 1);
}
inline std::vector<float> safe_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_SAFE_SOFTMAX, x, 1);
}
inline std::vector<float> online_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_ONLINE_SOFTMAX, x, 1);
}

// topk.hpp:54-68
inline topk_result topk_of(std::span<const float> values, std::size_t k) {
  return b200::topk_rows(-1, values, 1, k);
}
inline topk_result safe_softmax_then_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_UNFUSED_TOPK, x, 1, k);
}
inline topk_result safe_softmax_fused_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_FUSED_TOPK, x, 1, k);
}
inline topk_result online_softmax_topk(std::span<const float> x, std::size_t k) {
  return b200::topk_rows(OSMX_ONLINE_SOFTMAX_FUSED_TOPK, x, 1, k);
}

// Batched forms: x is rows x V row-major; results row-major.
namespace batched {
inline std::vector<float> naive_softmax(std::span<const float> x, std::size_t rows) {
  return b200::softmax_rows(OSMX_NAIVE_SOFTMAX, x, rows);
}
inline std::vector<float> safe_softmax(std::span<const float> x, std::size_t rows) {
  return b200::softmax_rows(OSMX_SAFE_SOFTMAX, x, rows);
}
inline std::vector<float> online_softmax(std::span<const float> x, std::size_t rows) {
  return b200::softmax_rows(OSMX_ONLINE_SOFTMAX, x, rows);
}
inline topk_result online_softmax_topk(std::span<const float> x, std::size_t rows, std::size_t k) {
  return b200::topk_rows(OSMX_ONLINE_SOFTMAX_FUSED_TOPK, x, rows, k);
}
inline topk_result safe_softmax_fused_topk(std::span<const float> x, std::size_t rows, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_FUSED_TOPK, x, rows, k);
}
inline topk_result safe_softmax_then_topk(std::span<const float> x, std::size_t rows, std::size_t k) {
  return b200::topk_rows(OSMX_SAFE_SOFTMAX_UNFUSED_TOPK, x, rows, k);
}
inline topk_result topk_of(std::span<const float> x, std::size_t rows, std::size_t k) {
  return b200::topk_rows(-1, x, rows, k);
}
}  // namespace batched

}  // namespace osmx
