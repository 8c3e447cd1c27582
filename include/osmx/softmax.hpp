// include/osmx/softmax.hpp -- the reference's softmax API (proj/include/osmx/
// softmax.hpp:17-28) on the B200: span in, fresh vector out, the reference's
// exceptions.  Every call runs the sm_100a kernels through the host-buffer
// C-ABI (osmx_softmax_host_multi); there is no CPU path.
//
// Batched forms (osmx::batched) take a row-major rows x V batch -- the shape
// the reference's bench drives one row at a time (bench.cpp:34-96) -- and an
// optional device list (rows sharded over the GPUs, one host thread each).
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "b200_runtime.hpp"

namespace osmx {
namespace b200 {

inline std::vector<float> softmax_rows(int alg, std::span<const float> x, std::size_t rows,
                                       const std::vector<int>& devs) {
  if (rows == 0) return {};
  const std::size_t V = x.size() / rows;
  if (V == 0) throw empty_input_error();
  std::vector<float> y(x.size());
  throw_status(osmx_softmax_host_multi(alg, x.data(), (int64_t)rows, (int64_t)V, y.data(), devs.data(),
                                       (int32_t)devs.size(), nullptr));
  return y;
}

}  // namespace b200

// softmax.hpp:17 (Alg. 1), :22 (Alg. 2), :28 (Alg. 3).
inline std::vector<float> naive_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_NAIVE_SOFTMAX, x, 1, b200::devices());
}
inline std::vector<float> safe_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_SAFE_SOFTMAX, x, 1, b200::devices());
}
inline std::vector<float> online_softmax(std::span<const float> x) {
  return b200::softmax_rows(OSMX_ONLINE_SOFTMAX, x, 1, b200::devices());
}

namespace batched {
inline std::vector<float> naive_softmax(std::span<const float> x, std::size_t rows,
                                        const std::vector<int>& devs = b200::devices()) {
  return b200::softmax_rows(OSMX_NAIVE_SOFTMAX, x, rows, devs);
}
inline std::vector<float> safe_softmax(std::span<const float> x, std::size_t rows,
                                       const std::vector<int>& devs = b200::devices()) {
  return b200::softmax_rows(OSMX_SAFE_SOFTMAX, x, rows, devs);
}
inline std::vector<float> online_softmax(std::span<const float> x, std::size_t rows,
                                         const std::vector<int>& devs = b200::devices()) {
  return b200::softmax_rows(OSMX_ONLINE_SOFTMAX, x, rows, devs);
}
}  // namespace batched

}  // namespace osmx
