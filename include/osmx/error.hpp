// include/osmx/error.hpp -- the reference's exception types (proj/include/
// osmx/error.hpp:8-25): same names, same base (std::invalid_argument), same
// what() strings, so `catch (const osmx::non_finite_error&)` in a reference
// caller keeps working against the B200 build.  The C-ABI status codes 1..4
// map onto them (include/osmx_b200.h).
#pragma once

#include <stdexcept>
#include <string>

namespace osmx {

#define OSMX_B200_ARGUMENT_ERROR(type, text)              \
  struct type : std::invalid_argument {                   \
    type() : std::invalid_argument(text) {}               \
  };

OSMX_B200_ARGUMENT_ERROR(empty_input_error, "empty input vector")                   // V == 0
OSMX_B200_ARGUMENT_ERROR(non_finite_error, "non-finite input element")              // NaN / +-inf
OSMX_B200_ARGUMENT_ERROR(invalid_k_error, "k must satisfy 1 <= k <= input size")    // k outside [1, V]
OSMX_B200_ARGUMENT_ERROR(invalid_chunk_error, "chunk length must be >= 1")          // chunk_len == 0

#undef OSMX_B200_ARGUMENT_ERROR

// Device-side failures the CPU reference cannot have (CUDA errors, k above
// the record capacity of the split path).
struct device_error : std::runtime_error {
  explicit device_error(const std::string& m) : std::runtime_error(m) {}
};

}  // namespace osmx
