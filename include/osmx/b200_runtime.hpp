// include/osmx/b200_runtime.hpp -- shared plumbing of the C++ facade
// (osmx/{softmax,topk,normalizer}.hpp over include/osmx_b200.h): the device
// list the host-buffer calls shard a batch over, and the status -> exception
// mapping (error.hpp:8-25).
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../osmx_b200.h"
#include "error.hpp"

namespace osmx {
namespace b200 {

// Devices a host-buffer call shards its rows over (contiguous blocks, one
// host thread per entry inside the library, osmx_*_host_multi).  Default
// {0}.  A device may appear more than once.
struct device_list {
  std::mutex mu;
  std::vector<int> ids{0};
};
inline device_list& devices_ref() {
  static device_list d;
  return d;
}
inline void set_devices(const std::vector<int>& ids) {
  if (ids.empty()) throw std::invalid_argument("osmx::b200::set_devices: empty device list");
  auto& d = devices_ref();
  std::lock_guard<std::mutex> lock(d.mu);
  d.ids = ids;
}
inline void set_device(int id) { set_devices({id}); }
inline std::vector<int> devices() {
  auto& d = devices_ref();
  std::lock_guard<std::mutex> lock(d.mu);
  return d.ids;
}

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

}  // namespace b200
}  // namespace osmx
