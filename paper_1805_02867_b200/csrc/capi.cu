// capi.cu -- the extern "C" boundary (include/osmx_b200.h): argument
// validation with the reference's error precedence, workspace sizing,
// dispatch to the launch layer, the non-finite status channel, and the
// pipelined host-buffer path.
//
// Validation order follows the reference: require_nonempty before
// require_valid_k (kernels.hpp:24-30, topk.cpp:38-39); non-finite input is
// detected during the first pass (kernels.hpp:14-15, :32-35) and reported
// through the workspace flag instead of an exception.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <set>
#include <utility>
#include <string>
#include <vector>

#include "../../include/osmx_b200.h"
#include "common.cuh"
#include "internal.hpp"

namespace osmx_host {

namespace {
std::mutex g_tune_mu;
Tuning g_tune;                   // process-wide defaults (osmx_config_set)
thread_local Tuning t_tune;      // snapshot in force for this thread's call
thread_local int t_scope = 0;    // open TuningScopes on this thread
}  // namespace

Tuning tuning_defaults() {
  std::lock_guard<std::mutex> lock(g_tune_mu);
  return g_tune;
}
void tuning_set_defaults(const Tuning& t) {
  std::lock_guard<std::mutex> lock(g_tune_mu);
  g_tune = t;
}
Tuning& tuning() {
  if (t_scope == 0) t_tune = tuning_defaults();  // outside a call: fresh snapshot
  return t_tune;
}
TuningScope::TuningScope(const Tuning* t) : outer_(t_scope == 0) {
  if (outer_)
    t_tune = t ? *t : tuning_defaults();
  else {
    saved_ = t_tune;
    if (t) t_tune = *t;
  }
  ++t_scope;
}
TuningScope::~TuningScope() {
  --t_scope;
  if (!outer_) t_tune = saved_;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

cudaError_t side_stream(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  struct Side {
    cudaStream_t s = nullptr;
    cudaEvent_t f = nullptr, j = nullptr;
  };
  thread_local Side sides[64];  // per host thread and device: no sharing between concurrent callers
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  Side& sd = sides[dev];
  if (!sd.s) {
    cudaError_t e = cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sd.f, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sd.j, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  *side = sd.s;
  *fork = sd.f;
  *join = sd.j;
  return cudaSuccess;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

bool first_use_on_device(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  return seen.insert({dev, fn}).second;
}

static std::atomic<long long> g_host_chunk_mb{512};

static size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// Split-region bytes (after the header) and, for the unfused pipelines, the
// materialised probability matrix (placed after the split region).
static size_t split_region(int alg, long long rows, long long V, int k) {
  size_t b = 0;
  switch (alg) {
    case kNaive:
    case kSafe:
    case kOnline:
      if (softmax_uses_split(rows, V)) b = softmax_split_ws(rows, V);
      break;
    case kSafeFusedTopk:
    case kOnlineFusedTopk:
      if (k > kMaxK) b = topk_large_ws(rows, V, k);
      else if (topk_split(rows, V)) b = topk_split_ws(alg, rows, V, k);
      break;
    case kSliceRecord:  // always the split path (piece records + combine)
      b = topk_split_ws(kOnlineFusedTopk, rows, V, k);
      break;
    case kProjTopk:
      b = proj_topk_ws(rows, V, k);
      break;
    case kSafeUnfusedTopk:
    case kOnlineUnfusedTopk:
    case kTopkOf: {
      if (softmax_uses_split(rows, V)) b = std::max(b, softmax_split_ws(rows, V));
      if (k > kMaxK) b = std::max(b, topk_large_ws(rows, V, k));
      else if (topk_split(rows, V)) b = std::max(b, topk_split_ws(kTopkOf, rows, V, k));
      break;
    }
    default:
      break;
  }
  return align256(b);
}

size_t workspace_bytes(int alg, long long rows, long long V, int k) {
  if (rows < 1 || V < 1) return osmx_dev::kWsHeader;
  size_t b = osmx_dev::kWsHeader + split_region(alg, rows, V, k);
  if (alg == kSafeUnfusedTopk || alg == kOnlineUnfusedTopk) b += align256((size_t)rows * (size_t)V * sizeof(float));
  return b;
}

}  // namespace osmx_host

using namespace osmx_host;

namespace {

thread_local std::string t_cuda_err;

osmx_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return OSMX_OK;
  t_cuda_err = cudaGetErrorString(e);
  return OSMX_ERR_CUDA;
}

bool is_softmax(int alg) { return alg == kNaive || alg == kSafe || alg == kOnline; }
bool is_topk(int alg) {
  return alg == kSafeUnfusedTopk || alg == kSafeFusedTopk || alg == kOnlineFusedTopk || alg == kOnlineUnfusedTopk;
}

osmx_status check_common(const void* x, long long ld, long long rows, long long V) {
  if (V < 1) return OSMX_ERR_EMPTY;  // require_nonempty, kernels.hpp:24-26
  if (rows < 0 || ld < V) return OSMX_ERR_INVALID_ARG;
  if (rows > 0 && !x) return OSMX_ERR_INVALID_ARG;
  return OSMX_OK;
}

osmx_status check_k(long long V, int k, long long rows = 1) {
  if (k < 1 || (long long)k > V) return OSMX_ERR_INVALID_K;  // require_valid_k, kernels.hpp:28-30
  if (k > kMaxK && !topk_large_supported(rows, V, k)) return OSMX_ERR_UNSUPPORTED;
  return OSMX_OK;
}

osmx_status run_topk_alg(int alg, const float* x, long long ldx, long long rows, long long V, int k,
                         float* vals, long long* idx, void* ws, size_t ws_bytes, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  switch (alg) {
    case kOnlineFusedTopk: e = launch_topk_mode(0, x, ldx, rows, V, k, vals, idx, ws, st); break;
    case kSafeFusedTopk: e = launch_topk_mode(2, x, ldx, rows, V, k, vals, idx, ws, st); break;
    case kTopkOf: e = launch_topk_mode(1, x, ldx, rows, V, k, vals, idx, ws, st); break;
    case kSafeUnfusedTopk:
    case kOnlineUnfusedTopk: {
      // softmax -> materialised y (workspace tail) -> topk_of(y), the
      // reference's safe_softmax_then_topk (topk.cpp:30-35).
      char* y = static_cast<char*>(ws) + osmx_dev::kWsHeader + split_region(alg, rows, V, k);
      (void)ws_bytes;
      e = launch_softmax(alg == kSafeUnfusedTopk ? kSafe : kOnline, x, ldx, reinterpret_cast<float*>(y), V, rows,
                         V, ws, ws_bytes, st);
      if (e == cudaSuccess) e = launch_topk_mode(1, reinterpret_cast<float*>(y), V, rows, V, k, vals, idx, ws, st);
      break;
    }
    default:
      return OSMX_ERR_INVALID_ARG;
  }
  return cuda_status(e);
}

}  // namespace

extern "C" {

int osmx_version(void) { return OSMX_VERSION; }

const char* osmx_status_string(osmx_status s) {
  switch (s) {
    case OSMX_OK: return "ok";
    case OSMX_ERR_EMPTY: return "empty input vector";
    case OSMX_ERR_NON_FINITE: return "non-finite input element";
    case OSMX_ERR_INVALID_K: return "k must satisfy 1 <= k <= input size";
    case OSMX_ERR_INVALID_CHUNK: return "chunk length must be >= 1";
    case OSMX_ERR_INVALID_ARG: return "invalid argument";
    case OSMX_ERR_CUDA: return "CUDA error";
    case OSMX_ERR_UNSUPPORTED: return "unsupported (records: k above OSMX_MAX_K; large k: rows * k >= 2^31)";
    case OSMX_ERR_NCCL: return "NCCL error";
  }
  return "unknown status";
}

const char* osmx_last_cuda_error(void) { return t_cuda_err.c_str(); }

size_t osmx_workspace_bytes(int alg, int64_t rows, int64_t V, int32_t k) {
  TuningScope scope;
  return workspace_bytes(alg, rows, V, k);
}

osmx_status osmx_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws || ws_bytes < (size_t)osmx_dev::kWsHeader) return OSMX_ERR_INVALID_ARG;
  return cuda_status(cudaMemsetAsync(ws, 0, osmx_dev::kWsHeader, static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_check_status(void* ws, void* stream, int64_t* first_bad_row) {
  if (!ws) return OSMX_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long bad = 0;
  cudaError_t e = cudaMemcpyAsync(&bad, ws, sizeof(bad), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && bad) e = cudaMemsetAsync(ws, 0, sizeof(bad), st);
  if (e == cudaSuccess && bad) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  const long long row = bad ? (long long)(0x7fffffffffffffffULL - bad) : -1;
  if (first_bad_row) *first_bad_row = row;
  return bad ? OSMX_ERR_NON_FINITE : OSMX_OK;
}

osmx_status osmx_softmax(int alg, const float* x, int64_t ldx, float* y, int64_t ldy, int64_t rows, int64_t V,
                         void* ws, size_t ws_bytes, void* stream) {
  if (!is_softmax(alg)) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  osmx_status s = check_common(x, ldx, rows, V);
  if (s) return s;
  if (ldy < V || (rows > 0 && !y) || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  if (ws_bytes < workspace_bytes(alg, rows, V, 0)) return OSMX_ERR_INVALID_ARG;
  return cuda_status(launch_softmax(alg, x, ldx, y, ldy, rows, V, ws, ws_bytes, static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_softmax_topk(int alg, const float* x, int64_t ldx, int64_t rows, int64_t V, int32_t k,
                              float* vals, int64_t* idx, void* ws, size_t ws_bytes, void* stream) {
  if (!is_topk(alg)) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  osmx_status s = check_common(x, ldx, rows, V);
  if (s) return s;
  if ((s = check_k(V, k, rows))) return s;
  if ((rows > 0 && (!vals || !idx)) || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  if (ws_bytes < workspace_bytes(alg, rows, V, k)) return OSMX_ERR_INVALID_ARG;
  return run_topk_alg(alg, x, ldx, rows, V, k, vals, reinterpret_cast<long long*>(idx), ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

osmx_status osmx_topk(const float* v, int64_t ld, int64_t rows, int64_t V, int32_t k, float* vals, int64_t* idx,
                      void* ws, size_t ws_bytes, void* stream) {
  TuningScope scope;
  osmx_status s = check_common(v, ld, rows, V);
  if (s) return s;
  if ((s = check_k(V, k, rows))) return s;
  if ((rows > 0 && (!vals || !idx)) || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  if (ws_bytes < workspace_bytes(kTopkOf, rows, V, k)) return OSMX_ERR_INVALID_ARG;
  return run_topk_alg(kTopkOf, v, ld, rows, V, k, vals, reinterpret_cast<long long*>(idx), ws, ws_bytes,
                      static_cast<cudaStream_t>(stream));
}

osmx_status osmx_proj_softmax_topk(const void* h, int64_t rows, int64_t D, const void* w, int64_t V, int32_t k,
                                   float* vals, int64_t* idx, void* ws, size_t ws_bytes, void* stream) {
  TuningScope scope;
  if (V < 1 || D < 1) return OSMX_ERR_EMPTY;
  if (k < 1 || (long long)k > V) return OSMX_ERR_INVALID_K;
  if (k > kMaxK) return OSMX_ERR_UNSUPPORTED;
  if (rows < 0 || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  // TMA: 16-byte aligned bases and row strides (D % 8 bf16), 32-bit coordinates
  if (!h || !w || !vals || !idx || (D % 8) || ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(w)) & 15) ||
      rows > (1LL << 31) - 1 || V > (1LL << 31) - 1 || D > (1LL << 31) - 1)
    return OSMX_ERR_INVALID_ARG;
  if (ws_bytes < workspace_bytes(kProjTopk, rows, V, k)) return OSMX_ERR_INVALID_ARG;
  return cuda_status(launch_proj_topk(h, rows, D, w, V, k, vals, reinterpret_cast<long long*>(idx), ws,
                                      static_cast<cudaStream_t>(stream)));
}

size_t osmx_normalizer_workspace_bytes(int64_t rows, int64_t V, int64_t chunk, int32_t precision) {
  return normalizer_ws(rows, V, chunk < 0 ? 0 : chunk, precision == 64 ? 64 : 32);
}

osmx_status osmx_normalizer(const float* x, int64_t ldx, int64_t rows, int64_t V, int64_t chunk, float* m,
                            float* d, void* ws, size_t ws_bytes, void* stream) {
  TuningScope scope;
  osmx_status s = check_common(x, ldx, rows, V);
  if (s) return s;
  if (chunk < 0) return OSMX_ERR_INVALID_CHUNK;
  if ((rows > 0 && (!m || !d)) || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  if (ws_bytes < normalizer_ws(rows, V, chunk, 32)) return OSMX_ERR_INVALID_ARG;
  return cuda_status(launch_normalizer(x, ldx, rows, V, chunk, m, d, ws, static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_normalizer_f64(const float* x, int64_t ldx, int64_t rows, int64_t V, int64_t chunk, double* m,
                                double* d, void* ws, size_t ws_bytes, void* stream) {
  TuningScope scope;
  osmx_status s = check_common(x, ldx, rows, V);
  if (s) return s;
  if (chunk < 0) return OSMX_ERR_INVALID_CHUNK;
  if ((rows > 0 && (!m || !d)) || !ws) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  if (ws_bytes < normalizer_ws(rows, V, chunk, 64)) return OSMX_ERR_INVALID_ARG;
  return cuda_status(launch_normalizer_f64(x, ldx, rows, V, chunk, m, d, ws, static_cast<cudaStream_t>(stream)));
}

size_t osmx_record_bytes(int32_t k) { return record_bytes(k > 0 ? k : 1); }

osmx_status osmx_slice_record(const float* x, int64_t V, int64_t col0, int32_t k, void* record, void* ws,
                              size_t ws_bytes, void* stream) {
  if (V < 1) return OSMX_ERR_EMPTY;
  if (!x || !record || !ws || col0 < 0) return OSMX_ERR_INVALID_ARG;
  if (k < 0 || k > kMaxK) return k < 0 ? OSMX_ERR_INVALID_K : OSMX_ERR_UNSUPPORTED;
  const int kk = k > 0 ? k : 1;
  // the slice may hold fewer than k elements; the merged row must not
  TuningScope scope;  // the forced split shape below lives only in this call's snapshot
  const size_t need = workspace_bytes(9, 1, V, kk);
  if (ws_bytes < need) return OSMX_ERR_INVALID_ARG;
  tuning().shape = kShapeSplit;
  return cuda_status(launch_slice_record(x, V, col0, k, record, ws, ws_bytes, static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_records_combine(const void* records, int32_t n, int32_t k, void* out_record, float* vals,
                                 int64_t* idx, void* ws, size_t ws_bytes, void* stream) {
  if (!records || n < 1 || !ws || ws_bytes < (size_t)osmx_dev::kWsHeader) return OSMX_ERR_INVALID_ARG;
  if (k < 0 || k > kMaxK) return k < 0 ? OSMX_ERR_INVALID_K : OSMX_ERR_UNSUPPORTED;
  if (k > 0 && (!vals) != (!idx)) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  return cuda_status(launch_records_combine(records, n, k, out_record, vals, reinterpret_cast<long long*>(idx), ws,
                                            static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_scale_with_record(const float* x, int64_t V, const void* record, float* y, void* stream) {
  if (V < 1) return OSMX_ERR_EMPTY;
  if (!x || !record || !y) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  return cuda_status(launch_scale_with_record(x, V, record, y, static_cast<cudaStream_t>(stream)));
}

uint64_t osmx_launch_count(void) { return g_launches.load(); }

osmx_status osmx_diag_read_probe(const void* x, size_t bytes, float* sink, void* stream) {
  if (!x || !sink || (reinterpret_cast<uintptr_t>(x) & 15)) return OSMX_ERR_INVALID_ARG;
  return cuda_status(launch_read_probe(x, bytes, sink, static_cast<cudaStream_t>(stream)));
}

osmx_status osmx_config_set(const char* key, int64_t value) {
  if (!key) return OSMX_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lock(g_tune_mu);  // process-wide defaults
  auto& t = g_tune;
  if (!strcmp(key, "shape")) {
    if (value < 0 || value > 5) return OSMX_ERR_INVALID_ARG;
    t.shape = (int)value;
  } else if (!strcmp(key, "resident_max_v")) {
    if (value < 0 || value > 16384) return OSMX_ERR_INVALID_ARG;
    t.resident_max_v = (int)value;
  } else if (!strcmp(key, "split_chunk")) {
    if (value < 0) return OSMX_ERR_INVALID_ARG;
    t.split_chunk = value;
  } else if (!strcmp(key, "stream_threads")) {
    if (value != 0 && value != 256 && value != 512 && value != 1024) return OSMX_ERR_INVALID_ARG;
    t.stream_threads = (int)value;
  } else if (!strcmp(key, "stream_ctas")) {
    if (value < 0 || value > 32) return OSMX_ERR_INVALID_ARG;
    t.stream_ctas = (int)value;
  } else if (!strcmp(key, "split_fuse")) {
    if (value < 0 || value > 1) return OSMX_ERR_INVALID_ARG;
    t.split_fuse = (int)value;
  } else if (!strcmp(key, "topk_block")) {
    if (value != 0 && value != 32 && value != 128) return OSMX_ERR_INVALID_ARG;
    t.topk_block = (int)value;
  } else if (!strcmp(key, "topk_threads")) {
    if (value != 0 && value != 32 && value != 128 && value != 256 && value != 512) return OSMX_ERR_INVALID_ARG;
    t.topk_threads = (int)value;
  } else if (!strcmp(key, "cluster_size")) {
    if (value < 0 || value > 16) return OSMX_ERR_INVALID_ARG;
    t.cluster_size = (int)value;
  } else if (!strcmp(key, "staged_gw")) {
    if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8 && value != 16) return OSMX_ERR_INVALID_ARG;
    t.staged_gw = (int)value;
  } else if (!strcmp(key, "staged_ng")) {
    if (value < 0 || value > 31) return OSMX_ERR_INVALID_ARG;
    t.staged_ng = (int)value;
  } else if (!strcmp(key, "staged_kb")) {
    if (value != 0 && (value < 16 || value > 227)) return OSMX_ERR_INVALID_ARG;
    t.staged_kb = (int)value;
  } else if (!strcmp(key, "split_cta")) {
    if (value < -1 || value > 4) return OSMX_ERR_INVALID_ARG;
    t.split_cta = (int)value;
  } else if (!strcmp(key, "proj_bn")) {
    if (value != 0 && value != 128 && value != 224 && value != 256) return OSMX_ERR_INVALID_ARG;
    t.proj_bn = (int)value;
  } else if (!strcmp(key, "topk_pipe")) {
    if (value < 0 || value > 6) return OSMX_ERR_INVALID_ARG;
    t.topk_pipe = (int)value;
  } else if (!strcmp(key, "topk_u8")) {
    if (value < -1 || value > 1) return OSMX_ERR_INVALID_ARG;
    t.topk_u8 = (int)value;
  } else if (!strcmp(key, "l2_prefetch")) {
    if (value < -1 || value > 64) return OSMX_ERR_INVALID_ARG;
    t.l2_prefetch = (int)value;
  } else if (!strcmp(key, "tma")) {
    if (value < 0 || value > 2) return OSMX_ERR_INVALID_ARG;
    t.tma = (int)value;
  } else if (!strcmp(key, "corun")) {
    if (value < -1 || value > 99) return OSMX_ERR_INVALID_ARG;
    t.corun = (int)value;
  } else if (!strcmp(key, "large_fast")) {
    if (value < 0 || value > 1) return OSMX_ERR_INVALID_ARG;
    t.large_fast = (int)value;
  } else if (!strcmp(key, "tma_cfg")) {
    if (value < -1 || value > 2) return OSMX_ERR_INVALID_ARG;
    t.tma_cfg = (int)value;
  } else if (!strcmp(key, "host_chunk_mb")) {
    if (value < 1) return OSMX_ERR_INVALID_ARG;
    g_host_chunk_mb = value;
  } else {
    return OSMX_ERR_INVALID_ARG;
  }
  return OSMX_OK;
}

int64_t osmx_config_get(const char* key) {
  if (!key) return -1;
  const Tuning t = tuning_defaults();
  if (!strcmp(key, "shape")) return t.shape;
  if (!strcmp(key, "resident_max_v")) return t.resident_max_v;
  if (!strcmp(key, "split_chunk")) return t.split_chunk;
  if (!strcmp(key, "stream_threads")) return t.stream_threads;
  if (!strcmp(key, "topk_threads")) return t.topk_threads;
  if (!strcmp(key, "topk_block")) return t.topk_block;
  if (!strcmp(key, "split_fuse")) return t.split_fuse;
  if (!strcmp(key, "tma")) return t.tma;
  if (!strcmp(key, "tma_cfg")) return t.tma_cfg;
  if (!strcmp(key, "large_fast")) return t.large_fast;
  if (!strcmp(key, "corun")) return t.corun;
  if (!strcmp(key, "l2_prefetch")) return t.l2_prefetch;
  if (!strcmp(key, "topk_u8")) return t.topk_u8;
  if (!strcmp(key, "topk_pipe")) return t.topk_pipe;
  if (!strcmp(key, "proj_bn")) return t.proj_bn;
  if (!strcmp(key, "split_cta")) return t.split_cta;
  if (!strcmp(key, "stream_ctas")) return t.stream_ctas;
  if (!strcmp(key, "staged_gw")) return t.staged_gw;
  if (!strcmp(key, "cluster_size")) return t.cluster_size;
  if (!strcmp(key, "staged_ng")) return t.staged_ng;
  if (!strcmp(key, "staged_kb")) return t.staged_kb;
  if (!strcmp(key, "host_chunk_mb")) return g_host_chunk_mb;
  return -1;
}

}  // extern "C"

// ------------------------------------------------------ host-buffer path --
namespace {

// Staging of one host thread on one device: two slots, each with its own
// stream, input block, output block and workspace, so block i+1's H2D
// overlaps block i's kernel and block i-1's D2H.  Keyed by (device, slot):
// a multi-device call that lists a device twice drives it from two threads
// with two contexts.
struct HostCtx {
  std::mutex mu;
  cudaStream_t st[2] = {nullptr, nullptr};
  void* xin[2] = {nullptr, nullptr};
  void* out[2] = {nullptr, nullptr};
  void* ws[2] = {nullptr, nullptr};
  size_t xin_b = 0, out_b = 0, ws_b = 0;

  cudaError_t ensure(size_t xb, size_t ob, size_t wb) {
    cudaError_t e = cudaSuccess;
    if (!st[0]) {
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    }
    auto grow = [&](void* (&p)[2], size_t& have, size_t want) {
      if (e != cudaSuccess || want <= have) return;
      for (int i = 0; i < 2; ++i) {
        if (p[i]) cudaFree(p[i]);
        p[i] = nullptr;
      }
      have = 0;
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&p[i], want);
      if (e == cudaSuccess) have = want;
    };
    grow(xin, xin_b, xb);
    grow(out, out_b, ob);
    const size_t wsb0 = ws_b;
    grow(ws, ws_b, wb);
    if (e == cudaSuccess && ws_b != wsb0)
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMemset(ws[i], 0, osmx_dev::kWsHeader);
    return e;
  }
  void release() {
    for (int i = 0; i < 2; ++i) {
      if (xin[i]) cudaFree(xin[i]);
      if (out[i]) cudaFree(out[i]);
      if (ws[i]) cudaFree(ws[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
      xin[i] = out[i] = ws[i] = nullptr;
      st[i] = nullptr;
    }
    xin_b = out_b = ws_b = 0;
  }
};

std::mutex g_ctx_mu;
std::map<std::pair<int, int>, std::unique_ptr<HostCtx>> g_ctx;

HostCtx& host_ctx(int device, int slot) {
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  auto& p = g_ctx[{device, slot}];
  if (!p) p.reset(new HostCtx);
  return *p;
}

// What one row block runs: a softmax (out1 = y), a top-K (out1 = vals,
// out2 = idx; alg kTopkOf for osmx_topk_host) or a normalizer (out1 = m,
// out2 = d, float or double by `prec`).
struct HostOp {
  enum Kind { kSoftmax, kTopk, kNorm } kind;
  int alg;
  int k;
  long long chunk = 0;
  int prec = 32;
  size_t out1_row(long long V) const {
    switch (kind) {
      case kSoftmax: return (size_t)V * sizeof(float);
      case kTopk: return (size_t)k * sizeof(float);
      default: return prec == 64 ? sizeof(double) : sizeof(float);
    }
  }
  size_t out2_row() const {
    switch (kind) {
      case kSoftmax: return 0;
      case kTopk: return (size_t)k * sizeof(long long);
      default: return prec == 64 ? sizeof(double) : sizeof(float);
    }
  }
  size_t ws_bytes(long long rows, long long V) const {
    return kind == kNorm ? normalizer_ws(rows, V, chunk, prec) : workspace_bytes(alg, rows, V, k);
  }
  osmx_status launch(const float* dx, long long nr, long long V, char* o1, char* o2, void* ws, size_t wsb,
                     cudaStream_t st) const {
    switch (kind) {
      case kSoftmax:
        return cuda_status(launch_softmax(alg, dx, V, reinterpret_cast<float*>(o1), V, nr, V, ws, wsb, st));
      case kTopk:
        return run_topk_alg(alg, dx, V, nr, V, k, reinterpret_cast<float*>(o1), reinterpret_cast<long long*>(o2),
                            ws, wsb, st);
      default:
        if (prec == 64)
          return cuda_status(launch_normalizer_f64(dx, V, nr, V, chunk, reinterpret_cast<double*>(o1),
                                                   reinterpret_cast<double*>(o2), ws, st));
        return cuda_status(launch_normalizer(dx, V, nr, V, chunk, reinterpret_cast<float*>(o1),
                                             reinterpret_cast<float*>(o2), ws, st));
    }
  }
};

// The second output block (int64 indices) starts 256-byte aligned after the
// first (rpb*k floats): int64 stores need 8-byte alignment.
size_t out2_offset(long long rpb, size_t out_row_bytes) { return ((size_t)rpb * out_row_bytes + 255) / 256 * 256; }

// Rows [0, rows) of x on one device through ctx (device, slot), in blocks of
// rpb rows.  *first_bad = lowest non-finite row (local) or -1.
osmx_status host_run(const HostOp& op, int device, int slot, const float* x, long long rows, long long V,
                     char* out1, char* out2, long long chunk_mb, long long* first_bad) {
  HostCtx& c = host_ctx(device, slot);
  std::lock_guard<std::mutex> lock(c.mu);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_status(e);
  const size_t row_b = (size_t)V * sizeof(float);
  const size_t o1 = op.out1_row(V), o2 = op.out2_row();
  long long rpb = (long long)std::max<size_t>(1, ((size_t)chunk_mb << 20) / row_b);
  rpb = std::min(rpb, rows);
  // The launch layer picks a kernel shape per block, so the short tail block
  // may take a path (split records) the full blocks do not: size the
  // workspace for both.
  const long long tail = rows % rpb;
  size_t wsb = op.ws_bytes(rpb, V);
  if (tail) wsb = std::max(wsb, op.ws_bytes(tail, V));
  e = c.ensure(rpb * row_b, std::max<size_t>(out2_offset(rpb, o1) + (size_t)rpb * o2 + 256, 256), wsb);
  if (e != cudaSuccess) return cuda_status(e);
  osmx_status st = OSMX_OK;
  const long long nblk = (rows + rpb - 1) / rpb;
  std::vector<long long> bases((size_t)nblk, 0);
  for (long long b = 0; b < nblk && st == OSMX_OK; ++b) {
    const int s = (int)(b & 1);
    const long long r0 = b * rpb;
    const long long nr = std::min(rpb, rows - r0);
    bases[b] = r0;
    e = cudaMemcpyAsync(static_cast<char*>(c.ws[s]) + offsetof(osmx_dev::WsHeader, row_base), &bases[b],
                        sizeof(long long), cudaMemcpyHostToDevice, c.st[s]);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c.xin[s], x + r0 * V, (size_t)nr * row_b, cudaMemcpyHostToDevice, c.st[s]);
    if (e != cudaSuccess) {
      st = cuda_status(e);
      break;
    }
    const float* dx = static_cast<const float*>(c.xin[s]);
    char* dout = static_cast<char*>(c.out[s]);
    st = op.launch(dx, nr, V, dout, dout + out2_offset(rpb, o1), c.ws[s], c.ws_b, c.st[s]);
    if (st != OSMX_OK) break;
    e = cudaMemcpyAsync(out1 + r0 * o1, dout, (size_t)nr * o1, cudaMemcpyDeviceToHost, c.st[s]);
    if (e == cudaSuccess && out2)
      e = cudaMemcpyAsync(out2 + r0 * o2, dout + out2_offset(rpb, o1), (size_t)nr * o2, cudaMemcpyDeviceToHost,
                          c.st[s]);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  // Status: each slot's flag holds the lowest bad (block-local + row_base)
  // row of its blocks.  Both streams are drained even after an error, so
  // `bases` outlives every copy that reads it.
  long long bad_row = -1;
  for (int s = 0; s < 2; ++s) {
    if (!c.st[s]) continue;
    unsigned long long bad = 0;
    e = cudaMemcpyAsync(&bad, c.ws[s], sizeof(bad), cudaMemcpyDeviceToHost, c.st[s]);
    const cudaError_t e2 = cudaStreamSynchronize(c.st[s]);
    if (e == cudaSuccess) e = e2;
    if (e != cudaSuccess) {
      if (st == OSMX_OK) st = cuda_status(e);
      continue;
    }
    if (bad) {
      const long long r = (long long)(0x7fffffffffffffffULL - bad);
      bad_row = bad_row < 0 ? r : std::min(bad_row, r);
      cudaMemsetAsync(c.ws[s], 0, sizeof(bad), c.st[s]);
      cudaStreamSynchronize(c.st[s]);
    }
  }
  *first_bad = bad_row;
  return st;
}

// Row sharder of the host path (the reference's run_batch stripes rows over
// std::threads, bench.cpp:66-96): device list entry i gets the contiguous
// rows [rows*i/n, rows*(i+1)/n) and its own host thread, staging context and
// PCIe link.  Errors: the first failing device (list order) wins; else the
// lowest non-finite row over all devices.
osmx_status host_multi(const HostOp& op, const float* x, long long rows, long long V, void* out1, void* out2,
                       const int* devices, int n, int64_t* first_bad_row) {
  if (first_bad_row) *first_bad_row = -1;
  if (n < 1 || !devices) return OSMX_ERR_INVALID_ARG;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_status(e);
  for (int i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= ndev) return OSMX_ERR_INVALID_ARG;
  if (rows == 0) return OSMX_OK;
  const Tuning snap = tuning();  // the caller's knobs, for every worker
  const long long chunk_mb = g_host_chunk_mb.load();
  const size_t o1 = op.out1_row(V), o2 = op.out2_row();
  std::vector<osmx_status> st((size_t)n, OSMX_OK);
  std::vector<long long> bad((size_t)n, -1);
  std::vector<std::string> err((size_t)n);
  int prev = 0;
  cudaGetDevice(&prev);
  auto work = [&](int i) {
    TuningScope scope(&snap);
    int slot = 0;
    for (int j = 0; j < i; ++j) slot += devices[j] == devices[i];
    const long long r0 = rows * i / n, r1 = rows * (i + 1) / n;
    if (r1 <= r0) return;
    st[i] = host_run(op, devices[i], slot, x + r0 * V, r1 - r0, V, static_cast<char*>(out1) + r0 * o1,
                     out2 ? static_cast<char*>(out2) + r0 * o2 : nullptr, chunk_mb, &bad[i]);
    if (bad[i] >= 0) bad[i] += r0;
    err[i] = t_cuda_err;
  };
  if (n == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    th.reserve((size_t)n - 1);
    for (int i = 1; i < n; ++i) th.emplace_back(work, i);
    work(0);
    for (auto& t : th) t.join();
  }
  cudaSetDevice(prev);
  long long first = -1;
  for (int i = 0; i < n; ++i) {
    if (st[i] != OSMX_OK) {
      t_cuda_err = err[i];
      return st[i];
    }
    if (bad[i] >= 0) first = first < 0 ? bad[i] : std::min(first, bad[i]);
  }
  if (first_bad_row) *first_bad_row = first;
  return first >= 0 ? OSMX_ERR_NON_FINITE : OSMX_OK;
}

osmx_status softmax_host_multi(int alg, const float* x, int64_t rows, int64_t V, float* y, const int* devices,
                               int n, int64_t* first_bad_row) {
  if (first_bad_row) *first_bad_row = -1;
  if (!is_softmax(alg)) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  osmx_status s = check_common(x, V, rows, V);
  if (s) return s;
  if (rows > 0 && !y) return OSMX_ERR_INVALID_ARG;
  return host_multi(HostOp{HostOp::kSoftmax, alg, 0}, x, rows, V, y, nullptr, devices, n, first_bad_row);
}

osmx_status topk_host_multi(int alg, const float* x, int64_t rows, int64_t V, int32_t k, float* vals, int64_t* idx,
                            const int* devices, int n, int64_t* first_bad_row) {
  if (first_bad_row) *first_bad_row = -1;
  if (alg != kTopkOf && !is_topk(alg)) return OSMX_ERR_INVALID_ARG;
  TuningScope scope;
  osmx_status s = check_common(x, V, rows, V);
  if (s) return s;
  if ((s = check_k(V, k))) return s;
  if (rows > 0 && (!vals || !idx)) return OSMX_ERR_INVALID_ARG;
  return host_multi(HostOp{HostOp::kTopk, alg, k}, x, rows, V, vals, idx, devices, n, first_bad_row);
}

osmx_status normalizer_host_multi(const float* x, int64_t rows, int64_t V, int64_t chunk, int precision, void* m,
                                  void* d, const int* devices, int n, int64_t* first_bad_row) {
  if (first_bad_row) *first_bad_row = -1;
  TuningScope scope;
  osmx_status s = check_common(x, V, rows, V);
  if (s) return s;
  if (chunk < 0) return OSMX_ERR_INVALID_CHUNK;
  if ((precision != 32 && precision != 64) || (rows > 0 && (!m || !d))) return OSMX_ERR_INVALID_ARG;
  HostOp op{HostOp::kNorm, kNormalizer, 0};
  op.chunk = chunk;
  op.prec = precision;
  return host_multi(op, x, rows, V, m, d, devices, n, first_bad_row);
}

}  // namespace

extern "C" {

osmx_status osmx_softmax_host(int alg, const float* x, int64_t rows, int64_t V, float* y, int device,
                              int64_t* first_bad_row) {
  return softmax_host_multi(alg, x, rows, V, y, &device, 1, first_bad_row);
}

osmx_status osmx_softmax_topk_host(int alg, const float* x, int64_t rows, int64_t V, int32_t k, float* vals,
                                   int64_t* idx, int device, int64_t* first_bad_row) {
  if (!is_topk(alg)) return OSMX_ERR_INVALID_ARG;
  return topk_host_multi(alg, x, rows, V, k, vals, idx, &device, 1, first_bad_row);
}

osmx_status osmx_topk_host(const float* v, int64_t rows, int64_t V, int32_t k, float* vals, int64_t* idx,
                           int device, int64_t* first_bad_row) {
  return topk_host_multi(kTopkOf, v, rows, V, k, vals, idx, &device, 1, first_bad_row);
}

osmx_status osmx_softmax_host_multi(int alg, const float* x, int64_t rows, int64_t V, float* y,
                                    const int* devices, int32_t n_devices, int64_t* first_bad_row) {
  return softmax_host_multi(alg, x, rows, V, y, devices, n_devices, first_bad_row);
}

osmx_status osmx_softmax_topk_host_multi(int alg, const float* x, int64_t rows, int64_t V, int32_t k, float* vals,
                                         int64_t* idx, const int* devices, int32_t n_devices,
                                         int64_t* first_bad_row) {
  if (!is_topk(alg)) return OSMX_ERR_INVALID_ARG;
  return topk_host_multi(alg, x, rows, V, k, vals, idx, devices, n_devices, first_bad_row);
}

osmx_status osmx_topk_host_multi(const float* v, int64_t rows, int64_t V, int32_t k, float* vals, int64_t* idx,
                                 const int* devices, int32_t n_devices, int64_t* first_bad_row) {
  return topk_host_multi(kTopkOf, v, rows, V, k, vals, idx, devices, n_devices, first_bad_row);
}

osmx_status osmx_normalizer_host(const float* x, int64_t rows, int64_t V, int64_t chunk, int32_t precision,
                                 void* m, void* d, const int* devices, int32_t n_devices, int64_t* first_bad_row) {
  return normalizer_host_multi(x, rows, V, chunk, precision, m, d, devices, n_devices, first_bad_row);
}

void osmx_host_release(void) {
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& kv : g_ctx) {
    std::lock_guard<std::mutex> l2(kv.second->mu);
    if (kv.second->st[0]) {
      cudaSetDevice(kv.first.first);
      kv.second->release();
    }
  }
  cudaSetDevice(prev);
}

}  // extern "C"
