// vsplit.cu -- the cross-GPU V-split of one huge row (configs[4]) behind the
// C-ABI, NCCL on the caller's stream, no host round trip:
//
//   slice record (one launch, topk_wide.cu) -> ncclAllGather of the fixed-size
//   records (in place, rank order) -> one combine launch that merges them in
//   rank (= column) order -> vals / idx, or the merged (M, D) and the scale
//   pass over this rank's slice (softmax).
//
// The merge order is the reference's chunked normalizer (normalizer.hpp:
// 74-85) with the chunk boundaries at the rank boundaries; the top-K merge
// is the total order (value desc, index asc) of topk.hpp:37-43.  Every call
// is stream-ordered and CUDA-graph capturable (NCCL collectives capture).
//
// NCCL is resolved at run time (dlopen), preferring a libnccl.so.2 that is
// already loaded in the process (torch's), so a communicator made by either
// library is driven by the same one.  No link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "../../include/osmx_b200.h"
#include "common.cuh"
#include "internal.hpp"

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name)); };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.comm_count, "ncclCommCount");
    sym(api.comm_user_rank, "ncclCommUserRank");
    sym(api.all_gather, "ncclAllGather");
    sym(api.error_string, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count && api.comm_user_rank &&
             api.all_gather && api.error_string;
  });
  return api;
}

thread_local std::string t_nccl_err;

osmx_status nccl_status(ncclResult_t r) {
  if (r == ncclSuccess) return OSMX_OK;
  t_nccl_err = nccl().error_string ? nccl().error_string(r) : "nccl error";
  return OSMX_ERR_NCCL;
}
osmx_status cuda_st(cudaError_t e) {
  if (e == cudaSuccess) return OSMX_OK;
  t_nccl_err = cudaGetErrorString(e);
  return OSMX_ERR_CUDA;
}

// The merge identity (-inf, 0) with no candidates: the record of an empty
// slice (a rank whose column range is empty still joins the all-gather).
__global__ void k_identity_record(char* rec, int k) {
  const int t = threadIdx.x;
  if (t == 0) {
    float* h = reinterpret_cast<float*>(rec);
    h[0] = osmx_dev::kNegInf;
    h[1] = 0.0f;
    h[2] = -osmx_dev::kNegInf;
    reinterpret_cast<int*>(rec)[3] = k;
  }
  const size_t vo = 16, io = 16 + ((size_t)(4 * k + 7) / 8) * 8;
  for (int r = t; r < k; r += blockDim.x) {
    reinterpret_cast<float*>(rec + vo)[r] = osmx_dev::kNegInf;
    reinterpret_cast<long long*>(rec + io)[r] = -1LL;
  }
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// [header + slice-record region][gather buffer: nranks records][merged record]
size_t vsplit_layout(long long V, int kk, int nranks, size_t* gather_off, size_t* merged_off) {
  const size_t base = align256(osmx_host::workspace_bytes(osmx_host::kSliceRecord, 1, std::max(V, 1LL), kk));
  const size_t rb = osmx_host::record_bytes(kk);
  if (gather_off) *gather_off = base;
  if (merged_off) *merged_off = base + align256((size_t)nranks * rb);
  return base + align256((size_t)nranks * rb) + align256(rb);
}

// slice record -> all-gather; returns the gather buffer (nranks records).
osmx_status record_and_gather(const float* x, long long V, long long col0, int kk, ncclComm_t comm, char* ws,
                              size_t ws_bytes, cudaStream_t st, int* nranks_out, char** gather_out,
                              char** merged_out) {
  const NcclApi& api = nccl();
  if (!api.ok) {
    t_nccl_err = "libnccl.so.2 not found";
    return OSMX_ERR_NCCL;
  }
  int nranks = 0, rank = 0;
  osmx_status s = nccl_status(api.comm_count(comm, &nranks));
  if (!s) s = nccl_status(api.comm_user_rank(comm, &rank));
  if (s) return s;
  size_t goff = 0, moff = 0;
  if (ws_bytes < vsplit_layout(V, kk, nranks, &goff, &moff)) return OSMX_ERR_INVALID_ARG;
  const size_t rb = osmx_host::record_bytes(kk);
  char* gather = ws + goff;
  char* mine = gather + (size_t)rank * rb;
  if (V > 0) {
    osmx_host::TuningScope scope;
    osmx_host::tuning().shape = osmx_host::kShapeSplit;
    s = cuda_st(osmx_host::launch_slice_record(x, V, col0, kk, mine, ws, ws_bytes, st));
  } else {
    k_identity_record<<<1, 32, 0, st>>>(mine, kk);
    osmx_host::count_launch();
    s = cuda_st(cudaGetLastError());
  }
  if (s) return s;
  // in place: rank r's record already sits at gather + r * rb
  s = nccl_status(api.all_gather(mine, gather, rb, ncclUint8, comm, st));
  if (s) return s;
  *nranks_out = nranks;
  *gather_out = gather;
  *merged_out = ws + moff;
  return OSMX_OK;
}

}  // namespace

extern "C" {

const char* osmx_last_nccl_error(void) { return t_nccl_err.c_str(); }

int osmx_nccl_available(void) { return nccl().ok ? 1 : 0; }

osmx_status osmx_nccl_get_unique_id(void* id) {
  if (!id) return OSMX_ERR_INVALID_ARG;
  if (!nccl().ok) return OSMX_ERR_NCCL;
  ncclUniqueId u;
  osmx_status s = nccl_status(nccl().get_unique_id(&u));
  if (!s) std::memcpy(id, &u, sizeof(u));
  return s;
}

osmx_status osmx_nccl_comm_init(void** comm, int32_t nranks, const void* id, int32_t rank) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return OSMX_ERR_INVALID_ARG;
  if (!nccl().ok) return OSMX_ERR_NCCL;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  osmx_status s = nccl_status(nccl().comm_init_rank(&c, nranks, u, rank));
  if (!s) *comm = c;
  return s;
}

osmx_status osmx_nccl_comm_destroy(void* comm) {
  if (!comm) return OSMX_ERR_INVALID_ARG;
  if (!nccl().ok) return OSMX_ERR_NCCL;
  return nccl_status(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
}

size_t osmx_vsplit_workspace_bytes(int64_t V_slice, int32_t k, int32_t nranks) {
  if (nranks < 1) nranks = 1;
  osmx_host::TuningScope scope;
  osmx_host::tuning().shape = osmx_host::kShapeSplit;
  return vsplit_layout(V_slice, k > 0 ? k : 1, nranks, nullptr, nullptr);
}

osmx_status osmx_vsplit_softmax_topk(const float* x, int64_t V_slice, int64_t col0, int32_t k, void* comm,
                                     float* vals, int64_t* idx, void* ws, size_t ws_bytes, void* stream) {
  if (k < 1) return OSMX_ERR_INVALID_K;
  if (k > OSMX_MAX_K) return OSMX_ERR_UNSUPPORTED;
  if (V_slice < 0 || col0 < 0 || (V_slice > 0 && !x) || !comm || !vals || !idx || !ws) return OSMX_ERR_INVALID_ARG;
  osmx_host::TuningScope scope;
  osmx_host::tuning().shape = osmx_host::kShapeSplit;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int n = 0;
  char *gather = nullptr, *merged = nullptr;
  osmx_status s = record_and_gather(x, V_slice, col0, k, static_cast<ncclComm_t>(comm), static_cast<char*>(ws),
                                    ws_bytes, st, &n, &gather, &merged);
  if (s) return s;
  return cuda_st(osmx_host::launch_records_combine(gather, n, k, merged, vals, reinterpret_cast<long long*>(idx), ws,
                                                   st));
}

osmx_status osmx_vsplit_softmax(const float* x, int64_t V_slice, int64_t col0, float* y, void* comm, void* ws,
                                size_t ws_bytes, void* stream) {
  if (V_slice < 0 || col0 < 0 || (V_slice > 0 && (!x || !y)) || !comm || !ws) return OSMX_ERR_INVALID_ARG;
  osmx_host::TuningScope scope;
  osmx_host::tuning().shape = osmx_host::kShapeSplit;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int n = 0;
  char *gather = nullptr, *merged = nullptr;
  osmx_status s = record_and_gather(x, V_slice, col0, 1, static_cast<ncclComm_t>(comm), static_cast<char*>(ws),
                                    ws_bytes, st, &n, &gather, &merged);
  if (s) return s;
  s = cuda_st(osmx_host::launch_records_combine(gather, n, 0, merged, nullptr, nullptr, ws, st));
  if (s || V_slice == 0) return s;
  return cuda_st(osmx_host::launch_scale_with_record(x, V_slice, merged, y, st));
}

}  // extern "C"
