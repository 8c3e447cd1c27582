// internal.hpp -- host-side launch layer shared by the kernel translation
// units and the C-ABI (capi.cu).  Plain C++; no torch types anywhere.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace osmx_host {

// Algorithm ids: the reference's algorithm enum order (counting.hpp:17-24)
// plus the unfused online->TopK pipeline the north star adds.
enum Alg : int {
  kNaive = 0,
  kSafe = 1,
  kOnline = 2,
  kSafeUnfusedTopk = 3,
  kSafeFusedTopk = 4,
  kOnlineFusedTopk = 5,
  kOnlineUnfusedTopk = 6,
  kTopkOf = 7,
  kNormalizer = 8,
  kSliceRecord = 9,  // osmx_slice_record (workspace sizing only)
  kProjTopk = 10,    // osmx_proj_softmax_topk (projection fused with the online softmax top-K)
};

// Kernel-shape families chosen per (rows, V) by the launch layer.
enum Shape : int {
  kShapeAuto = 0,
  kShapeResident = 1,  // row held in registers by a group of <= 1024 threads
  kShapeStream = 2,    // one CTA per row, every pass streams global memory
  kShapeSplit = 3,     // row split over S CTAs, (m,d)/top-K records + combine
  kShapeStaged = 4,    // rows staged in a TMA-fed shared-memory ring (persistent)
  kShapeCluster = 5,   // row slices staged across a thread-block cluster (DSMEM merge)
};

struct Tuning {
  int shape = kShapeAuto;       // force a family (0 = heuristic)
  int resident_max_v = 2048;    // largest V held in registers (above: staged up to 16K)
  long long split_chunk = 0;    // elements per CTA in split mode (0 = auto)
  int stream_threads = 0;       // CTA size for stream kernels (0 = auto)
  int stream_ctas = 0;          // stream softmax: persistent CTAs per SM + evict-last pass 1 (0 = off)
  int topk_threads = 0;         // CTA size for the fused top-K (0 = auto)
  int cluster_size = 0;         // cluster softmax: CTAs per row (0 auto; 1..16)
  int staged_gw = 0;            // staged softmax: warps per row group (0 auto; 1,2,4,8,16)
  int staged_ng = 0;            // staged softmax: row groups per CTA (0 auto; clamped to the slots)
  int staged_kb = 0;            // staged softmax: ring (shared memory) per CTA, KB (0 auto)
  int split_cta = -1;           // top-K split path: -1 auto, 0 warp-per-piece records, 1 CTA-per-chunk
                                // (legacy), 2 TMA-ring CTA per piece, 3 one-launch grid-stride
                                // (topk_wide.cu), 4 one row: TMA ring over dynamic chunks
  int proj_bn = 0;              // fused projection vocabulary tile (0 auto; 128, 256)
  int topk_pipe = 0;            // warp-per-row top-K via a cp.async smem pipeline (0 off; 1..3 layouts)
  int topk_u8 = -1;             // warp-per-row top-K with 8 float4s in flight (-1 auto)
  int l2_prefetch = -1;         // bulk L2 prefetch distance in batches (0 off, -1 auto)
  int split_fuse = 0;           // TMA split records: merge in the piece kernel (last piece, ticket) (1) or
                                // in a separate PDL combine launch (0; measured 2-3% faster on configs[4])
  int topk_block = 0;           // threads per CTA of the one-wave warp-per-row top-K (0 auto = 32, 32, 128)
  int tma = 0;                  // TMA-ring top-K: 0 off (default: the warp-per-row
                                // LDG kernel measures faster), 1 auto, 2 force
  int corun = -1;               // 16-CTA-cluster rows: percent of rows for the cluster kernel, the rest
                                // streamed concurrently on a side stream (-1 auto, 0 off)
  int large_fast = 1;           // k > 32: two-pass shared-memory path (1) or the radix + CUB path (0)
  int tma_cfg = -1;             // TMA-ring layout for fused k <= 5 (topk_tma.cu TmaCfg: -1 auto, 0, 1, 2)
};
// The knobs in force for the current call on this thread.  osmx_config_set
// writes process-wide defaults; every C-ABI entry point opens a TuningScope,
// which snapshots them into thread-local storage for the whole call, so a
// call never sees another thread's change (the reference is reentrant,
// softmax.hpp:8-9) and a call-local override (osmx_slice_record's forced
// split shape) never leaks into other threads or later calls.
Tuning& tuning();
Tuning tuning_defaults();
void tuning_set_defaults(const Tuning& t);
struct TuningScope {
  explicit TuningScope(const Tuning* t = nullptr);
  ~TuningScope();
  TuningScope(const TuningScope&) = delete;
  TuningScope& operator=(const TuningScope&) = delete;
 private:
  Tuning saved_;
  bool outer_;
};

// Kernel-launch tally (every launch the library issues increments it).
void count_launch(int n = 1);

int num_sms();

// A per-thread, per-device side stream and fork / join events (capi.cu).
cudaError_t side_stream(cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join);

// True the first time it is called for (current device, fn): function
// attributes (dynamic shared memory, cluster size) are per device context.
bool first_use_on_device(const void* fn);

// ---------------------------------------------------------------- launchers
// All pointers are device pointers.  ws points at the workspace header; the
// split region (if any) starts at ws + kWsHeader.  Return cudaError_t.

cudaError_t launch_softmax(int alg, const float* x, long long ldx, float* y, long long ldy,
                           long long rows, long long V, void* ws, size_t ws_bytes, cudaStream_t st);

cudaError_t launch_topk(int alg, const float* x, long long ldx, long long rows, long long V, int k,
                        float* vals, long long* idx, void* ws, size_t ws_bytes, cudaStream_t st);

// normalizer.cu: run_normalizer / run_normalizer_chunked (normalizer.hpp:61-85).
// chunk 0 = unchunked; precision 32 (float state) or 64 (double state).
cudaError_t launch_normalizer(const float* x, long long ldx, long long rows, long long V,
                              long long chunk, float* m, float* d, void* ws, cudaStream_t st);
cudaError_t launch_normalizer_f64(const float* x, long long ldx, long long rows, long long V,
                                  long long chunk, double* m, double* d, void* ws, cudaStream_t st);
size_t normalizer_ws(long long rows, long long V, long long chunk, int precision);

// Split-mode record of one row slice: (m, d, min) + k candidates.
size_t record_bytes(int k);
// Partial record of one row slice [x, x+V) whose global column offset is
// col0; the combine of n records (rank order) into one record, and into the
// final (vals, idx) when k > 0; the softmax scale pass against a record.
cudaError_t launch_slice_record(const float* x, long long V, long long col0, int k, void* record,
                                void* ws, size_t ws_bytes, cudaStream_t st);
cudaError_t launch_records_combine(const void* records, int n, int k, void* out_record,
                                   float* vals, long long* idx, void* ws, cudaStream_t st);
cudaError_t launch_scale_with_record(const float* x, long long V, const void* record, float* y,
                                     cudaStream_t st);

size_t workspace_bytes(int alg, long long rows, long long V, int k);

// softmax.cu
size_t softmax_split_ws(long long rows, long long V);
int resident_limit(bool vec);  // largest V for the resident family
bool softmax_uses_split(long long rows, long long V);
// Safe split phases 0 and 1 (row max, then d against it) into 16-byte
// records {float m, float mn, double d} (the safe fused top-K's first passes).
cudaError_t launch_safe_split_stats(const float* x, long long ldx, long long rows, long long V,
                                    long long chunk, void* srec, cudaStream_t st);

// topk.cu.  mode: 0 fused online, 1 topk_of, 2 safe fused.
size_t topk_split_ws(int alg, long long rows, long long V, int k);
bool topk_split(long long rows, long long V);
cudaError_t launch_topk_mode(int mode, const float* x, long long ldx, long long rows, long long V,
                             int k, float* vals, long long* idx, void* ws, cudaStream_t st);

// proj_topk.cu: logits = H W^T on tcgen05 tensor cores, never written to
// HBM; per-(row, 256-column tile) records + the split combine.
size_t proj_topk_ws(long long rows, long long V, int k);
cudaError_t launch_proj_topk(const void* h, long long rows, long long D, const void* w, long long V, int k,
                             float* vals, long long* idx, void* ws, cudaStream_t st);

// Diagnostic read stream (tools/read_peak.cu's probe), capi.cu osmx_diag_read_probe.
cudaError_t launch_read_probe(const void* x, size_t bytes, float* sink, cudaStream_t st);

// Largest k served by the register top-K lists (and by split records).
constexpr int kMaxK = 32;

// topk_large.cu: any k above kMaxK (radix select + ordered compaction +
// stable segmented sort).  region = workspace after the header.
size_t topk_large_ws(long long rows, long long V, int k);
// TMA-ring top-K in record mode (split path): resident CTAs on the device
// for this k, and the launch over rows * R pieces of `chunk` columns.
long long topk_tma_slots(int k);
// One row, dynamic stage-sized chunks claimed from a workspace counter, one
// record per resident CTA, the last CTA merges (topk_tma.cu).
cudaError_t launch_topk_tma_dyn(int mode, const float* x, long long V, int k, float* vals, long long* idx, void* ws,
                                cudaStream_t st, long long col0, char* rec, char* out_rec);
// topk_wide.cu: one-launch grid-stride split with a fused last-CTA combine
// (few rows, V < 2^31, rows <= 992): resident CTAs for this k and the launch.
long long topk_wide_slots(int k);
cudaError_t launch_topk_wide(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                             float* vals, long long* idx, void* ws, cudaStream_t st, long long col0, char* out_rec);
// vals / out_rec non-null: the last-finishing piece of each row merges the
// row's records in the same launch (rows <= kWsMaxTickets); else the caller
// launches the combine.
cudaError_t launch_topk_tma_records(int mode, const float* x, long long ldx, long long pieces, long long V, int k,
                                    void* ws, cudaStream_t st, int R, long long chunk, long long col0, char* rec,
                                    float* vals = nullptr, long long* idx = nullptr, char* out_rec = nullptr);
bool topk_large_supported(long long rows, long long V, int k);
cudaError_t launch_topk_large(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                              float* vals, long long* idx, void* ws, void* region, cudaStream_t st);

}  // namespace osmx_host
