/*
 * osmx_b200.h -- C-ABI of the B200 (sm_100a) implementation of the online-
 * normalizer softmax and fused softmax+TopK (arXiv 1805.02867).
 *
 * This is the drop-in boundary for the reference library `osmx`
 * (/root/reference/proj).  The reference has no FFI: its seam is the C++
 * header API.  Each entry point below names the
 * reference interface it replaces; include/osmx/b200.hpp re-exposes them
 * under the reference's own C++ signatures and exception types.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes; no C++ or torch types.
 *   - Device-pointer entry points are stream-ordered, allocate nothing, and
 *     return argument errors synchronously.  `stream` is a cudaStream_t
 *     (NULL = legacy default stream).
 *   - Rows are row-major with a leading dimension in ELEMENTS (ld >= V).
 *   - The workspace `ws` is caller-owned device memory of at least
 *     osmx_workspace_bytes(...) bytes, zero-initialised once with
 *     osmx_workspace_init.  Non-finite input rows are reported through it
 *     (osmx_check_status), like the reference's non_finite_error
 *     (error.hpp:13-15); their outputs are unspecified.  A workspace also
 *     carries the split paths' records, ticket counters and chunk counter
 *     (reset by the kernels that use them): calls that may run concurrently
 *     (different streams) need different workspaces; calls ordered on one
 *     stream may share one.
 *   - Host-buffer entry points (suffix _host) mirror the reference's
 *     span-in / vector-out functions for a whole batch: they copy in, run,
 *     copy out and synchronise, and report non-finite input synchronously.
 */
#ifndef OSMX_B200_H
#define OSMX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  1..4 are the reference's four exception types
 * (error.hpp:8-25), in that order. */
typedef enum {
  OSMX_OK = 0,
  OSMX_ERR_EMPTY = 1,         /* empty_input_error   error.hpp:8-10  */
  OSMX_ERR_NON_FINITE = 2,    /* non_finite_error    error.hpp:13-15 */
  OSMX_ERR_INVALID_K = 3,     /* invalid_k_error     error.hpp:18-20 */
  OSMX_ERR_INVALID_CHUNK = 4, /* invalid_chunk_error error.hpp:23-25 */
  OSMX_ERR_INVALID_ARG = 5,   /* null pointer, ld < V, bad enum, ws too small */
  OSMX_ERR_CUDA = 6,          /* a CUDA runtime error (see osmx_last_cuda_error) */
  OSMX_ERR_UNSUPPORTED = 7,   /* split / slice records with k > OSMX_MAX_K; top-K with
                                 V >= 2^31 or rows * k >= 2^31 when k > OSMX_MAX_K */
  OSMX_ERR_NCCL = 8           /* NCCL missing or a NCCL call failed (osmx_last_nccl_error) */
} osmx_status;

/* Algorithm ids: the reference's `algorithm` enum order (counting.hpp:17-24)
 * plus the unfused online->TopK pipeline the north star compares against. */
typedef enum {
  OSMX_NAIVE_SOFTMAX = 0,               /* naive_softmax           softmax.hpp:17 */
  OSMX_SAFE_SOFTMAX = 1,                /* safe_softmax            softmax.hpp:22 */
  OSMX_ONLINE_SOFTMAX = 2,              /* online_softmax          softmax.hpp:28 */
  OSMX_SAFE_SOFTMAX_UNFUSED_TOPK = 3,   /* safe_softmax_then_topk  topk.hpp:58 */
  OSMX_SAFE_SOFTMAX_FUSED_TOPK = 4,     /* safe_softmax_fused_topk topk.hpp:63 */
  OSMX_ONLINE_SOFTMAX_FUSED_TOPK = 5,   /* online_softmax_topk     topk.hpp:68 */
  OSMX_ONLINE_SOFTMAX_UNFUSED_TOPK = 6  /* online_softmax then topk_of (new) */
} osmx_algorithm;

/* Largest k of the fused register top-K lists and of the fixed-size split /
 * slice records.  Top-K calls accept any 1 <= k <= V (the reference's
 * contract, kernels.hpp:28-30); k > OSMX_MAX_K takes the radix-select path
 * (csrc/topk_large.cu), whose workspace grows with rows * k. */
#define OSMX_MAX_K 32
#define OSMX_VERSION 100

int osmx_version(void);
const char* osmx_status_string(osmx_status s);
/* The last CUDA error string seen by this thread (empty if none). */
const char* osmx_last_cuda_error(void);

/* ---------------------------------------------------------- workspace -- */

/* Bytes of workspace for one call of `alg` on rows x V (k for top-K algs;
 * alg 7 = osmx_topk, 8 = osmx_normalizer, 9 = osmx_slice_record,
 * 10 = osmx_proj_softmax_topk with V = vocabulary columns). 
 * Always >= 128 (the status header). */
size_t osmx_workspace_bytes(int alg, int64_t rows, int64_t V, int32_t k);
osmx_status osmx_workspace_init(void* ws, size_t ws_bytes, void* stream);
/* Synchronises `stream`, reads the non-finite flag the kernels set since the
 * last check, and clears it.  *first_bad_row = -1 when every row was finite,
 * else the lowest row index that held a NaN/inf (then returns
 * OSMX_ERR_NON_FINITE). */
osmx_status osmx_check_status(void* ws, void* stream, int64_t* first_bad_row);

/* ------------------------------------------------- batched, device ptrs -- */

/* Softmax of every row.  alg in {NAIVE, SAFE, ONLINE}_SOFTMAX.
 * Replaces naive_softmax / safe_softmax / online_softmax (softmax.hpp:17-28,
 * softmax.cpp:19-29) applied to each row; y is caller-owned (the reference
 * returns a fresh std::vector, softmax.cpp:12). */
osmx_status osmx_softmax(int alg, const float* x, int64_t ldx, float* y, int64_t ldy, int64_t rows,
                         int64_t V, void* ws, size_t ws_bytes, void* stream);

/* Top-K of every row's softmax: vals/idx are rows x k (row-major).
 * alg in {SAFE_SOFTMAX_UNFUSED_TOPK, SAFE_SOFTMAX_FUSED_TOPK,
 * ONLINE_SOFTMAX_FUSED_TOPK, ONLINE_SOFTMAX_UNFUSED_TOPK}.
 * Replaces safe_softmax_then_topk / safe_softmax_fused_topk /
 * online_softmax_topk (topk.hpp:58-68, topk.cpp:30-55). */
osmx_status osmx_softmax_topk(int alg, const float* x, int64_t ldx, int64_t rows, int64_t V,
                              int32_t k, float* vals, int64_t* idx, void* ws, size_t ws_bytes,
                              void* stream);

/* Top-K of arbitrary values per row.  Replaces topk_of (topk.hpp:54,
 * topk.cpp:20-28). */
/* The projection layer fused with the online softmax + top-K:
 * for each of `rows` bf16 vectors h (row-major rows x D) and the bf16 weight
 * W (row-major V x D), the top-k of softmax(h W^T) -- values e^(z - m)/d and
 * column indices, ties to the lower column -- without writing the logits z
 * (tcgen05 tensor cores, fp32 accumulation).  D % 8 == 0, h / W 16-byte
 * aligned, 1 <= k <= OSMX_MAX_K.  This op has no reference counterpart; its
 * result equals online_softmax_topk (topk.hpp:68) of the fp32 logits. */
osmx_status osmx_proj_softmax_topk(const void* h, int64_t rows, int64_t D, const void* w, int64_t V, int32_t k,
                                   float* vals, int64_t* idx, void* ws, size_t ws_bytes, void* stream);

osmx_status osmx_topk(const float* v, int64_t ld, int64_t rows, int64_t V, int32_t k, float* vals,
                      int64_t* idx, void* ws, size_t ws_bytes, void* stream);

/* (m, d) of every row.  Replaces run_normalizer<T> /
 * run_normalizer_chunked<T> (normalizer.hpp:61-85): chunk = 0 is the
 * unchunked pass; chunk > 0 reduces every contiguous chunk of `chunk`
 * elements to a state and merges the chunk states left to right
 * (normalizer.hpp:77-83), one record per chunk in the workspace.  (The
 * reference rejects chunk_len == 0 with invalid_chunk_error; its C++ facade
 * include/osmx/normalizer.hpp keeps that check, 0 here means "unchunked".)
 * chunk >= V is one chunk, bit-identical to chunk = 0 (test_normalizer.cpp
 * "single chunk is bit-identical to sequential").  The workspace must hold
 * osmx_normalizer_workspace_bytes(rows, V, chunk, 32 | 64) bytes.
 * _f64 keeps the state in double like norm_state<double> (the reference's
 * kernels accumulate d in double, kernels.hpp:65). */
size_t osmx_normalizer_workspace_bytes(int64_t rows, int64_t V, int64_t chunk, int32_t precision);
osmx_status osmx_normalizer(const float* x, int64_t ldx, int64_t rows, int64_t V, int64_t chunk,
                            float* m, float* d, void* ws, size_t ws_bytes, void* stream);
osmx_status osmx_normalizer_f64(const float* x, int64_t ldx, int64_t rows, int64_t V, int64_t chunk,
                                double* m, double* d, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------- V-split records (multi-GPU rows) -- */

/* A record is the (m, d) state plus k (value, index) candidates of one row
 * slice: the operand of the paper's merge (Eq. 4-5; normalizer.hpp:52-58,
 * topk.hpp:34-44).  Fixed size per k, so n records all-gather as one
 * contiguous buffer. */
size_t osmx_record_bytes(int32_t k);
/* Record of the slice x[0..V) of one row whose first element is global
 * column col0.  k = 0: (m, d) only (softmax V-split). */
osmx_status osmx_slice_record(const float* x, int64_t V, int64_t col0, int32_t k, void* record,
                              void* ws, size_t ws_bytes, void* stream);
/* Merge n records (in rank / column order) into out_record (optional) and,
 * for k > 0, into the final vals[k] = e^(u - M)/D, idx[k] (optional). */
osmx_status osmx_records_combine(const void* records, int32_t n, int32_t k, void* out_record,
                                 float* vals, int64_t* idx, void* ws, size_t ws_bytes,
                                 void* stream);
/* y = e^(x - M)/D over a slice, (M, D) from a combined record. */
osmx_status osmx_scale_with_record(const float* x, int64_t V, const void* record, float* y,
                                   void* stream);

/* ------------------------------------------- V-split over NCCL (C5) -- */

/* One row too long for one device, split into contiguous column slices, one
 * per rank of an NCCL communicator (rank r holds columns [col0, col0 +
 * V_slice); slices in rank order cover the row).  Each call is three
 * stream-ordered steps on `stream`, capturable in a CUDA graph, no host
 * synchronisation: this rank's slice record (one launch) -> ONE
 * ncclAllGather of the fixed-size records (in place, rank order) -> the
 * rank-order merge (normalizer.hpp:74-85 with the chunk boundaries at the
 * rank boundaries; top-K under (value desc, index asc), topk.hpp:37-43).
 * Every rank gets the same outputs.  An empty slice (V_slice = 0) joins with
 * the merge identity.  Non-finite input is reported through ws (row 0) by
 * osmx_check_status.  `comm` is an ncclComm_t: from osmx_nccl_comm_init or
 * the caller's own (NCCL is loaded at run time, preferring the libnccl.so.2
 * already in the process). */
int osmx_nccl_available(void);
const char* osmx_last_nccl_error(void);
/* 128-byte ncclUniqueId (rank 0 makes it, the caller broadcasts it). */
osmx_status osmx_nccl_get_unique_id(void* id128);
osmx_status osmx_nccl_comm_init(void** comm, int32_t nranks, const void* id128, int32_t rank);
osmx_status osmx_nccl_comm_destroy(void* comm);
size_t osmx_vsplit_workspace_bytes(int64_t V_slice, int32_t k, int32_t nranks);
/* online_softmax_topk (topk.hpp:68) of the whole row: vals[k], idx[k] with
 * global column indices, on every rank. */
osmx_status osmx_vsplit_softmax_topk(const float* x_slice, int64_t V_slice, int64_t col0, int32_t k, void* comm,
                                     float* vals, int64_t* idx, void* ws, size_t ws_bytes, void* stream);
/* online_softmax (softmax.hpp:28) of the whole row: this rank's slice of it
 * in y_slice (V_slice floats).  ws: osmx_vsplit_workspace_bytes(V_slice, 0, n). */
osmx_status osmx_vsplit_softmax(const float* x_slice, int64_t V_slice, int64_t col0, float* y_slice, void* comm,
                                void* ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------- host buffers (e2e) -- */

/* Batched host-memory versions of the same algorithms: x, y, vals, idx are
 * HOST pointers (pinned memory is copied directly; pageable memory is
 * staged by the driver).  The library streams row blocks through device
 * staging buffers on `device`, overlapping H2D, kernels and D2H on two CUDA
 * streams, and returns after the results are in host memory.
 * first_bad_row (optional) receives -1 or the first non-finite row. */
osmx_status osmx_softmax_host(int alg, const float* x, int64_t rows, int64_t V, float* y,
                              int device, int64_t* first_bad_row);
osmx_status osmx_softmax_topk_host(int alg, const float* x, int64_t rows, int64_t V, int32_t k,
                                   float* vals, int64_t* idx, int device, int64_t* first_bad_row);
/* topk_of over host values (topk.hpp:54). */
osmx_status osmx_topk_host(const float* v, int64_t rows, int64_t V, int32_t k, float* vals, int64_t* idx,
                           int device, int64_t* first_bad_row);
/* Multi-device row sharder of the host path (the reference's run_batch
 * stripes rows over std::threads, bench.cpp:66-96): devices[i] takes the
 * contiguous rows [rows*i/n, rows*(i+1)/n) on its own host thread, staging
 * buffers, streams and PCIe link; no inter-device communication.  A device
 * may be listed more than once (one staging context per entry).  Errors: the
 * first failing entry in list order; else OSMX_ERR_NON_FINITE with the lowest
 * bad row over all devices.  Thread-safe; launch knobs are the caller's
 * osmx_config_set defaults at the time of the call. */
osmx_status osmx_softmax_host_multi(int alg, const float* x, int64_t rows, int64_t V, float* y,
                                    const int* devices, int32_t n_devices, int64_t* first_bad_row);
osmx_status osmx_softmax_topk_host_multi(int alg, const float* x, int64_t rows, int64_t V, int32_t k,
                                         float* vals, int64_t* idx, const int* devices, int32_t n_devices,
                                         int64_t* first_bad_row);
osmx_status osmx_topk_host_multi(const float* v, int64_t rows, int64_t V, int32_t k, float* vals,
                                 int64_t* idx, const int* devices, int32_t n_devices,
                                 int64_t* first_bad_row);
/* Host-buffer normalizer (run_normalizer / run_normalizer_chunked over a
 * batch of rows): m, d are rows floats (precision 32) or doubles (64). */
osmx_status osmx_normalizer_host(const float* x, int64_t rows, int64_t V, int64_t chunk, int32_t precision,
                                 void* m, void* d, const int* devices, int32_t n_devices,
                                 int64_t* first_bad_row);
/* Release the per-device staging buffers of the host path. */
void osmx_host_release(void);

/* ---------------------------------------------------------- telemetry -- */

/* Number of kernel launches issued by this library since load. */
uint64_t osmx_launch_count(void);
/* Diagnostic: a pure read stream over `bytes` (16-byte aligned) -- the
 * 128-bit grid-stride max-fold the fused top-K's loads reduce to -- so a
 * bench can state the achievable read bandwidth of the same buffer.
 * Writes one float to `sink` (device); stream-ordered. */
osmx_status osmx_diag_read_probe(const void* x, size_t bytes, float* sink, void* stream);
/* Launch-layer knobs (tuning and measurement only):
 *   "shape"          0 auto, 1 resident, 2 stream, 3 split, 4 staged, 5 cluster-staged
 *   "resident_max_v" largest V held in registers (<= 16384)
 *   "split_chunk"    elements per CTA / warp piece in split mode (0 = auto)
 *   "stream_threads" CTA size of the stream kernels (0, 256, 512, 1024)
 *   "stream_ctas"    persistent stream CTAs per SM with evict-last pass 1 (0 = off)
 *   "staged_gw" / "staged_ng" / "staged_kb" / "cluster_size"   staged layouts (0 = auto)
 *   "topk_threads"   threads per row of the row top-K (0 auto, 32, 128, 256, 512)
 *   "topk_u8" / "topk_pipe" / "l2_prefetch" / "tma"   top-K row-kernel variants
 *   "split_cta"      top-K split records: -1 auto, 0 warp pieces, 1 CTA chunks,
 *                    2 TMA-ring CTA pieces, 3 one-launch grid-stride, 4 one row:
 *                    TMA ring over dynamically claimed chunks (auto for one row)
 *   "split_fuse"     TMA pieces: merge in the last piece CTA (1) or a combine launch (0)
 *   "tma_cfg"        TMA-ring layout for fused k <= 5 (-1 auto, 0, 1, 2)
 *   "topk_block"     threads per CTA of the one-wave warp-per-row top-K (0 auto, 32, 128)
 *   "large_fast"     k > 32: two-pass shared-memory selection (1) or radix + CUB (0)
 *   "corun"          online softmax, 16-CTA-cluster rows: percent of rows in clusters,
 *                    the rest streamed on a side stream (-1 auto = 80, 0 off)
 *   "proj_bn"        fused projection vocabulary tile (0 auto, 128, 224, 256)
 *   "host_chunk_mb"  staging block of the host path (default 512)
 * Returns OSMX_ERR_INVALID_ARG for an unknown key or value. */
osmx_status osmx_config_set(const char* key, int64_t value);
int64_t osmx_config_get(const char* key);

#ifdef __cplusplus
}
#endif

#endif /* OSMX_B200_H */
