// normalizer.cu -- batched run_normalizer<T> / run_normalizer_chunked<T>
// (reference normalizer.hpp:61-85) for T = float and double.
//
// The chunked contract: each contiguous chunk of chunk_len elements is
// reduced to a norm_state, and the chunk states are merged LEFT TO RIGHT
// (normalizer.hpp:77-83).  Here:
//   k_norm_chunks  one group per (row, chunk) -> record (m, d) in T.  Chunks
//                  of <= 32 elements are absorbed sequentially by one thread
//                  (the reference's own order, add() of normalizer.hpp:32-41);
//                  longer chunks by a warp or a CTA (per-lane sequential adds,
//                  then an Eq. 4 merge tree).
//   k_norm_fold    one thread per row folds its chunk records in chunk
//                  order with the reference's merge (identity operands
//                  returned unchanged, normalizer.hpp:53-58).
// T = double keeps the reference's double accumulation (kernels.hpp:65) with
// the double exp; T = float uses expf like norm_state<float>.
// The unchunked fp32 normalizer (chunk == 0, or one chunk per row) is the
// log2-domain CTA reduction k_normalizer (softmax_impl.cuh).
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

using namespace osmx_dev;

namespace {

template <class T>
struct NState {
  T m;
  T d;
};

__device__ __forceinline__ float exp_t(float x) { return expf(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }
// Separately rounded multiply / add: the reference (x86-64 host code) never
// fuses a*b + c, so neither do we (nvcc would contract it into an FMA).
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <class T>
__device__ __forceinline__ NState<T> ns_identity() {
  return NState<T>{-(T)INFINITY, (T)0};
}

// norm_state::add (normalizer.hpp:32-41): the first element gives (x, 1)
// because exp(-inf) == 0.
template <class T>
__device__ __forceinline__ void ns_add(NState<T>& s, T x) {
  if (x > s.m) {
    s.d = add_rn(mul_rn(s.d, exp_t(s.m - x)), (T)1);
    s.m = x;
  } else {
    s.d = add_rn(s.d, exp_t(x - s.m));
  }
}

// merge (normalizer.hpp:53-58).
template <class T>
__device__ __forceinline__ NState<T> ns_merge(NState<T> a, NState<T> b) {
  if (isinf(a.m) && a.m < 0) return b;
  if (isinf(b.m) && b.m < 0) return a;
  const T m = a.m > b.m ? a.m : b.m;
  return NState<T>{m, add_rn(mul_rn(a.d, exp_t(a.m - m)), mul_rn(b.d, exp_t(b.m - m)))};
}

template <class T>
__device__ __forceinline__ NState<T> ns_shfl_merge(NState<T> s, int width) {
  for (int o = width / 2; o > 0; o >>= 1) {
    NState<T> t{__shfl_xor_sync(0xffffffffu, s.m, o), __shfl_xor_sync(0xffffffffu, s.d, o)};
    // lanes merge in index order (lower lane first) so every lane agrees
    s = ((threadIdx.x & o) == 0) ? ns_merge(s, t) : ns_merge(t, s);
  }
  return s;
}

// G threads per chunk: 1 (sequential), 32 (warp) or BLOCK (CTA).
template <class T, int G, int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_norm_chunks(const float* __restrict__ x, long long ldx, long long rows, long long V, long long chunk,
                  long long nch, NState<T>* __restrict__ rec, void* ws) {
  constexpr int GPB = BLOCK / G;  // groups per CTA
  const long long total = rows * nch;
  const int t = threadIdx.x % G;
  for (long long gi = (long long)blockIdx.x * GPB + threadIdx.x / G; gi - threadIdx.x / G < total;
       gi += (long long)gridDim.x * GPB) {
    const bool live = gi < total;
    const long long row = live ? gi / nch : 0, c = live ? gi % nch : 0;
    const long long c0 = c * chunk;
    const long long n = live ? std::min(chunk, V - c0) : 0;
    const float* p = x + row * ldx + c0;
    NState<T> s = ns_identity<T>();
    bool bad = false;
    for (long long j = t; j < n; j += G) {
      const float v = p[j];
      bad |= !isfinite(v);
      ns_add(s, (T)v);
    }
    if constexpr (G == 32) {
      s = ns_shfl_merge(s, 32);
      bad = __any_sync(0xffffffffu, bad);
    } else if constexpr (G == BLOCK) {
      s = ns_shfl_merge(s, 32);
      bad = __syncthreads_or(bad);
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
      constexpr int NW = BLOCK / 32;
      __shared__ NState<T> part[NW];
      if (l == 0) part[w] = s;
      __syncthreads();
      if (w == 0) {
        s = l < NW ? part[l] : ns_identity<T>();
        s = ns_shfl_merge(s, 32);
      }
      __syncthreads();
    }
    if (live && t == 0) {
      rec[gi] = s;
      if (bad) flag_bad_row(ws, row);
    }
  }
}

template <class T, class TO>
__global__ void __launch_bounds__(128)
    k_norm_fold(const NState<T>* __restrict__ rec, long long rows, long long nch, TO* __restrict__ m,
                TO* __restrict__ d) {
  pdl_wait();  // records come from k_norm_chunks
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const NState<T>* r = rec + row * nch;
  NState<T> acc = ns_identity<T>();
  for (long long c = 0; c < nch; ++c) acc = ns_merge(acc, r[c]);
  m[row] = (TO)acc.m;
  d[row] = (TO)acc.d;
}

inline long long n_chunks(long long V, long long chunk) { return (V + chunk - 1) / chunk; }

template <class T, class TO>
cudaError_t run_chunked(const float* x, long long ldx, long long rows, long long V, long long chunk, TO* m, TO* d,
                        void* ws, cudaStream_t st) {
  const long long nch = n_chunks(V, chunk);
  auto* rec = reinterpret_cast<NState<T>*>(static_cast<char*>(ws) + kWsHeader);
  const long long total = rows * nch;
  const long long cap = 1LL << 30;
  if (chunk <= 32) {
    const long long grid = std::min<long long>((total + 255) / 256, cap);
    k_norm_chunks<T, 1, 256><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, chunk, nch, rec, ws);
  } else if (chunk <= 8192) {
    const long long grid = std::min<long long>((total + 7) / 8, cap);
    k_norm_chunks<T, 32, 256><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, chunk, nch, rec, ws);
  } else {
    const long long grid = std::min<long long>(total, cap);
    k_norm_chunks<T, 256, 256><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, chunk, nch, rec, ws);
  }
  osmx_host::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_norm_fold<T, TO>, dim3((unsigned)((rows + 127) / 128)), dim3(128), 0, st,
                 (const NState<T>*)rec, rows, nch, m, d);
  osmx_host::count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

namespace osmx_host {

cudaError_t launch_normalizer_f32_tree(const float* x, long long ldx, long long rows, long long V, float* m,
                                       float* d, void* ws, cudaStream_t st);

bool normalizer_uses_tree(long long V, long long chunk, int precision) {
  return precision == 32 && (chunk == 0 || chunk >= V);
}

size_t normalizer_ws(long long rows, long long V, long long chunk, int precision) {
  if (rows < 1 || V < 1 || normalizer_uses_tree(V, chunk, precision)) return kWsHeader;
  const long long c = (chunk == 0 || chunk > V) ? V : chunk;
  const size_t rec = precision == 64 ? sizeof(NState<double>) : sizeof(NState<float>);
  return kWsHeader + ((size_t)rows * (size_t)n_chunks(V, c) * rec + 255) / 256 * 256;
}

cudaError_t launch_normalizer(const float* x, long long ldx, long long rows, long long V, long long chunk,
                              float* m, float* d, void* ws, cudaStream_t st) {
  if (normalizer_uses_tree(V, chunk, 32)) return launch_normalizer_f32_tree(x, ldx, rows, V, m, d, ws, st);
  return run_chunked<float, float>(x, ldx, rows, V, chunk, m, d, ws, st);
}

cudaError_t launch_normalizer_f64(const float* x, long long ldx, long long rows, long long V, long long chunk,
                                  double* m, double* d, void* ws, cudaStream_t st) {
  const long long c = (chunk == 0 || chunk > V) ? V : chunk;
  return run_chunked<double, double>(x, ldx, rows, V, c, m, d, ws, st);
}

}  // namespace osmx_host
