// topk_impl.cuh -- batched top-K kernels for sm_100a.
//
// Replaces the reference's
//   online_softmax_topk_kernel      kernels.hpp:108-125  (Alg. 4: ONE access
//                                   per element; (m,d) and the top-K of the
//                                   raw logits in the same pass)
//   topk_kernel / topk_of           kernels.hpp:72-83, topk.cpp:20-28
//   safe_softmax_fused_topk_kernel  kernels.hpp:87-104 (3 passes, selection
//                                   on float(e^(x-m)/d))
// The unfused pipelines (safe_softmax_then_topk, topk.cpp:30-35, and the
// online->TopK comparator of the north star) are a softmax kernel followed
// by the topk_of kernel here.
//
// Selection is exact: per-thread register lists insert with the reference's
// strict '>' (topk.hpp:37-43) over elements seen in increasing index order,
// and every merge level (warp, CTA, split chunk, GPU) uses the total order
// (value desc, index asc) of oracle.cpp:48-51.  Indices are int64 on output
// (topk.hpp:16).
#pragma once
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"
#include "stream.cuh"

using namespace osmx_dev;

namespace {

enum Mode : int { kModeFused = 0, kModeTopkOf = 1, kModeSafe = 2 };

// ----------------------------------------------------- record (chunk) --
// Shared by the split path and the cross-GPU combine:
//   float m, d, mn; int k; float v[k] (8-byte padded); int64 idx[k]
struct RecHdr {
  float m;
  float d;
  float mn;  // min of the slice (or NaN when a non-finite value was seen)
  int k;
};
__host__ __device__ inline size_t rec_vals_off() { return sizeof(RecHdr); }
__host__ __device__ inline size_t rec_idx_off(int k) { return sizeof(RecHdr) + ((size_t)(4 * k + 7) / 8) * 8; }
__host__ __device__ inline size_t rec_bytes_(int k) { return ((rec_idx_off(k) + 8 * (size_t)k) + 15) / 16 * 16; }

// --------------------------------------------------- per-thread pass --
// State of one thread over the elements it owns: (m, d), min / check,
// and the top list.  FUSED: list over raw x + online (m,d).  TOPK_OF: list
// over x + finiteness check.  SAFE (select pass): list over p.
template <int KC, int U, int MODE, int G>
struct Pass {
  TopList<KC> L;
  L2Acc acc;  // online (m, d) of the fused mode
  float mn = -kNegInf, chk = 0.0f;
  float M = 0.0f;   // SAFE select pass: row max
  double D = 1.0;   //                   and the double normalizer
  // SAFE: x-space image of the admission bound.  The key float(e^(x-M)/D)
  // is monotone in x, so key(x) >= T implies x >= M + ln(T D) up to the
  // roundings of x - M, expf and the quotient (a few 1e-7 relative); xlo
  // sits 1e-5 (relative) below that, and a batch whose raw max is under it
  // skips the double-precision key entirely.
  float xlo = kNegInf;
  __device__ __forceinline__ void upd_xlo() {
    if constexpr (MODE == kModeSafe) {
      if (T > 0.0f) {
        const double xl = (double)M + log((double)T * D);
        xlo = (float)(xl - 1e-5 * (1.0 + fabs(xl) + fabs(xl - (double)M)));
      }
    }
  }

  __device__ __forceinline__ void scalar(float v, int j, int k) {
    if constexpr (MODE == kModeFused) {
      mn = fminf(mn, v);
      acc.add1(v);
      L.offer(v, j);
    } else if constexpr (MODE == kModeTopkOf) {
      chk = fmaf(v, 0.0f, chk);  // NaN iff some element was inf / NaN
      L.offer(v, j);
    } else {
      L.offer(safe_key_ref(v, M, D), j);
    }
  }
  __device__ __forceinline__ void batch(const Seg& s, float4 (&v)[U], long long q0, int cnt, int k) {
    batch_j(v, cnt, (int)body_index(s, q0, 0), 4 * G);
  }
  // Warp-shared admission bound: the max over (converged) lanes of their own
  // k-th best.  Every lane's k-th best is <= the row's k-th best, so an
  // element below T can never be selected; elements equal to T are kept
  // (index ties).  It keeps warps out of the insertion path after the first
  // few batches -- without it one inserting lane drags the whole warp in.
  float T = kNegInf;
  int* Tsh = nullptr;    // CTA-shared bound (ordered-int float) when the CTA owns one row
  float best = kNegInf;  // the lane's best key so far
  int kk = 1;            // runtime k (set by the kernel)

  __device__ __forceinline__ static int f2o(float f) {
    const int i = __float_as_int(f);
    return i ^ ((i >> 31) & 0x7fffffff);
  }
  __device__ __forceinline__ static float o2f(int i) { return __int_as_float(i ^ ((i >> 31) & 0x7fffffff)); }

  template <class KeyF>
  __device__ __forceinline__ void select_batch(float4 (&v)[U], int cnt, int j0, int jstride, float bkey,
                                               KeyF&& key) {
    const unsigned mask = __activemask();
    best = fmaxf(best, bkey);
    bool want = bkey > L.thr() && bkey >= T;
    // common case: one vote, no lane can admit anything
    if (!__any_sync(mask, want)) return;
    if (Tsh) {
      T = fmaxf(T, o2f(*reinterpret_cast<volatile int*>(Tsh)));  // other warps' progress
      want = bkey > L.thr() && bkey >= T;
    }
    if (!Tsh || __any_sync(mask, want)) {
      // Raise T before inserting: the k-th largest of the lanes' bests
      // (this batch included) is a valid lower bound of the row's k-th best
      // (k distinct elements >= it), so only elements >= it are offered --
      // in the first batch that is ~k elements per warp instead of all.
      if (__popc(mask) >= kk) {
        int mine = f2o(best), kth = mine;
        for (int r = 0; r < kk; ++r) {
          kth = __reduce_max_sync(mask, mine);
          const unsigned who = __ballot_sync(mask, mine == kth);
          if ((int)(threadIdx.x & 31) == __ffs(who) - 1) mine = f2o(kNegInf);
        }
        T = fmaxf(T, o2f(kth));
      }
      if (bkey > L.thr() && bkey >= T) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u >= cnt) break;  // padding of the last batch is never offered
          // key is monotone: one test per float4 before the per-element ones
          if (!(key(fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w))) >= T)) continue;
          const int j = j0 + u * jstride;
          const float k0 = key(v[u].x), k1 = key(v[u].y), k2 = key(v[u].z), k3 = key(v[u].w);
          if (k0 >= T) L.offer(k0, j);
          if (k1 >= T) L.offer(k1, j + 1);
          if (k2 >= T) L.offer(k2, j + 2);
          if (k3 >= T) L.offer(k3, j + 3);
        }
      }
      // the best lane k-th is a lower bound too
      T = fmaxf(T, o2f(__reduce_max_sync(mask, f2o(L.thr()))));
      if (Tsh && (int)(threadIdx.x & 31) == __ffs(mask) - 1) atomicMax(Tsh, f2o(T));
      upd_xlo();
    }
  }

  // v[u] holds elements j0 + u*jstride + {0,1,2,3} (u < cnt valid).
  __device__ __forceinline__ void batch_j(float4 (&v)[U], int cnt, int j0, int jstride) {
    if constexpr (MODE == kModeFused) {
      float bm = kNegInf, bn = -kNegInf;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
        if (u < cnt) bn = fminf(bn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
      }
      if (cnt > 0) {  // an empty batch (TMA tail) must not touch (m, d): e^(-inf - -inf)
        mn = fminf(mn, bn);
        acc.raise(bm);
        acc.add_batch<U>(v);
      }
      select_batch(v, cnt, j0, jstride, bm, [](float e) { return e; });
    } else if constexpr (MODE == kModeTopkOf) {
      float bm = kNegInf;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
        if (u < cnt) {
          chk = fmaf(v[u].x, 0.0f, chk);
          chk = fmaf(v[u].y, 0.0f, chk);
          chk = fmaf(v[u].z, 0.0f, chk);
          chk = fmaf(v[u].w, 0.0f, chk);
        }
      }
      select_batch(v, cnt, j0, jstride, bm, [](float e) { return e; });
    } else {
      // p is monotone in x for a fixed row (M, D): filter on the batch max.
      float bm = kNegInf;
#pragma unroll
      for (int u = 0; u < U; ++u) bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
      // no lane can admit anything: skip the keys (warp-uniform)
      if (!__any_sync(__activemask(), bm >= xlo)) return;
      const float Mr = M;
      const double Dr = D;
      select_batch(v, cnt, j0, jstride, safe_key_ref(bm, Mr, Dr),
                   [Mr, Dr](float e) { return safe_key_ref(e, Mr, Dr); });
    }
  }
};

// Safe fused top-K needs the row max and 1/d before the selection pass.
template <int G, int U>
__device__ __forceinline__ void safe_max_min(const Seg& s, int t, float& m, float& mn) {
  stream_seg<G, U, false>(
      s, t,
      [&](float v, long long) {
        m = fmaxf(m, v);
        mn = fminf(mn, v);
        if (v != v) mn = v;
      },
      [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
          if (u < cnt) mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
        }
      });
}
// d = sum exp(double(x) - m) in double, as the reference (kernels.hpp:95-96):
// the selection keys divide by it, so it must be accurate far below an fp32
// ulp for the keys to round like the reference's.  Padding (-inf) adds 0.
template <int G, int U>
__device__ __forceinline__ double safe_sum(const Seg& s, int t, float M, const double* tab) {
  const double Md = (double)M;
  double d = 0.0;
  stream_seg<G, U, false>(
      s, t, [&](float v, long long) { d += exp_neg_d((double)v - Md, tab); },
      [&](float4 (&v)[U], long long, int) {
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          sum += (exp_neg_d((double)v[u].x - Md, tab) + exp_neg_d((double)v[u].y - Md, tab)) +
                 (exp_neg_d((double)v[u].z - Md, tab) + exp_neg_d((double)v[u].w - Md, tab));
        d += sum;
      });
  return d;
}

template <int G, int U, int KC, int MODE>
__device__ __forceinline__ void run_pass(Pass<KC, U, MODE, G>& P, const Seg& s, int t, int k, int pf = 0) {
  stream_seg<G, U, MODE == kModeSafe>(
      s, t, [&](float v, long long j) { P.scalar(v, (int)j, k); },
      [&](float4 (&v)[U], long long q0, int cnt) { P.batch(s, v, q0, cnt, k); }, pf);
}

// Cross-warp merge for a CTA-wide group: each warp's k winners go to smem,
// warp 0 merges them.  sv/si hold NW*KC entries.
template <int NW, int KC, class Sink>
__device__ __forceinline__ void cta_merge(TopList<KC>& L, int k, float* sv, int* si, Sink&& sink) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  L.normalize(k);
  group_merge<32>(L, k, [&](int r, float v, int i) {
    if (l == 0) {
      sv[w * KC + r] = v;
      si[w * KC + r] = i;
    }
  });
  __syncthreads();
  if (w == 0) {
    TopList<KC> M;
    M.init_empty();
    if (l < NW) {
#pragma unroll
      for (int r = 0; r < KC; ++r)
        if (r < k) {
          M.v[r] = sv[l * KC + r];
          M.i[r] = si[l * KC + r];
        }
    }
    group_merge<32>(M, k, sink);
  }
  __syncthreads();
}

// ---------------------------------------------------------- row kernel --
// G threads per row (G == 32: warp per row, BLOCK/32 rows per CTA; G ==
// BLOCK: CTA per row).  Rows are visited grid-stride.
// NST > 0 (warp per row only): the body streams through a per-warp
// cp.async shared-memory pipeline of NST stages (stream_seg_pipe).
//
// Record mode (rec != nullptr; fused and topk_of): "rows" are pieces of R
// per input row -- piece s covers columns [r*chunk, min(V, (r+1)*chunk)) of
// input row s / R, r = s % R -- and each piece writes a split record (m, d,
// min, k raw candidates with global column indices + col0) instead of final
// outputs; k_topk_combine_cta merges the R records of a row.
template <int G, int BLOCK, int KC, int MODE, int U, int MINB, int NST = 0>
__global__ void __launch_bounds__(BLOCK, MINB)
    k_topk_rows(const float* __restrict__ x, long long ldx, long long rows, long long V, int k,
                float* __restrict__ vals, long long* __restrict__ idx, void* ws, int pf, int R = 0,
                long long chunk = 0, long long col0 = 0, char* __restrict__ rec = nullptr) {
  constexpr int NW = BLOCK / 32;
  constexpr int RPC = BLOCK / G;
  static_assert(NST <= 0 || G == 32, "the cp.async pipeline is per warp");
  __shared__ __align__(16) float4 pipe_buf[NST > 0 ? NW * NST * U * 32 : (NST == -2 ? NW * 3 * U * 32 : 1)];
  __shared__ __align__(8) uint64_t bulk_bar[NST == -2 ? NW * 3 : 1];  // per-warp bulk ring (NST = -2)
  __shared__ float smf[2 * NW];
  __shared__ double smd[NW];
  __shared__ float sv[NW * KC];
  __shared__ int si[NW * KC];
  __shared__ int tsh[2];  // CTA-shared admission bound, double-buffered by row parity
  __shared__ double exp2tab[MODE == kModeSafe ? 32 : 1];  // safe: exp_neg_d's table
  const int t = threadIdx.x % G;
  const long long nrow_groups = (rows + RPC - 1) / RPC;
  if (threadIdx.x == 0) tsh[0] = tsh[1] = Pass<KC, U, MODE, G>::f2o(kNegInf);
  if constexpr (MODE == kModeSafe) exp2_tab_init(exp2tab);
  if constexpr (NST == -2) {
    if (threadIdx.x == 0) {
      for (int b = 0; b < NW * 3; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(&bulk_bar[b])))
                     : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  long long bulk_g = 0;  // per-warp running chunk count of the bulk ring
  int it = 0;
  for (long long rg = blockIdx.x; rg < nrow_groups; rg += gridDim.x, ++it) {
    // slot it&1 serves this row; the other slot is reset for the next row
    // (every thread passed the previous row's final barrier before this).
    if (G == BLOCK && threadIdx.x == 0) tsh[(it + 1) & 1] = Pass<KC, U, MODE, G>::f2o(kNegInf);
    const long long row = rg * RPC + threadIdx.x / G;
    const bool live = row < rows;
    long long piece0 = 0;  // record mode: first column of this piece
    Seg s;
    if (rec) {
      const long long ir = live ? row / R : 0;
      piece0 = live ? (row % R) * chunk : 0;
      s = make_seg(x + ir * ldx + piece0, live ? std::min(chunk, V - piece0) : 0);
    } else {
      s = make_seg(x + (live ? row : 0) * ldx, live ? V : 0);
    }
    Pass<KC, U, MODE, G> P;
    P.L.init(k);
    P.kk = k;
    if (G == BLOCK) P.Tsh = &tsh[it & 1];
    bool bad = false;
    float outM = 0.0f;
    double outR = 1.0;
    if constexpr (MODE == kModeSafe) {
      float m = kNegInf, mn = -kNegInf;
      safe_max_min<G, U>(s, t, m, mn);
      float M, MN;
      if constexpr (G == 32) {
        M = group_max<32>(m);
        MN = group_min<32>(mn);
      } else {
        M = cta_max<NW>(m, smf);
        MN = cta_min<NW>(mn, smf);
      }
      double d = safe_sum<G, U>(s, t, M, exp2tab);
      if constexpr (G == 32)
        d = group_sum_d<32>(d);
      else
        d = cta_sum_d<NW>(d, smd);
      P.M = M;
      P.D = d;
      bad = !(d == d) || !isfinite(M) || !(MN == MN) || MN == kNegInf;
    }
    if constexpr (NST == -2 && MODE != kModeSafe) {  // per-warp bulk-copy ring, 3 stages
      const int wv = threadIdx.x >> 5;
      stream_seg_bulk<U, 3>(
          s, t, [&](float v, long long j) { P.scalar(v, (int)j, k); },
          [&](float4 (&v)[U], long long q0, int cnt) { P.batch(s, v, q0, cnt, k); }, pipe_buf + wv * 3 * U * 32,
          bulk_bar + wv * 3, bulk_g);
    } else if constexpr (NST == -1 && MODE != kModeSafe) {  // register double buffering
      stream_seg_db<G, U>(
          s, t, [&](float v, long long j) { P.scalar(v, (int)j, k); },
          [&](float4 (&v)[U], long long q0, int cnt) { P.batch(s, v, q0, cnt, k); });
    } else if constexpr (NST > 0 && MODE != kModeSafe) {
      stream_seg_pipe<U, NST>(
          s, t, [&](float v, long long j) { P.scalar(v, (int)j, k); },
          [&](float4 (&v)[U], long long q0, int cnt) { P.batch(s, v, q0, cnt, k); },
          pipe_buf + (threadIdx.x >> 5) * (NST * U * 32));
    } else {
      run_pass<G, U, KC, MODE>(P, s, t, k, pf);
    }
    RecHdr hdr{kNegInf, 0.0f, 0.0f, k};
    if constexpr (MODE == kModeFused) {
      MD tot;
      float MN;
      if constexpr (G == 32) {
        tot = md_group_reduce<32>(P.acc.finish());
        MN = group_min<32>(P.mn);
      } else {
        tot = md_cta_reduce<NW>(P.acc.finish(), smf);
        MN = cta_min<NW>(P.mn, smf);
      }
      outM = tot.m;
      outR = 1.0 / (double)tot.d;
      bad = !(tot.d == tot.d) || !isfinite(tot.m) || MN == kNegInf;
      hdr = RecHdr{tot.m, tot.d, MN, k};
    } else if constexpr (MODE == kModeTopkOf) {
      float c;
      if constexpr (G == 32)
        c = group_sum<32>(P.chk);
      else
        c = cta_sum<NW>(P.chk, smf);
      bad = !(c == c);
      hdr.mn = (c == c) ? 0.0f : c;
    }
    char* my = rec && live ? rec + (size_t)row * rec_bytes_(k) : nullptr;
    auto sink = [&](int r, float v, int i) {
      if (live && (int)(threadIdx.x & 31) == (r & 31)) {
        if (my) {
          reinterpret_cast<float*>(my + rec_vals_off())[r] = v;
          reinterpret_cast<long long*>(my + rec_idx_off(k))[r] = i < 0 ? -1LL : (long long)i + piece0 + col0;
          return;
        }
        float out = v;
        if constexpr (MODE == kModeFused) out = out_md(v, outM, outR);  // kernels.hpp:122
        vals[row * k + r] = out;
        idx[row * k + r] = (long long)i;
      }
    };
    if constexpr (G == 32) {
      P.L.normalize(k);
      group_merge<32>(P.L, k, sink);
    } else {
      cta_merge<NW>(P.L, k, sv, si, sink);
    }
    if (my) {
      if (t == 0) *reinterpret_cast<RecHdr*>(my) = hdr;  // non-finite rows: flagged by the combine
    } else if (live && bad && t == 0) {
      flag_bad_row(ws, row);
    }
  }
}

// --------------------------------------------------------- split part --
// grid (S, rows): CTA (c, row) reduces chunk c of the row into a record.
// col0 shifts the global index (V-split across GPUs).  For kModeSafe the
// row (M, 1/d) come from the softmax split records (srec, phase 0/1).
struct SRecView {
  float m;
  float mn;
  double d;
};
template <int BLOCK, int KC, int MODE, int U>
__global__ void __launch_bounds__(BLOCK)
    k_topk_split_part(const float* __restrict__ x, long long ldx, long long V, long long chunk,
                      int k, long long col0, char* __restrict__ rec, const SRecView* __restrict__ srec) {
  constexpr int NW = BLOCK / 32;
  __shared__ float smf[2 * NW];
  __shared__ double smd[NW];
  __shared__ float sv[NW * KC];
  __shared__ int si[NW * KC];
  const int S = gridDim.x;
  const long long row = blockIdx.y;
  const long long c0 = (long long)blockIdx.x * chunk;
  const long long n = std::min(chunk, V - c0);
  const Seg s = make_seg(x + row * ldx + c0, n);
  const int t = threadIdx.x;
  __shared__ int tsh;
  if (t == 0) tsh = Pass<KC, U, MODE, BLOCK>::f2o(kNegInf);
  __syncthreads();
  Pass<KC, U, MODE, BLOCK> P;
  P.L.init(k);
  P.kk = k;
  P.Tsh = &tsh;
  float safe_mn = 0.0f;
  if constexpr (MODE == kModeSafe) {
    const SRecView* rr = srec + row * S;
    float M = kNegInf, mn = -kNegInf;
    double d = 0.0;
    for (int i = t; i < S; i += BLOCK) {
      M = fmaxf(M, rr[i].m);
      mn = fminf(mn, rr[i].mn);
      if (rr[i].mn != rr[i].mn) mn = kNegInf;
      d += rr[i].d;
    }
    M = cta_max<NW>(M, smf);
    mn = cta_min<NW>(mn, smf);
    d = cta_sum_d<NW>(d, smd);
    P.M = M;
    P.D = d;
    // poison the record when the row holds a non-finite value
    if (!(d == d) || !isfinite(M) || mn == kNegInf) safe_mn = __int_as_float(0x7fffffff);
  }
  run_pass<BLOCK, U, KC, MODE>(P, s, t, k);
  RecHdr h{0.0f, 0.0f, 0.0f, k};
  if constexpr (MODE == kModeFused) {
    MD tot = md_cta_reduce<NW>(P.acc.finish(), smf);
    h.m = tot.m;
    h.d = tot.d;
    h.mn = cta_min<NW>(P.mn, smf);
  } else if constexpr (MODE == kModeTopkOf) {
    const float c = cta_sum<NW>(P.chk, smf);
    h.mn = (c == c) ? 0.0f : c;
    h.m = kNegInf;
  } else {
    h.m = kNegInf;
    h.mn = safe_mn;
  }
  char* my = rec + ((size_t)row * S + blockIdx.x) * rec_bytes_(k);
  float* rv = reinterpret_cast<float*>(my + rec_vals_off());
  long long* ri = reinterpret_cast<long long*>(my + rec_idx_off(k));
  const long long base = c0 + col0;
  cta_merge<NW>(P.L, k, sv, si, [&](int r, float v, int i) {
    if ((int)(threadIdx.x & 31) == (r & 31)) {
      rv[r] = v;
      ri[r] = i < 0 ? -1LL : (long long)i + base;
    }
  });
  if (t == 0) *reinterpret_cast<RecHdr*>(my) = h;
}

// ------------------------------------------------------------- combine --
// One warp per row merges n records (rank / chunk order).  Writes the
// merged record (out_rec, optional) and the final (vals, idx) (optional).
// mode: kModeFused outputs e^(u - M)/D; others output the values as is.
template <int KC>
__global__ void __launch_bounds__(32)
    k_topk_combine(const char* __restrict__ rec, int n, int k, int mode, char* __restrict__ out_rec,
                   float* __restrict__ vals, long long* __restrict__ idx, long long row_base,
                   void* ws) {
  pdl_wait();  // records come from the previous kernel
  const long long row = blockIdx.x;
  const int l = threadIdx.x;
  const size_t rb = rec_bytes_(k);
  const char* rr = rec + (size_t)row * n * rb;
  MD a = md_identity();
  float mn = -kNegInf;
  bool nan_seen = false;
  TopList<KC, long long> L;
  L.init(k);
  for (int c = l; c < n; c += 32) {
    // every field of the record is loaded before any is used (independent
    // loads in flight together instead of one L2 round trip per field)
    const char* my = rr + (size_t)c * rb;
    const RecHdr h = *reinterpret_cast<const RecHdr*>(my);
    const float* rv = reinterpret_cast<const float*>(my + rec_vals_off());
    const long long* ri = reinterpret_cast<const long long*>(my + rec_idx_off(k));
    float cv[KC];
    long long ci[KC];
#pragma unroll
    for (int r = 0; r < KC; ++r) {
      cv[r] = r < k ? rv[r] : kNegInf;
      ci[r] = r < k ? ri[r] : -1LL;
    }
    a = md_merge(a, MD{h.m, h.d});
    if (h.mn != h.mn) nan_seen = true;
    mn = fminf(mn, h.mn);
#pragma unroll
    for (int r = 0; r < KC; ++r)
      if (r < k) L.offer_ordered(cv[r], ci[r]);
  }
  a = md_group_reduce<32>(a);
  mn = group_min<32>(mn);
  nan_seen = __any_sync(0xffffffffu, nan_seen);
  bool bad;
  if (mode == kModeFused)
    bad = !(a.d == a.d) || !isfinite(a.m) || mn == kNegInf || nan_seen;
  else
    bad = nan_seen;
  const double R = 1.0 / (double)a.d;
  char* orec = out_rec ? out_rec + (size_t)row * rb : nullptr;
  L.normalize(k);
  group_merge<32>(L, k, [&](int r, float v, long long i) {
    if ((l & 31) == (r & 31)) {
      if (orec) {
        reinterpret_cast<float*>(orec + rec_vals_off())[r] = v;
        reinterpret_cast<long long*>(orec + rec_idx_off(k))[r] = i;
      }
      if (vals) {
        vals[row * k + r] = mode == kModeFused ? out_md(v, a.m, R) : v;
        idx[row * k + r] = i;
      }
    }
  });
  if (l == 0) {
    if (orec) *reinterpret_cast<RecHdr*>(orec) = RecHdr{a.m, a.d, nan_seen ? __int_as_float(0x7fffffff) : mn, k};
    if (bad && ws) flag_bad_row(ws, row_base + row);
  }
}

// CTA-wide combine of the n records of a row (NT threads; for rows split
// into many pieces): thread t merges records t, t+NT, ... (Eq. 4 merge and
// the (value desc, index asc) list), then the CTA reduces.  Same outputs as
// k_topk_combine.
//
// Two-level use: grid.y = G > 1 splits each row's records into G groups;
// CTA (row, g) merges its group into record g of the row in out_rec (no
// final outputs), and a second launch merges the G records.
// Each thread sees its records in increasing column order and each record
// in (value desc, index asc) order, so equal values reach a thread's list
// in increasing index order and the cheap strict-'>' insertion keeps the
// reference's tie order; the warp / CTA merges use the full order.
// The body of the CTA-wide combine, shared with the one-launch wide-row
// kernel (topk_wide.cu) and the TMA record kernels (topk_tma.cu), where the
// records come from other CTAs of the same launch: CG = true loads them
// L2-coherent (ld.global.cg) after the ticket.
template <int KC, int NT>
struct CombineSmem {
  float sm_m[NT / 32], sm_d[NT / 32], sm_mn[NT / 32], sm_nan[NT / 32];
  float sv[(NT / 32) * KC];
  long long si[(NT / 32) * KC];
};
template <bool CG, class T>
__device__ __forceinline__ T rec_ld(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// One record's candidates as a left-aligned list (a record is sorted under
// (value desc, index asc); slots past k hold (-inf, -1)).
template <bool CG, int KC>
__device__ __forceinline__ void rec_list(const char* my, int k, TopList<KC, long long>& L) {
  const float* rv = reinterpret_cast<const float*>(my + rec_vals_off());
  const long long* ri = reinterpret_cast<const long long*>(my + rec_idx_off(k));
#pragma unroll
  for (int r = 0; r < KC; ++r) {
    L.v[r] = r < k ? rec_ld<CG>(rv + r) : kNegInf;
    L.i[r] = r < k ? rec_ld<CG>(ri + r) : -1LL;
  }
}
// k rounds of a warp arg-max where every lane holds TWO sorted lists: the
// lane's candidate is the better of the two heads, and the winning lane
// pops the list it came from -- the 2-way merge of each lane's lists is
// folded into the warp merge, so a lane never builds a merged list.
template <int KC, class Sink>
__device__ __forceinline__ void group_merge2(TopList<KC, long long>& A, TopList<KC, long long>& B, int k,
                                             Sink&& sink) {
  const int lane = (int)(threadIdx.x & 31u);
  for (int r = 0; r < k; ++r) {
    const bool useB = TopList<KC, long long>::before_(B.v[0], B.i[0], A.v[0], A.i[0]);
    const float hv = useB ? B.v[0] : A.v[0];
    const long long hi = useB ? B.i[0] : A.i[0];
    const int kv = ord_key(hv);
    const int mx = __reduce_max_sync(0xffffffffu, kv);
    const bool top = kv == mx;
    const unsigned long long u = top ? static_cast<unsigned long long>(hi) : ~0ull;
    const unsigned h = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(u >> 32));
    const unsigned lo =
        __reduce_min_sync(0xffffffffu, static_cast<unsigned>(u >> 32) == h ? static_cast<unsigned>(u) : 0xffffffffu);
    const unsigned long long wv = (static_cast<unsigned long long>(h) << 32) | lo;
    const int bl = __ffs(__ballot_sync(0xffffffffu, top && u == wv)) - 1;
    const float bv = __shfl_sync(0xffffffffu, hv, bl);
    if (lane == bl) {
      if (useB) B.pop();
      else A.pop();
    }
    sink(r, bv, static_cast<long long>(wv));
  }
}
// rr: the row's n records.  orec (optional) receives the merged record;
// vals/idx (optional) the row's final k outputs; a bad row is flagged as
// bad_row in ws when `flag`.  Threads 0..NT-1 take part; `sync` is their
// barrier (__syncthreads, or a named barrier when other warps of the CTA
// have exited).
//
// Latency-bound (one CTA at the end of a launch), so the critical path is
// kept short: thread t loads records t and t + NT together (one L2 round
// trip) as two sorted lists, merges their (m, d) (Eq. 4), and the warp
// merge takes the better head of the two per round (group_merge2); records
// past 2 * NT (rare) are inserted into the second list under the full
// order.  Warp winners go through shared memory to warp 0, whose lanes hold
// one warp's sorted list each.  Every merge level uses (value desc, index
// asc), so any record order gives the reference's selection (COLS: the
// records happen to be in column order -- kept for the callers' clarity).
template <int KC, int NT, bool CG, class Sync = CtaSync, bool COLS = true>
__device__ __forceinline__ void combine_records_cta(const char* __restrict__ rr, int n, int k, int mode,
                                                    char* __restrict__ orec, float* __restrict__ vals,
                                                    long long* __restrict__ idx, void* ws, long long bad_row,
                                                    bool flag, CombineSmem<KC, NT>& sm, Sync sync = Sync()) {
  constexpr int NW = NT / 32;
  static_assert(NW <= 32, "warp 0 merges one list per warp");
  const int t = threadIdx.x, l = t & 31, w = t >> 5;
  const size_t rb = rec_bytes_(k);
  TopList<KC, long long> A, B;
  A.init_empty();
  B.init_empty();
  float4 h0 = make_float4(kNegInf, 0.0f, -kNegInf, 0.0f), h1 = h0;  // (m, d, min, -) identities
  if (t < n) {
    h0 = rec_ld<CG>(reinterpret_cast<const float4*>(rr + (size_t)t * rb));
    rec_list<CG>(rr + (size_t)t * rb, k, A);
  }
  if (t + NT < n) {
    h1 = rec_ld<CG>(reinterpret_cast<const float4*>(rr + (size_t)(t + NT) * rb));
    rec_list<CG>(rr + (size_t)(t + NT) * rb, k, B);
  }
  OSMX_STAMP(0);
  MD a = md_merge(MD{h0.x, h0.y}, MD{h1.x, h1.y});
  float mn = fminf(h0.z, h1.z);
  float nan_seen = (h0.z != h0.z || h1.z != h1.z) ? 1.0f : 0.0f;
  for (int c = t + 2 * NT; c < n; c += NT) {
    const float4 hv = rec_ld<CG>(reinterpret_cast<const float4*>(rr + (size_t)c * rb));
    TopList<KC, long long> C;
    rec_list<CG>(rr + (size_t)c * rb, k, C);
    a = md_merge(a, MD{hv.x, hv.y});
    if (hv.z != hv.z) nan_seen = 1.0f;
    mn = fminf(mn, hv.z);
#pragma unroll
    for (int r = 0; r < KC; ++r)
      if (r < k) B.offer_ordered(C.v[r], C.i[r]);
  }
  // one round of CTA reductions: (m, d), min and the NaN count together
  a = md_group_reduce<32>(a);
  mn = group_min<32>(mn);
  nan_seen = group_sum<32>(nan_seen);
  OSMX_STAMP(1);
  group_merge2(A, B, k, [&](int r, float v, long long i) {
    if (l == 0) {
      sm.sv[w * KC + r] = v;
      sm.si[w * KC + r] = i;
    }
  });
  if (l == 0) {
    sm.sm_m[w] = a.m;
    sm.sm_d[w] = a.d;
    sm.sm_mn[w] = mn;
    sm.sm_nan[w] = nan_seen;
  }
  OSMX_STAMP(2);
  sync();
  OSMX_STAMP(3);
  if (w == 0) {
    a = l < NW ? MD{sm.sm_m[l], sm.sm_d[l]} : md_identity();
    mn = l < NW ? sm.sm_mn[l] : -kNegInf;
    nan_seen = l < NW ? sm.sm_nan[l] : 0.0f;
    a = md_group_reduce<32>(a);
    mn = group_min<32>(mn);
    nan_seen = group_sum<32>(nan_seen);
    bool bad;
    if (mode == kModeFused)
      bad = !(a.d == a.d) || !isfinite(a.m) || mn == kNegInf || nan_seen > 0.0f;
    else
      bad = nan_seen > 0.0f;
    OSMX_STAMP(7);
    const double R = 1.0 / (double)a.d;
    TopList<KC, long long> M;
    M.init_empty();
    if (l < NW) {
#pragma unroll
      for (int r = 0; r < KC; ++r)
        if (r < k) {
          M.v[r] = sm.sv[l * KC + r];
          M.i[r] = sm.si[l * KC + r];
        }
    }
    OSMX_STAMP(8);
    group_merge<32>(M, k, [&](int r, float v, long long i) {
      if (l == (r & 31)) {
        if (orec) {
          reinterpret_cast<float*>(orec + rec_vals_off())[r] = v;
          reinterpret_cast<long long*>(orec + rec_idx_off(k))[r] = i;
        }
        if (vals) {
          vals[r] = mode == kModeFused ? out_md(v, a.m, R) : v;
          idx[r] = i;
        }
      }
    });
    if (l == 0) {
      if (orec) *reinterpret_cast<RecHdr*>(orec) = RecHdr{a.m, a.d, nan_seen > 0.0f ? __int_as_float(0x7fffffff) : mn, k};
      if (flag && bad && ws) flag_bad_row(ws, bad_row);
    }
    OSMX_STAMP(4);
  }
  sync();  // the scratch may be reused by the caller
}

template <int KC, int NT>
__global__ void __launch_bounds__(NT)
    k_topk_combine_cta(const char* __restrict__ rec, int n, int k, int mode, char* __restrict__ out_rec,
                       float* __restrict__ vals, long long* __restrict__ idx, long long row_base, void* ws) {
  __shared__ CombineSmem<KC, NT> sm;
  pdl_wait();  // records come from the previous kernel
  const long long row = blockIdx.x;
  const int G = gridDim.y, g = blockIdx.y;
  const int per = (n + G - 1) / G;
  const int c0 = g * per, c1 = min(n, c0 + per);
  const char* rr = rec + ((size_t)row * n + c0) * rec_bytes_(k);
  char* orec = out_rec ? out_rec + ((size_t)row * G + g) * rec_bytes_(k) : nullptr;
  const bool last = G == 1;  // first level of two: records only
  combine_records_cta<KC, NT, false>(rr, c1 > c0 ? c1 - c0 : 0, k, mode, orec, last && vals ? vals + row * k : nullptr,
                                     last && vals ? idx + row * k : nullptr, ws, row_base + row, last, sm);
}

// ------------------------------------------------------------ launchers --

// Threads per row: enough rows in flight to fill every SM several times,
// as few threads per row as that allows (the per-row epilogue -- (m,d)
// reduce and k-round merge -- is paid once per row, and small CTAs let
// other CTAs on the SM keep streaming while one merges).
inline int topk_row_threads(long long rows, long long V) {
  const int forced = osmx_host::tuning().topk_threads;
  if (forced) return forced;
  const long long sms = osmx_host::num_sms();
  // measured on B200 (profiles/): warp-per-row reads C4 at 7.1 TB/s vs 6.5
  // (128 threads) and 5.9 (256); it wins down to ~4000 rows.
  // 4000 rows: warp/row 4.7-7.0 TB/s vs 3.5-6.5 (128 thr); 1000 rows: 128 thr
  // 2.9-4.8 TB/s vs 1.6-2.3 (warp/row) -- tools/shape_sweep.py, cold L2.
  // (Those early rejections of deeper per-warp pipelining were for many-row
  // launches; for one wave of rows the register double-buffered variant is
  // the default, see run_rows.)
  // 1184..1775 rows: warp per row (double-buffered) up to V = 64K (1600 x
  // 32K: 0.058 vs 0.068 ms), a 256-thread CTA per row above (1600 x 1M:
  // 1.00 vs 1.18 ms for 128 threads); fewer rows: 128-thread CTAs.
  if (V <= 2048 || rows >= 12 * sms) return 32;
  if (rows >= 8 * sms) return V <= 65536 ? 32 : 256;
  if (rows >= 2 * sms) return 128;
  return 256;
}

template <int KC, int MODE>
cudaError_t run_rows(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                     long long* idx, void* ws, cudaStream_t st) {
  const int g = topk_row_threads(rows, V);
  // Bulk L2 prefetch one batch ahead (auto, rows >= ~2 waves of warps):
  // +1.4-5% at 16384-65536 rows (C4: 7.19 -> 7.29-7.39 TB/s, 98-99% of a
  // pure-read probe's 7.43, tools/read_peak.cu); -1..-6% at 4000 rows.
  int pf = osmx_host::tuning().l2_prefetch;
  if (pf < 0) pf = (g == 32 && V >= 32768 && rows >= 32LL * osmx_host::num_sms() * 2) ? 1 : 0;
  int u8 = osmx_host::tuning().topk_u8;
  // measured (tools/shape_sweep.py, 4000 rows): +8-9% at V = 16K-32K, +1% at
  // 64K, -2% at 128K (rows long enough to amortise the serial load->compute).
  if (u8 < 0) u8 = (g == 32 && V >= 8192 && V <= 65536 && rows <= 28LL * osmx_host::num_sms()) ? 1 : 0;
  int pipe = V < (1LL << 33) ? osmx_host::tuning().topk_pipe : 0;  // 32-bit float4 counts
  // One wave of rows with V >= 16K: register double buffering (2 x 4 float4s
  // per lane, loads of batch i+1 in flight while batch i is processed):
  // 4000 rows: +0.4% (32K), +6% (64K), +1.3% (128K) over the U = 8 variant.
  if (pipe == 0 && osmx_host::tuning().topk_pipe == 0 && g == 32 && V >= 16384 &&
      rows <= 28LL * osmx_host::num_sms() && osmx_host::tuning().topk_u8 < 0 && osmx_host::tuning().topk_threads == 0)
    pipe = 4;
  if (g == 32 && pipe > 0) {
    // per-warp cp.async pipeline: 4-warp CTAs, U float4s x NST stages per lane
    const long long grid = std::min<long long>((rows + 3) / 4, 1LL << 30);
    if (pipe == 6)  // per-warp bulk-copy ring: 3 x 2 KB chunks in flight per warp
      k_topk_rows<32, 128, KC, MODE, 4, 7, -2><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (pipe == 4 && osmx_host::tuning().topk_block != 128)
      // one warp per CTA: the one wave of rows spreads over the SMs one warp
      // at a time (27-28 per SM at 4000 rows) instead of in 4-warp CTAs
      // (6 or 7 per SM: 24 vs 28 warps, the 24-warp SMs idle at the end).
      // B200, 4000 rows (tools/runs/r2_i.sh): 16K -4.3%, 32K -1.2%, 64K
      // -0.8%, 128K -0.4% time vs 4-warp CTAs.
      k_topk_rows<32, 32, KC, MODE, 4, 28, -1><<<(unsigned)std::min<long long>(rows, 1LL << 30), 32, 0, st>>>(
          x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (pipe == 4)  // register double buffering, 2 x 4 float4s per lane
      k_topk_rows<32, 128, KC, MODE, 4, 7, -1><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (pipe == 5)  // register double buffering, 2 x 2 float4s per lane
      k_topk_rows<32, 128, KC, MODE, 2, 8, -1><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (pipe == 1)
      k_topk_rows<32, 128, KC, MODE, 4, 8, 3><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (pipe == 2)
      k_topk_rows<32, 128, KC, MODE, 2, 8, 4><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else
      k_topk_rows<32, 128, KC, MODE, 4, 7, 2><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
  } else if (g == 32 && u8) {
    pf = osmx_host::tuning().l2_prefetch > 0 ? pf : 0;
    // One wave of rows (<= 28 warps per SM): occupancy is set by the row
    // count, not by registers, so each lane keeps 8 float4s in flight
    // (4-warp CTAs, <= 72 registers: 7 CTAs = 28 warps per SM).
    const long long grid = std::min<long long>((rows + 3) / 4, 1LL << 30);
    k_topk_rows<32, 128, KC, MODE, 8, 7><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
  } else if (g == 32) {
    constexpr int RPC = 256 / 32;
    const long long groups = (rows + RPC - 1) / RPC;
    const long long grid = std::min<long long>(groups, 1LL << 30);
    if (V <= 2048)
      k_topk_rows<32, 256, KC, MODE, 2, 4><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else
      k_topk_rows<32, 256, KC, MODE, 4, 4><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
  } else {
    const long long grid = std::min<long long>(rows, 1LL << 30);
    if (g == 128)
      k_topk_rows<128, 128, KC, MODE, 4, 8><<<(unsigned)grid, 128, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else if (g == 512)
      k_topk_rows<512, 512, KC, MODE, 4, 2><<<(unsigned)grid, 512, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
    else
      k_topk_rows<256, 256, KC, MODE, 4, 4><<<(unsigned)grid, 256, 0, st>>>(x, ldx, rows, V, k, vals, idx, ws, pf);
  }
  osmx_host::count_launch();
  return cudaGetLastError();
}

constexpr int kSplitBlock = 512;
constexpr int kSplitU = 4;

long long topk_split_chunk(long long rows, long long V) {
  long long ch = osmx_host::tuning().split_chunk;
  if (ch <= 0) {
    const long long target = 4LL * osmx_host::num_sms();
    long long per_row = std::max<long long>(1, target / std::max<long long>(rows, 1));
    ch = (V + per_row - 1) / per_row;
    ch = std::max<long long>(ch, 32768);
  }
  return (ch + 15) / 16 * 16;
}

// Piece length of the warp-per-piece split path: about one wave of warps
// (28 per SM) over the whole problem, 8K..64K elements, a multiple of 16.
long long topk_piece_chunk(long long rows, long long V) {
  long long ch = osmx_host::tuning().split_chunk;
  if (ch <= 0) {
    const long long waves = 28LL * osmx_host::num_sms();
    ch = (rows * V + waves - 1) / waves;
    ch = std::min<long long>(std::max<long long>(ch, 8192), 65536);
  }
  return (ch + 15) / 16 * 16;
}

// Piece length of the TMA-ring split path: floor(slots / rows) pieces per
// row, so that rows x pieces never exceeds the resident CTAs (one wave), at
// least 16K elements each, a multiple of 16.
long long topk_tma_piece_chunk(long long rows, long long V, int k) {
  long long ch = osmx_host::tuning().split_chunk;
  if (ch <= 0) {
    const long long per_row = std::max<long long>(1, osmx_host::topk_tma_slots(k) / std::max<long long>(rows, 1));
    ch = (V + per_row - 1) / per_row;
    ch = std::max<long long>((ch + 15) / 16 * 16, 16384);
  }
  return (ch + 15) / 16 * 16;
}

// The one-launch wide-row kernel: ticket counters for <= kWsMaxTickets rows,
// 32-bit in-row element indices.
bool topk_wide_ok(long long rows, long long V) { return rows <= kWsMaxTickets && V < (1LL << 31) - 4096; }

template <int KC, int MODE>
cudaError_t run_split(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                      long long* idx, void* ws, cudaStream_t st, long long col0, char* out_rec) {
  const long long ch = topk_split_chunk(rows, V);
  const long long S = (V + ch - 1) / ch;
  char* base = static_cast<char*>(ws) + kWsHeader;
  char* rec = base;
  const SRecView* srec = nullptr;
  if constexpr (MODE == kModeSafe) {
    // Row max / normalizer from the softmax split phases.
    srec = reinterpret_cast<const SRecView*>(base);
    rec = base + ((size_t)(rows * S) * sizeof(SRecView) + 255) / 256 * 256;
    cudaError_t e = osmx_host::launch_safe_split_stats(x, ldx, rows, V, ch, const_cast<SRecView*>(srec), st);
    if (e != cudaSuccess) return e;
  }
  if constexpr (MODE != kModeSafe) {
    int how = osmx_host::tuning().split_cta;
    // TMA-ring pieces (one wave of CTAs, floor(slots / rows) pieces per row)
    // except for many short rows (B200, tools/runs/g44.sh, g45.sh; ms, TMA
    // vs warp pieces): 1 x 2^26 0.062 vs 0.067, 8 x 1M 0.026 vs 0.029,
    // 64 x 1M 0.062 vs 0.068, 400 x 1M 0.270 vs 0.314; but 128 x 256K 0.045
    // vs 0.038.
    // One row (configs[4], the V-split slices): the TMA ring over dynamically
    // claimed chunks, combine fused in the last CTA -- 1 x 2^26: 0.0521 ms
    // vs 0.0558 for static pieces + a combine launch (tools/runs/r2_s.sh).
    if (how < 0) how = rows == 1 ? 4 : (rows >= 64 && rows * V <= (1LL << 25)) ? 0 : 2;
    if (how == 4) {
      if (rows == 1 && topk_wide_ok(rows, V))
        return osmx_host::launch_topk_tma_dyn(MODE, x, V, k, vals, idx, ws, st, col0, rec, out_rec);
      how = 2;  // several rows, or 32-bit element indices overflow: static TMA pieces
    }
    if (how == 3 && topk_wide_ok(rows, V))
      return osmx_host::launch_topk_wide(MODE, x, ldx, rows, V, k, vals, idx, ws, st, col0, out_rec);
    if (how == 2) {
      // One TMA-ring CTA per piece: about one piece per resident CTA over the
      // whole problem, then one CTA-wide combine per row.
      const long long pc = topk_tma_piece_chunk(rows, V, k);
      const long long R = (V + pc - 1) / pc;
      if (rows <= kWsMaxTickets && osmx_host::tuning().split_fuse == 1)  // combine fused (ticket)
        return osmx_host::launch_topk_tma_records(MODE, x, ldx, rows * R, V, k, ws, st, (int)R, pc, col0, rec, vals,
                                                  idx, out_rec);
      cudaError_t e = osmx_host::launch_topk_tma_records(MODE, x, ldx, rows * R, V, k, ws, st, (int)R, pc, col0, rec);
      if (e != cudaSuccess) return e;
      if (R >= 64)
        launch_pdl(k_topk_combine_cta<KC, 256>, dim3((unsigned)rows), dim3(256), 0, st, (const char*)rec, (int)R, k,
                   (int)MODE, out_rec, vals, idx, 0LL, ws);
      else
        launch_pdl(k_topk_combine<KC>, dim3((unsigned)rows), dim3(32), 0, st, (const char*)rec, (int)R, k, (int)MODE,
                   out_rec, vals, idx, 0LL, ws);
      osmx_host::count_launch();
      return cudaGetLastError();
    }
    if (how == 0) {
      // Warp-per-piece records (the warp-per-row kernel in record mode: one
      // ~16K-element piece per warp, about one wave of warps over the whole
      // problem), then a CTA-wide combine per row.
      const long long pc = topk_piece_chunk(rows, V);
      const long long R = (V + pc - 1) / pc;
      const long long pieces = rows * R;
      if (pieces <= 28LL * osmx_host::num_sms() && pc >= 8192) {
        const long long grid = (pieces + 3) / 4;
        if (osmx_host::tuning().topk_pipe == 0)  // one wave: register double buffering
          k_topk_rows<32, 128, KC, MODE, 4, 7, -1><<<(unsigned)grid, 128, 0, st>>>(x, ldx, pieces, V, k, nullptr,
                                                                                nullptr, ws, 0, (int)R, pc, col0, rec);
        else
          k_topk_rows<32, 128, KC, MODE, 8, 7><<<(unsigned)grid, 128, 0, st>>>(x, ldx, pieces, V, k, nullptr, nullptr,
                                                                            ws, 0, (int)R, pc, col0, rec);
      } else {
        const long long grid = std::min<long long>((pieces + 7) / 8, 1LL << 30);
        k_topk_rows<32, 256, KC, MODE, 4, 4><<<(unsigned)grid, 256, 0, st>>>(x, ldx, pieces, V, k, nullptr, nullptr,
                                                                          ws, 0, (int)R, pc, col0, rec);
      }
      osmx_host::count_launch();
      if (R >= 1024) {
        // two levels: G groups of <= 256 records per row, then the G records
        const int G = (int)((R + 255) / 256);
        char* mid = rec + (size_t)(rows * R) * rec_bytes_(k);
        launch_pdl(k_topk_combine_cta<KC, 256>, dim3((unsigned)rows, (unsigned)G), dim3(256), 0, st,
                   (const char*)rec, (int)R, k, (int)MODE, mid, (float*)nullptr, (long long*)nullptr, 0LL, ws);
        if (G <= 64)  // one warp: no cross-warp merge on the last, tiny level
          launch_pdl(k_topk_combine<KC>, dim3((unsigned)rows), dim3(32), 0, st, (const char*)mid, G, k, (int)MODE,
                     out_rec, vals, idx, 0LL, ws);
        else
          launch_pdl(k_topk_combine_cta<KC, 256>, dim3((unsigned)rows), dim3(256), 0, st, (const char*)mid, G, k,
                     (int)MODE, out_rec, vals, idx, 0LL, ws);
        osmx_host::count_launch();
      } else if (R >= 64) {
        launch_pdl(k_topk_combine_cta<KC, 256>, dim3((unsigned)rows), dim3(256), 0, st, (const char*)rec, (int)R, k,
                   (int)MODE, out_rec, vals, idx, 0LL, ws);
      } else
        launch_pdl(k_topk_combine<KC>, dim3((unsigned)rows), dim3(32), 0, st, (const char*)rec, (int)R, k, (int)MODE,
                   out_rec, vals, idx, 0LL, ws);
      osmx_host::count_launch();
      return cudaGetLastError();
    }
  }
  dim3 grid((unsigned)S, (unsigned)rows);
  k_topk_split_part<kSplitBlock, KC, MODE, kSplitU><<<grid, kSplitBlock, 0, st>>>(x, ldx, V, ch, k, col0, rec, srec);
  osmx_host::count_launch();
  k_topk_combine<KC><<<(unsigned)rows, 32, 0, st>>>(rec, (int)S, k, MODE, out_rec, vals, idx, 0, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_mode(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                          long long* idx, void* ws, cudaStream_t st, bool split, long long col0,
                          char* out_rec) {
#define OSMX_KC_CASE(KC)                                                               \
  if (split) return run_split<KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, col0, out_rec); \
  return run_rows<KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st);
  if (k <= 1) { OSMX_KC_CASE(1) }
  if (k <= 5) { OSMX_KC_CASE(5) }
  if (k <= 8) { OSMX_KC_CASE(8) }
  if (k <= 16) { OSMX_KC_CASE(16) }
  { OSMX_KC_CASE(32) }
#undef OSMX_KC_CASE
}

bool topk_uses_split(long long rows, long long V) {
  const auto& tn = osmx_host::tuning();
  if (tn.shape == osmx_host::kShapeSplit) return true;
  if (tn.shape != osmx_host::kShapeAuto) return false;
  // split records (TMA pieces) beat the row kernels up to ~5 rows per SM
  // (tools/runs/g46.sh, g47.sh; ms, split vs rows: 444 x 1M 0.30 vs 0.48,
  // 700 x 1M 0.46 vs 0.54, 444 x 128K 0.054 vs 0.080), not at 1000 rows
  // (1M: 0.69 vs 0.64; 128K: 0.12 vs 0.10)
  return V > 65536 && rows < 5LL * osmx_host::num_sms();
}

template <int KC>
cudaError_t combine_kc(const void* records, int n, int k, void* out_record, float* vals,
                       long long* idx, void* ws, cudaStream_t st) {
  k_topk_combine<KC><<<1, 32, 0, st>>>(static_cast<const char*>(records), n, k,
                                       kModeFused,
                                       static_cast<char*>(out_record), vals, idx, 0, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

}  // namespace
