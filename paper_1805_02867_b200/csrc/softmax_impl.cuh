// softmax_impl.cuh -- batched naive / safe / online softmax for sm_100a.
//
// Replaces the reference's single-row kernel templates
//   naive_softmax_kernel   kernels.hpp:39-46   (Alg. 1)
//   safe_softmax_kernel    kernels.hpp:49-58   (Alg. 2, 3 passes, 4 accesses)
//   online_softmax_kernel  kernels.hpp:61-69   (Alg. 3, 2 passes, 3 accesses)
// and the chunked normalizer run_normalizer_chunked (normalizer.hpp:73-85)
// as the split-row combine.  Three kernel families (launch layer picks):
//
//   resident : a group of TPR threads owns one row and keeps it in
//              registers; the second (and third) pass of the algorithm
//              re-reads registers, so DRAM sees 1 read + 1 write.
//   stream   : one CTA per row, every pass streams global memory (the
//              paper's one-threadblock-per-vector design).
//   split    : the row is cut into S contiguous chunks, one CTA each; per
//              chunk records (m, d, min) are merged with the reference's
//              merge() and the scale pass runs per chunk.
//
// Numerics (SURVEY.md sec.7 risk 3): m is exact (a max), d accumulates in
// fp32 from ex2.approx terms against the running max (naive: fp64 sum, like
// the reference), outputs use the accurate expf and one IEEE reciprocal of
// d per row.  No fast-math, no FTZ on outputs.
#pragma once
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"
#include "softmax_staged.cuh"
#include "stream.cuh"

using namespace osmx_dev;

namespace {

// ----------------------------------------------------- group reductions --
// A group is TPR consecutive threads of a BLOCK-thread CTA (TPR <= 32: a
// sub-warp; TPR > 32: W = TPR/32 whole warps).  All threads of the CTA must
// call these together (they contain __syncthreads when TPR > 32).
template <int TPR, int BLOCK>
struct Grp {
  static constexpr int NW = BLOCK / 32;
  static constexpr int W = TPR / 32;

  template <class T, class Op>
  __device__ static T reduce(T v, Op op, T* sm) {
    if constexpr (TPR <= 32) {
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
      return v;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
      const int w = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) sm[w] = v;
      __syncthreads();
      const int g0 = (w / W) * W;
      T t = sm[g0];
#pragma unroll
      for (int i = 1; i < W; ++i) t = op(t, sm[g0 + i]);
      __syncthreads();
      return t;
    }
  }
  __device__ static MD md(MD s, float* sm) {
    if constexpr (TPR <= 32) {
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) {
        MD t{__shfl_xor_sync(0xffffffffu, s.m, o), __shfl_xor_sync(0xffffffffu, s.d, o)};
        s = md_merge(s, t);
      }
      return s;
    } else {
      s = md_group_reduce<32>(s);
      const int w = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) {
        sm[w] = s.m;
        sm[NW + w] = s.d;
      }
      __syncthreads();
      const int g0 = (w / W) * W;
      MD t{sm[g0], sm[NW + g0]};
#pragma unroll
      for (int i = 1; i < W; ++i) t = md_merge(t, MD{sm[g0 + i], sm[NW + g0 + i]});
      __syncthreads();
      return t;
    }
  }
};

struct OpMax {
  __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};
struct OpSum {
  __device__ float operator()(float a, float b) const { return a + b; }
};
struct OpSumD {
  __device__ double operator()(double a, double b) const { return a + b; }
};

__device__ __forceinline__ float nanf_() { return __int_as_float(0x7fffffff); }

// ------------------------------------------------------------- resident --
// EPT elements per thread (VEC: EPT/4 float4s).  Rows per CTA = BLOCK/TPR.
template <int TPR, int EPT, bool VEC, int ALG>
__global__ void __launch_bounds__(TPR > 256 ? TPR : 256)
    k_softmax_resident(const float* __restrict__ x, long long ldx, float* __restrict__ y,
                       long long ldy, long long rows, int V, void* ws) {
  constexpr int BLOCK = TPR > 256 ? TPR : 256;
  constexpr int RPC = BLOCK / TPR;
  using G = Grp<TPR, BLOCK>;
  __shared__ float smf[2 * (BLOCK / 32)];
  __shared__ double smd[BLOCK / 32];

  const int g = threadIdx.x % TPR;
  const long long row = (long long)blockIdx.x * RPC + threadIdx.x / TPR;
  const bool live = row < rows;
  const float* xr = x + (live ? row : 0) * ldx;
  float* yr = y + (live ? row : 0) * ldy;

  float a[EPT];
  bool bad = false;
  if constexpr (VEC) {
#pragma unroll
    for (int t = 0; t < EPT / 4; ++t) {
      const int q = g + TPR * t;
      float4 v = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      if (live && 4 * q < V) {
        v = ld_f4(xr + 4 * q);
        bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      }
      a[4 * t] = v.x;
      a[4 * t + 1] = v.y;
      a[4 * t + 2] = v.z;
      a[4 * t + 3] = v.w;
    }
  } else {
    // Rows not 16-byte aligned (V % 4 != 0 or an odd ld / base): float4 q
    // of the aligned base xr - phase holds elements 4q - phase .. 4q + 3 -
    // phase; interior float4s load with LDG.128, the <= 2 edge ones
    // element-wise (only in-row addresses are touched).
    const int phase = (int)((reinterpret_cast<uintptr_t>(xr) >> 2) & 3);
    const float* xb = xr - phase;
#pragma unroll
    for (int t = 0; t < EPT / 4; ++t) {
      const int q = g + TPR * t;
      const int e0 = 4 * q - phase;
      float4 v = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      if (live && e0 < V) {
        if (e0 >= 0 && e0 + 4 <= V) {
          v = ld_f4(xb + 4 * q);
        } else {
          if (e0 + 0 >= 0 && e0 + 0 < V) v.x = ld_f1(xr + e0 + 0);
          if (e0 + 1 >= 0 && e0 + 1 < V) v.y = ld_f1(xr + e0 + 1);
          if (e0 + 2 >= 0 && e0 + 2 < V) v.z = ld_f1(xr + e0 + 2);
          if (e0 + 3 >= 0 && e0 + 3 < V) v.w = ld_f1(xr + e0 + 3);
        }
        // masked lanes hold -inf (never "bad": -inf elements are detected below only if in-row)
        const bool in0 = e0 + 0 >= 0 && e0 + 0 < V, in1 = e0 + 1 >= 0 && e0 + 1 < V;
        const bool in2 = e0 + 2 >= 0 && e0 + 2 < V, in3 = e0 + 3 >= 0 && e0 + 3 < V;
        bad |= (in0 && !isfinite(v.x)) || (in1 && !isfinite(v.y)) || (in2 && !isfinite(v.z)) ||
               (in3 && !isfinite(v.w));
      }
      a[4 * t] = v.x;
      a[4 * t + 1] = v.y;
      a[4 * t + 2] = v.z;
      a[4 * t + 3] = v.w;
    }
  }

  // Returns (m, scale) such that y = f(x) * scale.
  float m = 0.0f, r = 0.0f;
  double rd = 0.0;
  Recip rc{0.0f, 0.0f};  // safe / online: 1/d as hi + lo
  bool row_bad = false;
  if constexpr (ALG == osmx_host::kOnline) {
    // Alg. 3 lines 1-6 on the thread's elements (max first, then one
    // rescale-free sum), then the group-wide merge (Eq. 4).
    float lm = kNegInf;
#pragma unroll
    for (int t = 0; t < EPT; ++t) lm = fmaxf(lm, a[t]);
    L2Acc acc;
    acc.raise(lm);
    if (lm != kNegInf) {
#pragma unroll
      for (int t = 0; t < EPT; ++t) acc.d += acc.term(a[t]);
    }
    MD s0 = acc.finish();
    if (bad) s0.d = nanf_();
    MD s = G::md(s0, smf);
    m = s.m;
    rc = recip_of((double)s.d);
    row_bad = !(s.d == s.d) || !isfinite(m);
  } else if constexpr (ALG == osmx_host::kSafe) {
    float lm = kNegInf;
#pragma unroll
    for (int t = 0; t < EPT; ++t) lm = fmaxf(lm, a[t]);
    m = G::reduce(lm, OpMax(), smf);
    SafeAcc acc;
    acc.raise(m);
#pragma unroll
    for (int t = 0; t < EPT; ++t) acc.d += acc.term(a[t]);
    double ld = (m == kNegInf) ? 0.0 : acc.d;
    if (bad) ld = (double)nanf_();
    const double d = G::reduce(ld, OpSumD(), smd);
    rc = recip_of(d);
    row_bad = !(d == d) || !isfinite(m);
  } else {  // naive: d = sum double(expf(x)), no max shift (kernels.hpp:43-45)
    double ld = 0.0;
#pragma unroll
    for (int t = 0; t < EPT; ++t) ld += (double)expf(a[t]);
    if (bad) ld = (double)nanf_();
    const double d = G::reduce(ld, OpSumD(), smd);
    rd = 1.0 / d;
    row_bad = !(d == d);
  }
  if (!live) return;
  if (row_bad) {
    if (g == 0) flag_bad_row(ws, row);
  }
  auto f = [&](float v) -> float {
    if constexpr (ALG == osmx_host::kNaive)
      return (float)((double)expf(v) * rd);
    else
      return out_soft<ALG == osmx_host::kSafe>(v, m, rc);
  };
  if constexpr (VEC) {
#pragma unroll
    for (int t = 0; t < EPT / 4; ++t) {
      const int q = g + TPR * t;
      if (4 * q < V)
        st_f4(yr + 4 * q, make_float4(f(a[4 * t]), f(a[4 * t + 1]), f(a[4 * t + 2]), f(a[4 * t + 3])));
    }
  } else {
    const int phase = (int)((reinterpret_cast<uintptr_t>(xr) >> 2) & 3);
    const bool same = ((reinterpret_cast<uintptr_t>(yr) >> 2) & 3) == (uintptr_t)phase;
    float* yb = yr - phase;
#pragma unroll
    for (int t = 0; t < EPT / 4; ++t) {
      const int q = g + TPR * t;
      const int e0 = 4 * q - phase;
      if (e0 >= V) continue;
      const float4 o = make_float4(f(a[4 * t]), f(a[4 * t + 1]), f(a[4 * t + 2]), f(a[4 * t + 3]));
      if (same && e0 >= 0 && e0 + 4 <= V) {
        st_f4(yb + 4 * q, o);
      } else {
        if (e0 + 0 >= 0 && e0 + 0 < V) st_f1(yr + e0 + 0, o.x);
        if (e0 + 1 >= 0 && e0 + 1 < V) st_f1(yr + e0 + 1, o.y);
        if (e0 + 2 >= 0 && e0 + 2 < V) st_f1(yr + e0 + 2, o.z);
        if (e0 + 3 >= 0 && e0 + 3 < V) st_f1(yr + e0 + 3, o.w);
      }
    }
  }
}

// --------------------------------------------------------------- stream --
// One CTA per row; every pass of the algorithm reads global memory.
template <int BLOCK, int U, int ALG, int P1 = 0>
__global__ void __launch_bounds__(BLOCK)
    k_softmax_stream(const float* __restrict__ x, long long ldx, float* __restrict__ y,
                     long long ldy, long long rows, long long V, void* ws, int pf, long long row0 = 0) {
  constexpr int NW = BLOCK / 32;
  __shared__ float smf[2 * NW];
  __shared__ double smd[NW];
  const int t = threadIdx.x;
  for (long long row = row0 + blockIdx.x; row < rows; row += gridDim.x) {
    const Seg s = make_seg(x + row * ldx, V);
    float* yr = y + row * ldy;
    float mn = -kNegInf;
    float M, r = 0.0f;
    double rd = 0.0;
    Recip rc{0.0f, 0.0f};  // safe / online: 1/d as hi + lo
    bool bad;
    if constexpr (ALG == osmx_host::kOnline) {
      // Pass 1: Alg. 3 lines 1-6, batch-max-first update per U float4s.
      L2Acc acc;
      stream_seg<BLOCK, U, P1>(
          s, t,
          [&](float v, long long) {
            mn = fminf(mn, v);
            acc.add1(v);
          },
          [&](float4 (&v)[U], long long, int cnt) {
            float bm = kNegInf, bn = -kNegInf;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
              if (u < cnt) bn = fminf(bn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
            }
            mn = fminf(mn, bn);
            acc.raise(bm);
            acc.add_batch<U>(v);
          },
          pf);
      MD tot = md_cta_reduce<NW>(acc.finish(), smf);
      mn = cta_min<NW>(mn, smf);
      M = tot.m;
      rc = recip_of((double)tot.d);
      bad = !(tot.d == tot.d) || !isfinite(M) || mn == kNegInf;
    } else if constexpr (ALG == osmx_host::kSafe) {
      // Pass 1: max (kernels.hpp:54).  Pass 2: normalizer (:56).
      float m = kNegInf;
      stream_seg<BLOCK, U, P1>(
          s, t,
          [&](float v, long long) {
            m = fmaxf(m, v);
            mn = fminf(mn, v);
            if (v != v) m = v;  // keep NaN visible
          },
          [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
              if (u < cnt) mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
            }
          },
          pf);
      M = cta_max<NW>(m, smf);
      mn = cta_min<NW>(mn, smf);
      SafeAcc sacc;  // sum e^(x - M), terms from x - M (shift invariant)
      sacc.raise(M);
      stream_seg<BLOCK, U, P1>(
          s, t, [&](float v, long long) { sacc.d += sacc.term(v); },
          [&](float4 (&v)[U], long long, int) { sacc.add_batch<U>(v); });
      double d = (M == kNegInf) ? 0.0 : sacc.d;
      d = cta_sum_d<NW>(d, smd);
      rc = recip_of(d);
      bad = !(d == d) || !isfinite(M) || mn == kNegInf;
    } else {
      // Naive: d = sum double(expf(x)) (kernels.hpp:43-44).
      double d = 0.0;
      float mx = kNegInf;
      stream_seg<BLOCK, U, P1>(
          s, t,
          [&](float v, long long) {
            d += (double)expf(v);
            mx = fmaxf(mx, v);
            mn = fminf(mn, v);
          },
          [&](float4 (&v)[U], long long, int cnt) {
            float part = 0.0f;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (u < cnt) {
                d += (double)expf(v[u].x) + (double)expf(v[u].y) + (double)expf(v[u].z) + (double)expf(v[u].w);
                mx = fmaxf(mx, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
                mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
              }
            }
            (void)part;
          });
      d = cta_sum_d<NW>(d, smd);
      mx = cta_max<NW>(mx, smf);
      mn = cta_min<NW>(mn, smf);
      rd = 1.0 / d;
      M = 0.0f;
      bad = !(d == d) || !isfinite(mx) || mn == kNegInf;
    }
    if (bad && t == 0) flag_bad_row(ws, row);
    // Final pass: y = e^(x - m) / d (kernels.hpp:57 / :68; naive :45),
    // walking the row backwards so its first reads hit the lines pass 1
    // (online, naive) read last.
    if constexpr (ALG == osmx_host::kNaive) {
      map_seg<BLOCK, U>(s, yr, t, [&](float v) { return (float)((double)expf(v) * rd); },
                        std::integral_constant<bool, true>{});
    } else if constexpr (ALG == osmx_host::kOnline) {
      map_seg<BLOCK, U>(s, yr, t, [&](float v) { return out_soft<ALG == osmx_host::kSafe>(v, M, rc); }, std::integral_constant<bool, true>{});
    } else {
      map_seg<BLOCK, U>(s, yr, t, [&](float v) { return out_soft<ALG == osmx_host::kSafe>(v, M, rc); });
    }
  }
}

// ---------------------------------------------------------------- split --
// Record of one chunk: m = running max (online) / max (safe, naive),
// mn = min (non-finite detection), d = normalizer (double so the naive sum
// does not overflow fp32 where the reference's double does not).
struct SRec {
  float m;
  float mn;
  double d;
};

// Phase 0 for all algorithms; phase 1 (safe only) recomputes d against the
// row max gathered from the phase-0 records.
template <int BLOCK, int U, int ALG, int PHASE>
__global__ void __launch_bounds__(BLOCK)
    k_softmax_split_part(const float* __restrict__ x, long long ldx, long long V, long long chunk,
                         SRec* __restrict__ rec) {
  constexpr int NW = BLOCK / 32;
  __shared__ float smf[2 * NW];
  __shared__ double smd[NW];
  const int S = gridDim.x;
  const long long row = blockIdx.y;
  const long long c0 = (long long)blockIdx.x * chunk;
  const long long n = std::min(chunk, V - c0);
  const Seg s = make_seg(x + row * ldx + c0, n);
  const int t = threadIdx.x;
  SRec* rr = rec + row * S;
  if constexpr (ALG == osmx_host::kSafe && PHASE == 2) {
    // the safe fused top-K's normalizer: d in double, exp(double(x) - M)
    // (reference kernels.hpp:95-96; its keys divide by d)
    float M = kNegInf;
    for (int i = t; i < S; i += BLOCK) M = fmaxf(M, rr[i].m);
    M = cta_max<NW>(M, smf);
    __shared__ double tab[32];
    exp2_tab_init(tab);
    __syncthreads();
    const double Md = (double)M;
    double d = 0.0;
    stream_seg<BLOCK, U, false>(
        s, t, [&](float v, long long) { d += exp_neg_d((double)v - Md, tab); },
        [&](float4 (&v)[U], long long, int) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            d += (exp_neg_d((double)v[u].x - Md, tab) + exp_neg_d((double)v[u].y - Md, tab)) +
                 (exp_neg_d((double)v[u].z - Md, tab) + exp_neg_d((double)v[u].w - Md, tab));
        });
    d = cta_sum_d<NW>(d, smd);
    __syncthreads();  // every thread has read rr[*].m before it is rewritten
    if (t == 0) rr[blockIdx.x].d = d;
    return;
  }
  if constexpr (ALG == osmx_host::kSafe && PHASE == 1) {
    float M = kNegInf;
    for (int i = t; i < S; i += BLOCK) M = fmaxf(M, rr[i].m);
    M = cta_max<NW>(M, smf);
    SafeAcc sacc;  // sum e^(x - M), terms from x - M (shift invariant)
    sacc.raise(M);
    stream_seg<BLOCK, U, false>(
        s, t, [&](float v, long long) { sacc.d += sacc.term(v); },
        [&](float4 (&v)[U], long long, int) { sacc.add_batch<U>(v); });
    double d = (M == kNegInf) ? 0.0 : sacc.d;
    d = cta_sum_d<NW>(d, smd);
    __syncthreads();  // every thread has read rr[*].m before it is rewritten
    if (t == 0) rr[blockIdx.x].d = d;
    return;
  }
  float mn = -kNegInf;
  if constexpr (ALG == osmx_host::kOnline) {
    L2Acc acc;
    stream_seg<BLOCK, U, false>(
        s, t,
        [&](float v, long long) {
          mn = fminf(mn, v);
          acc.add1(v);
        },
        [&](float4 (&v)[U], long long, int cnt) {
          float bm = kNegInf, bn = -kNegInf;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            if (u < cnt) bn = fminf(bn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
          }
          mn = fminf(mn, bn);
          acc.raise(bm);
          acc.add_batch<U>(v);
        });
    MD tot = md_cta_reduce<NW>(acc.finish(), smf);
    mn = cta_min<NW>(mn, smf);
    if (t == 0) rr[blockIdx.x] = SRec{tot.m, mn, (double)tot.d};
  } else if constexpr (ALG == osmx_host::kSafe) {
    float m = kNegInf;
    stream_seg<BLOCK, U, false>(
        s, t,
        [&](float v, long long) {
          m = fmaxf(m, v);
          mn = fminf(mn, v);
          if (v != v) m = v;
        },
        [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            if (u < cnt) mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
          }
        });
    m = cta_max<NW>(m, smf);
    mn = cta_min<NW>(mn, smf);
    if (t == 0) rr[blockIdx.x] = SRec{m, mn, 0.0};
  } else {
    double d = 0.0;
    float mx = kNegInf;
    stream_seg<BLOCK, U, false>(
        s, t,
        [&](float v, long long) {
          d += (double)expf(v);
          mx = fmaxf(mx, v);
          mn = fminf(mn, v);
        },
        [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (u < cnt) {
              d += (double)expf(v[u].x) + (double)expf(v[u].y) + (double)expf(v[u].z) + (double)expf(v[u].w);
              mx = fmaxf(mx, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
              mn = fminf(mn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
            }
          }
        });
    d = cta_sum_d<NW>(d, smd);
    mx = cta_max<NW>(mx, smf);
    mn = cta_min<NW>(mn, smf);
    if (t == 0) rr[blockIdx.x] = SRec{mx, mn, d};
  }
}

// Merge the S records of the row (every CTA does it; S*16 bytes from L2),
// flag the row once, then write y for this CTA's chunk.
template <int BLOCK, int U, int ALG>
__global__ void __launch_bounds__(BLOCK)
    k_softmax_split_scale(const float* __restrict__ x, long long ldx, float* __restrict__ y,
                          long long ldy, long long V, long long chunk, const SRec* __restrict__ rec,
                          void* ws) {
  constexpr int NW = BLOCK / 32;
  __shared__ float smf[2 * NW];
  __shared__ double smd[NW];
  const int S = gridDim.x;
  const long long row = blockIdx.y;
  const int t = threadIdx.x;
  pdl_wait();  // records come from the part kernel
  const SRec* rr = rec + row * S;
  float M = kNegInf, mn = -kNegInf, r = 0.0f;
  double rd = 0.0;
  Recip rc{0.0f, 0.0f};  // safe / online: 1/d as hi + lo
  bool bad;
  if constexpr (ALG == osmx_host::kOnline) {
    MD a = md_identity();
    for (int i = t; i < S; i += BLOCK) {
      a = md_merge(a, MD{rr[i].m, (float)rr[i].d});
      mn = fminf(mn, rr[i].mn);
    }
    a = md_cta_reduce<NW>(a, smf);
    mn = cta_min<NW>(mn, smf);
    M = a.m;
    rc = recip_of((double)a.d);
    bad = !(a.d == a.d) || !isfinite(M) || mn == kNegInf;
  } else if constexpr (ALG == osmx_host::kSafe) {
    double d = 0.0;
    for (int i = t; i < S; i += BLOCK) {
      M = fmaxf(M, rr[i].m);
      mn = fminf(mn, rr[i].mn);
      d += rr[i].d;
    }
    M = cta_max<NW>(M, smf);
    mn = cta_min<NW>(mn, smf);
    d = cta_sum_d<NW>(d, smd);
    rc = recip_of(d);
    bad = !(d == d) || !isfinite(M) || mn == kNegInf;
  } else {
    double d = 0.0;
    for (int i = t; i < S; i += BLOCK) {
      M = fmaxf(M, rr[i].m);
      mn = fminf(mn, rr[i].mn);
      d += rr[i].d;
    }
    M = cta_max<NW>(M, smf);
    mn = cta_min<NW>(mn, smf);
    d = cta_sum_d<NW>(d, smd);
    rd = 1.0 / d;
    bad = !(d == d) || !isfinite(M) || mn == kNegInf;
  }
  if (bad && t == 0 && blockIdx.x == 0) flag_bad_row(ws, row);
  // chunks in reverse order: the first CTAs re-read the chunks the part
  // kernel read last (still in L2 when the row is larger than L2)
  const long long c0 = (long long)(S - 1 - blockIdx.x) * chunk;
  const long long n = std::min(chunk, V - c0);
  const Seg s = make_seg(x + row * ldx + c0, n);
  float* yr = y + row * ldy + c0;
  if constexpr (ALG == osmx_host::kNaive) {
    map_seg<BLOCK, U>(s, yr, t, [&](float v) { return (float)((double)expf(v) * rd); },
                      std::integral_constant<bool, true>{});
  } else {
    map_seg<BLOCK, U>(s, yr, t, [&](float v) { return out_soft<ALG == osmx_host::kSafe>(v, M, rc); }, std::integral_constant<bool, true>{});
  }
}

// ------------------------------------------------------ normalizer only --
// Batched run_normalizer / run_normalizer_chunked (normalizer.hpp:61-85):
// (m, d) per row.  chunk > 0 reproduces the contiguous-chunk left-to-right
// merge order; chunk == 0 is the CTA-parallel evaluation.
template <int BLOCK, int U>
__global__ void __launch_bounds__(BLOCK)
    k_normalizer(const float* __restrict__ x, long long ldx, long long rows, long long V,
                 float* __restrict__ om, float* __restrict__ od, void* ws) {
  constexpr int NW = BLOCK / 32;
  __shared__ float smf[2 * NW];
  const int t = threadIdx.x;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const Seg s = make_seg(x + row * ldx, V);
    L2Acc acc;
    float mn = -kNegInf;
    stream_seg<BLOCK, U, false>(
        s, t,
        [&](float v, long long) {
          mn = fminf(mn, v);
          acc.add1(v);
        },
        [&](float4 (&v)[U], long long, int cnt) {
          float bm = kNegInf, bn = -kNegInf;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            if (u < cnt) bn = fminf(bn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
          }
          mn = fminf(mn, bn);
          acc.raise(bm);
          acc.add_batch<U>(v);
        });
    MD tot = md_cta_reduce<NW>(acc.finish(), smf);
    mn = cta_min<NW>(mn, smf);
    if (t == 0) {
      om[row] = tot.m;
      od[row] = tot.d;
      if (!(tot.d == tot.d) || !isfinite(tot.m) || mn == kNegInf) flag_bad_row(ws, row);
    }
  }
}

// ------------------------------------------------------------ launchers --

template <int TPR, int EPT, int ALG>
cudaError_t run_resident(bool vec, const float* x, long long ldx, float* y, long long ldy,
                         long long rows, long long V, void* ws, cudaStream_t st) {
  constexpr int BLOCK = TPR > 256 ? TPR : 256;
  constexpr int RPC = BLOCK / TPR;
  const long long grid = (rows + RPC - 1) / RPC;
  if (vec)
    k_softmax_resident<TPR, EPT, true, ALG><<<(unsigned)grid, BLOCK, 0, st>>>(x, ldx, y, ldy, rows, (int)V, ws);
  else
    k_softmax_resident<TPR, EPT, false, ALG><<<(unsigned)grid, BLOCK, 0, st>>>(x, ldx, y, ldy, rows, (int)V, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int ALG>
cudaError_t dispatch_resident(bool vec, const float* x, long long ldx, float* y, long long ldy,
                              long long rows, long long V_, void* ws, cudaStream_t st) {
  // shapes by capacity: unaligned rows span up to V + 3 float4 lanes
  const long long V = vec ? V_ : V_ + 3;
  auto run = [&](auto tpr, auto ept) {
    return run_resident<decltype(tpr)::value, decltype(ept)::value, ALG>(vec, x, ldx, y, ldy, rows, V_, ws, st);
  };
  using I8 = std::integral_constant<int, 8>;
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  using I128 = std::integral_constant<int, 128>;
  using I256 = std::integral_constant<int, 256>;
  using I512 = std::integral_constant<int, 512>;
  if (V <= 64) return run(I8{}, I8{});
  if (V <= 256) return run(I32{}, I8{});
  if (V <= 512) return run(I32{}, I16{});
  if (V <= 1024) return run(I32{}, I32{});
  if (V <= 2048) return run(I128{}, I16{});
  if (V <= 4096) return run(I256{}, I16{});
  if (V <= 8192) return run(I256{}, I32{});
  if (V <= 16384) return run(I512{}, I32{});
  return cudaErrorInvalidValue;
}

template <int ALG>
cudaError_t run_stream(const float* x, long long ldx, float* y, long long ldy, long long rows,
                       long long V, void* ws, cudaStream_t st, long long row0 = 0) {
  int threads = osmx_host::tuning().stream_threads;
  const int pf = std::max(0, osmx_host::tuning().l2_prefetch);  // off unless forced (measured: mixed)
  // 1024-thread CTAs for long rows (4000 rows, same box, tools/runs/r2_aa.sh):
  // online 131K 0.840 vs 0.916 ms, 316K 2.247 vs 2.406, 562K 4.210 vs 4.490,
  // 1M 7.109 vs 7.282; safe 316K 3.031 vs 3.147, 1M 9.428 vs 9.620.  The
  // fp64-summing naive kernel prefers 512 (562K: 4.424 vs 4.640).
  if (threads == 0) threads = V >= 65536 ? (ALG == osmx_host::kNaive ? 512 : 1024) : 256;
  const int keep = osmx_host::tuning().stream_ctas;  // > 0: persistent, CTAs per SM, evict-last pass 1
  if (keep > 0) {
    const long long grid = std::min<long long>(rows, (long long)keep * osmx_host::num_sms());
    if (threads == 1024)
      k_softmax_stream<1024, 4, ALG, 2><<<(unsigned)grid, 1024, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf);
    else if (threads == 512)
      k_softmax_stream<512, 4, ALG, 2><<<(unsigned)grid, 512, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf);
    else
      k_softmax_stream<256, 4, ALG, 2><<<(unsigned)grid, 256, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf);
    osmx_host::count_launch();
    return cudaGetLastError();
  }
  const long long grid = std::min<long long>(rows - row0, 1LL << 30);
  if (threads == 1024)
    k_softmax_stream<1024, 4, ALG><<<(unsigned)grid, 1024, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf, row0);
  else if (threads == 512)
    k_softmax_stream<512, 4, ALG><<<(unsigned)grid, 512, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf, row0);
  else
    k_softmax_stream<256, 4, ALG><<<(unsigned)grid, 256, 0, st>>>(x, ldx, y, ldy, rows, V, ws, pf, row0);
  osmx_host::count_launch();
  return cudaGetLastError();
}

constexpr int kSplitBlock = 512;
constexpr int kSplitU = 4;

long long split_chunk(long long rows, long long V) {
  long long ch = osmx_host::tuning().split_chunk;
  if (ch <= 0) {
    // ~14 CTAs per SM over the whole problem (3.5 waves of 512-thread CTAs;
    // measured on configs[4], tools/c5_sweep.py), at least 32K elements each.
    const long long target = 14LL * osmx_host::num_sms();
    long long per_row = std::max<long long>(1, target / std::max<long long>(rows, 1));
    ch = (V + per_row - 1) / per_row;
    ch = std::max<long long>(ch, 32768);
  }
  ch = (ch + 15) / 16 * 16;  // keeps every chunk in the row's 16-byte phase
  return ch;
}

template <int ALG>
cudaError_t run_split(const float* x, long long ldx, float* y, long long ldy, long long rows,
                      long long V, void* ws, cudaStream_t st) {
  const long long ch = split_chunk(rows, V);
  const long long S = (V + ch - 1) / ch;
  SRec* rec = reinterpret_cast<SRec*>(static_cast<char*>(ws) + kWsHeader);
  dim3 grid((unsigned)S, (unsigned)rows);
  k_softmax_split_part<kSplitBlock, kSplitU, ALG, 0><<<grid, kSplitBlock, 0, st>>>(x, ldx, V, ch, rec);
  osmx_host::count_launch();
  if (ALG == osmx_host::kSafe) {
    k_softmax_split_part<kSplitBlock, kSplitU, ALG, 1><<<grid, kSplitBlock, 0, st>>>(x, ldx, V, ch, rec);
    osmx_host::count_launch();
  }
  launch_pdl(k_softmax_split_scale<kSplitBlock, kSplitU, ALG>, grid, dim3(kSplitBlock), 0, st, x, ldx, y, ldy, V, ch,
             (const SRec*)rec, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int ALG>
cudaError_t launch_alg(const float* x, long long ldx, float* y, long long ldy, long long rows,
                       long long V, void* ws, cudaStream_t st) {
  const auto& tn = osmx_host::tuning();
  const bool vec = (V % 4 == 0) && (ldx % 4 == 0) && (ldy % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) && ((reinterpret_cast<uintptr_t>(y) & 15u) == 0);
  int shape = tn.shape;
  if (shape == osmx_host::kShapeAuto) {
    // Measured on B200 (tools/shape_sweep.py, inputs out of L2, 4000 and
    // 32768 rows): register-resident rows win up to V ~ 2048; the TMA-staged
    // shared-memory ring from there to 16K (1.1-1.5x the resident / stream
    // kernels at V = 3K-10K), cluster-staged rows up to 16 x 12288; beyond,
    // the stream kernel (one CTA per row) or the split kernel when there are
    // too few rows to fill the SMs.
    if (V <= osmx_host::resident_limit(vec))
      shape = osmx_host::kShapeResident;
    else if (V <= kStagedMaxV)
      shape = osmx_host::kShapeStaged;
    else if (V <= cluster_max_v<ALG>() && rows >= osmx_host::num_sms() / 2)
      shape = osmx_host::kShapeCluster;
    else if (rows >= 2LL * osmx_host::num_sms())
      shape = osmx_host::kShapeStream;
    else
      shape = osmx_host::kShapeSplit;
  }
  if (shape == osmx_host::kShapeResident && V + (vec ? 0 : 3) > 16384) shape = osmx_host::kShapeStream;
  if (shape == osmx_host::kShapeStaged || shape == osmx_host::kShapeCluster) {
    // Rows that only a 16-CTA cluster holds: 7 clusters fill 112 of the 148
    // SMs, so a share of the rows runs concurrently in the streaming kernel
    // on a side stream (fork / join by events on the caller's stream; both
    // flag bad rows with their global row index).
    // Auto: online softmax only, 80% of the rows in clusters (4000 x 177828:
    // 1.119 vs 1.178 ms, 196000: 1.255 vs 1.339; safe softmax measured
    // slower co-run, 1.39 vs 1.33 -- tools/runs/r2_bj.sh).
    const int co = tn.corun >= 0 ? tn.corun : (ALG == osmx_host::kOnline ? 80 : 0);
    if (co > 0 && co < 100 && tn.cluster_size == 0 && V <= kClusterMaxV && V > kStagedMaxV &&
        staged_cluster_size(V) == 16 && rows >= 2LL * osmx_host::num_sms()) {
      const long long r1 = rows * co / 100;
      cudaStream_t side;
      cudaEvent_t fork, join;
      cudaError_t e = osmx_host::side_stream(&side, &fork, &join);
      if (e == cudaSuccess) e = cudaEventRecord(fork, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
      if (e == cudaSuccess) e = run_staged<ALG>(x, ldx, y, ldy, r1, V, ws, st);
      if (e == cudaSuccess) e = run_stream<ALG>(x, ldx, y, ldy, rows, V, ws, side, r1);
      if (e == cudaSuccess) e = cudaEventRecord(join, side);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, join, 0);
      return e;
    }
    if (V <= kClusterMaxV || osmx_host::tuning().cluster_size > 0) return run_staged<ALG>(x, ldx, y, ldy, rows, V, ws, st);
    shape = osmx_host::kShapeStream;
  }
  if (shape == osmx_host::kShapeSplit && rows > 65535) shape = osmx_host::kShapeStream;
  if (shape == osmx_host::kShapeResident) return dispatch_resident<ALG>(vec, x, ldx, y, ldy, rows, V, ws, st);
  if (shape == osmx_host::kShapeSplit) return run_split<ALG>(x, ldx, y, ldy, rows, V, ws, st);
  return run_stream<ALG>(x, ldx, y, ldy, rows, V, ws, st);
}

}  // namespace
