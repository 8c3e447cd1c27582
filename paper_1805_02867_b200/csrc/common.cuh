// common.cuh -- device building blocks shared by every osmx sm_100a kernel.
//
//   * cache-hinted 128-bit / 32-bit global loads and streaming stores
//   * the online normalizer state (m, d) and its merge, Eq. 4/5 of the paper
//     (reference normalizer.hpp:24-58), at thread, group and CTA level
//   * the per-thread register top-K list with the reference's strict-'<'
//     insertion order (topk.hpp:34-44) and group/CTA merges under the total
//     order (value desc, index asc) (oracle.cpp:48-51)
//   * the workspace header that carries the non-finite-row flag
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace osmx_dev {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNegInf = -__builtin_huge_valf();

// ------------------------------------------------------------ memory ops --

// Read-only, no L1 allocation: every element is read by exactly one thread.
__device__ __forceinline__ float4 ld_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_f1(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// Last read of a line (final pass of a multi-pass kernel): evict-first
// L2 policy so the dead lines leave room for data still to be re-read.
__device__ __forceinline__ unsigned long long pol_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_f4_last(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol_evict_first()));
  return r;
}
__device__ __forceinline__ float ld_f1_last(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(r)
               : "l"(p), "l"(pol_evict_first()));
  return r;
}
// First read of data the same CTA reads again soon (two-pass kernels with a
// bounded in-flight footprint): evict-last L2 policy.
__device__ __forceinline__ unsigned long long pol_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_f4_keep(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol_evict_last()));
  return r;
}
__device__ __forceinline__ float ld_f1_keep(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(r)
               : "l"(p), "l"(pol_evict_last()));
  return r;
}
// Output is never re-read by the kernel: streaming (evict-first) stores.
__device__ __forceinline__ void st_f4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_f1(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ------------------------------------------------------------- exponent --

// 2^x, MUFU.EX2 (flushes results below 2^-126 to +0).  Only used for the
// normalizer accumulation where terms < 1e-38 cannot change d >= 1.
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// e^(x - m) for the normalizer: the subtraction is done first so the
// argument error stays relative to |x - m| (small where terms matter).
__device__ __forceinline__ float exp_sub(float x, float m) { return ex2((x - m) * kLog2e); }

// ------------------------------------ the reference's libm, bit for bit --
// The safe fused top-K selects on p = float(expf(x - m) / d) with d a double
// (reference kernels.hpp:95-98); matching its indices bit for bit needs the
// host's expf itself.  expf_ref is glibc's expf (the table-driven
// optimized-routines algorithm: N = 32 table, degree-3 polynomial, all in
// double, then one rounding to float), evaluated with the same IEEE double
// operations -- identical to glibc 2.39's expf for every float in
// [-130, 88] except two inputs whose results glibc corrects, listed below
// (checked exhaustively on the host, tools/expf_ref_check.c).
__device__ __constant__ unsigned long long kExpfTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

__device__ __forceinline__ float expf_ref(float x) {
  if (!(x > -150.0f)) return x == x ? 0.0f : x;  // underflow to +0 (and NaN through)
  if (x > 0x1.62e42ep+6f) return __int_as_float(0x7f800000);  // overflow to +inf
  if (__float_as_uint(x) == 0x4202422fu) return __uint_as_float(0x56fc9f1cu);  // glibc-corrected inputs
  if (__float_as_uint(x) == 0xc27c65d9u) return __uint_as_float(0x11fa2993u);
  const double z = __dmul_rn(0x1.71547652b82fep+5, (double)x);
  double kd = __dadd_rn(z, 0x1.8p+52);
  const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
  kd = __dsub_rn(kd, 0x1.8p+52);
  const double r = __dsub_rn(z, kd);
  const unsigned long long t = kExpfTab[ki & 31] + (ki << 47);
  const double sc = __longlong_as_double((long long)t);
  const double q = __fma_rn(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
  double y = __fma_rn(0x1.62e42ff0c52d6p-6, r, 1.0);
  y = __fma_rn(q, __dmul_rn(r, r), y);
  return __double2float_rn(__dmul_rn(y, sc));
}

// e^t in double for t <= 0, relative error ~1e-15: the safe normalizer
// d = sum exp(double(x) - m) (kernels.hpp:95-96) to far below an fp32 ulp,
// at 11 double ops per term (about half of libdevice's exp).  e^t =
// 2^(y/32), y = t * 32/ln2 split as ki + r (|r| <= 1/2, Cody-Waite with a
// two-part constant), 2^(r/32) by a degree-5 Taylor polynomial in r,
// 2^(ki/32) = 2^(ki>>5) * tab[ki & 31] with the table in shared memory
// (exp2_tab_init) -- a constant-bank lookup would serialise over the lanes'
// distinct indices.
__device__ __constant__ double kExp2Tab32[32] = {
    0x1.0000000000000p+0, 0x1.059b0d3158574p+0, 0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0,
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, 0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0,
    0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123422p+0, 0x1.44e086061892dp+0,
    0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0,
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0,
    0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0,
    0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0,
    0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0};

// Call with every thread of the CTA, before a barrier.
__device__ __forceinline__ void exp2_tab_init(double* tab) {
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Tab32[threadIdx.x];
}

__device__ __forceinline__ double exp_neg_d(double t, const double* tab) {
  if (!(t > -708.0)) return t == t ? 0.0 : t;  // underflow (and NaN through)
  const double y = __dmul_rn(t, 0x1.71547652b82fep+5);
  const double kd0 = __dadd_rn(y, 0x1.8p+52);
  const long long ki = __double_as_longlong(kd0) - 0x4338000000000000LL;
  const double kd = __dsub_rn(kd0, 0x1.8p+52);
  double r = __fma_rn(t, 0x1.71547652b82fep+5, -kd);
  r = __fma_rn(t, 0x1.777d0ffda0d24p-51, r);
  double p = __fma_rn(0x1.5d87fe78a6731p-35, r, 0x1.3b2ab6fba4e77p-27);
  p = __fma_rn(p, r, 0x1.c6b08d704a0c0p-20);
  p = __fma_rn(p, r, 0x1.ebfbdff82c58fp-13);
  p = __fma_rn(p, r, 0x1.62e42fefa39efp-6);
  p = __fma_rn(p, r, 1.0);
  const double sc = __longlong_as_double(__double_as_longlong(tab[ki & 31]) + ((ki >> 5) << 52));
  return __dmul_rn(p, sc);
}

// The reference's safe selection key (kernels.hpp:98): float(expf(x - m) / d),
// x - m rounded in float, the quotient in double.  Monotone non-decreasing in
// x (checked with expf_ref over [-130, 0]), so a batch max bounds a batch.
__device__ __forceinline__ float safe_key_ref(float x, float m, double d) {
  return __double2float_rn(__ddiv_rn((double)expf_ref(__fsub_rn(x, m)), d));
}

// ------------------------------------------------------- (m, d) monoid --

struct MD {
  float m;  // running maximum
  float d;  // sum of e^(x - m)
};

__device__ __forceinline__ MD md_identity() { return MD{kNegInf, 0.0f}; }

// 2^k for an integer-valued k <= 0 (or -inf): exact, by exponent bits.
__device__ __forceinline__ float pow2_int(float k) {
  return k < -126.0f ? 0.0f : __int_as_float(((int)k + 127) << 23);
}

// Per-thread online normalizer in the log2 domain (Alg. 3 lines 1-6 with a
// cheaper inner step).  d is kept relative to an INTEGER reference
// n = ceil(m * log2 e), so each term is one FFMA + one ex2:
//     e_j = 2^(x_j*L - n)        (x_j*L - n is exact before the one rounding)
// and a rescale when the max grows is an exact power of two.  finish()
// converts to the reference's (m, d = sum e^(x - m)) with one FFMA whose
// result lies in [0, 1) -- so |m| never enters a rounding error, unlike
// ex2(x*L - m*L).  The remaining approximation, L = RN(log2 e), perturbs
// each term by |x_j - m| * 2^-25, as in e^(x - m) itself.
//
// The log2 domain is exact only while RN(m * L) is within a few units of
// m * L: n = ceil(RN(m*L)) is then an integer next to the exact product and
// every term 2^(x*L - n) stays near 1 for x near m.  Once ulp(m * L) grows
// past ~2^7 (|m| > ~1.5e9) a term could reach 2^(ulp/2) and overflow, and for
// |m| >= 2^127 (e.g. a -FLT_MAX mask) n itself is infinite.  So a thread
// whose batch max has |bm| >= 2^20 switches to `huge` mode for the rest of
// the row: d relative to m in natural units, terms e^(x - m) -- a
// warp-uniform branch per batch, never taken on ordinary logits.
constexpr float kHugeX = 1048576.0f;  // 2^20

struct L2Acc {
  float m = kNegInf;  // running max (natural units)
  float n = kNegInf;  // integer reference, >= m * L up to rounding
  float d = 0.0f;     // sum 2^(x*L - n)   (huge: sum e^(x - m))
  bool huge = false;

  // Raise the reference for a batch whose max is bm (no-op if bm <= m).
  // Ordinary logits take the branch-free path: n only grows, and the
  // rescale 2^(n_old - n_new) is MUFU.EX2 of an integer <= 0 (exact; +0
  // while n is still -inf).  Every batch of every lane used to take the
  // divergent bm > m branch in some lane of the warp (ncu, configs[4]: 82%
  // of the warp-batches); this is 7 instructions and no branch.
  __device__ __forceinline__ void raise(float bm) {
    if (!huge && fabsf(bm) < kHugeX) {
      const float nn = fmaxf(n, ceilf(bm * kLog2e));
      d *= ex2(n - nn);
      n = nn;
      m = fmaxf(m, bm);
    } else {
      raise_slow(bm);
    }
  }
  // Huge magnitudes (|bm| >= 2^20, +-inf), NaN, and threads already in
  // natural units.
  __device__ __forceinline__ void raise_slow(float bm) {
    if (bm > m) {
      if (fabsf(bm) < kHugeX) {
        const float nn = ceilf(bm * kLog2e);
        if (!huge) {
          d *= pow2_int(n - nn);
        } else {  // back from natural units (a masked head): d e^(m-bm) 2^(bm L - nn)
          d *= exp_sub(m, bm) * ex2(fmaf(bm, kLog2e, -nn));
          huge = false;
        }
        n = nn;
      } else if (!huge) {  // leave the log2 domain: d relative to bm
        d = (m == kNegInf) ? d : d * ex2(fmaf(-bm, kLog2e, n));
        huge = isfinite(bm);
        n = bm;
        if (!huge) d *= 0.0f;  // +inf input: keep NaN poison, zero otherwise
      } else {
        d *= exp_sub(m, bm);
      }
      m = bm;
    }
  }
  __device__ __forceinline__ float term(float x) const {
    return huge ? exp_sub(x, m) : ex2(fmaf(x, kLog2e, -n));
  }
  template <int U>
  __device__ __forceinline__ void add_batch(const float4 (&v)[U]) {
    float s = 0.0f;
    if (!huge) {
      // paired FFMA2 / FADD2 (sm_100): the terms round like scalar
      // fmaf(x, L, -n); the batch sums in two float lanes, (a + c) + (b + e)
      // per float4 -- 2 FFMA2 + 4 MUFU + 2 FADD2 per 4 elements
      const float2 L2 = make_float2(kLog2e, kLog2e), N2 = make_float2(-n, -n);
      float2 s2 = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float2 t0 = __ffma2_rn(make_float2(v[u].x, v[u].y), L2, N2);
        const float2 t1 = __ffma2_rn(make_float2(v[u].z, v[u].w), L2, N2);
        const float2 p = __fadd2_rn(make_float2(ex2(t0.x), ex2(t0.y)), make_float2(ex2(t1.x), ex2(t1.y)));
        s2 = __fadd2_rn(s2, p);
      }
      s = s2.x + s2.y;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        s += (exp_sub(v[u].x, m) + exp_sub(v[u].y, m)) + (exp_sub(v[u].z, m) + exp_sub(v[u].w, m));
    }
    d += s;
  }
  __device__ __forceinline__ void add1(float x) {
    raise(x);
    d += term(x);
  }
  // d relative to m: divide by the term the max element itself contributed,
  // 2^(m*L - n) -- the same FFMA + ex2 as in add_batch -- so a row whose
  // other terms vanish gets d == 1 exactly, like the reference's first
  // absorb (normalizer.hpp:36-37).
  __device__ __forceinline__ MD finish() const {
    if (huge || m == kNegInf || !(m == m)) return MD{m, d};
    return MD{m, __fdiv_rn(d, ex2(fmaf(m, kLog2e, -n)))};
  }
};

// Safe-softmax normalizer (Alg. 2, kernels.hpp:55-56): the row max M is known
// before the sum, so every term is e^(x - M) computed from the difference
// x - M alone -- shifting a row by a constant that keeps x + c exact leaves
// every term, d and the outputs bit-identical, the reference's own
// shift-invariance property (test_softmax.cpp "shift invariance").  Like the
// reference, d is a double: the terms are the accurate expf of x - M (0 ulps
// from glibc's on 93% of floats, never more than 2 -- tools/expf_lab.cu; the
// ex2.approx of a rounded (x - M) * log2e would be off by ~|x - M| * 6e-8),
// summed four at a time in float and the partial sums in double.
struct SafeAcc {
  float M = kNegInf;
  double d = 0.0;
  __device__ __forceinline__ void raise(float m) { M = m; }
  __device__ __forceinline__ float termf(float x) const { return expf(x - M); }
  __device__ __forceinline__ double term(float x) const { return (double)termf(x); }
  __device__ __forceinline__ void add4(float a, float b, float c, float e) {
    d += (double)((termf(a) + termf(b)) + (termf(c) + termf(e)));
  }
  template <int U>
  __device__ __forceinline__ void add_batch(const float4 (&v)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) add4(v[u].x, v[u].y, v[u].z, v[u].w);
  }
};

// 1/d split into two floats (hi + lo = 1/d to ~2^-48) so an output
// y = e * (1/d) costs one FMUL and one FFMA and is rounded once:
// y = float(e^(x - m) / d) for the safe and online outputs (kernels.hpp:57,
// :68), the float expf of the float difference over the (double) d.
struct Recip {
  float hi, lo;
};
__device__ __forceinline__ Recip recip_of(double d) {
  const double r = 1.0 / d;
  const float hi = __double2float_rn(r);
  return Recip{hi, __double2float_rn(r - (double)hi)};
}
__device__ __forceinline__ float out_md(float x, float m, Recip r) {
  const float e = expf(x - m);
  return fmaf(e, r.hi, e * r.lo);
}
// The online softmax's output pass keeps the one-FMUL form e * float(1/d):
// its d is an fp32 sum already (Alg. 3), so the lo term buys nothing there,
// and the extra FMUL costs 3-5% in the staged kernels.
template <bool SAFE>
__device__ __forceinline__ float out_soft(float x, float m, Recip r) {
  if constexpr (SAFE) return out_md(x, m, r);
  else return expf(x - m) * r.hi;
}
// The same for a handful of values (top-K epilogues): the double quotient.
__device__ __forceinline__ float out_md(float x, float m, double rd) {
  return __double2float_rn(__dmul_rn((double)expf(x - m), rd));
}

// merge(), reference normalizer.hpp:52-58.  The identity (-inf, 0) is
// absorbing without the NaN that (-inf) - (-inf) would produce.
__device__ __forceinline__ MD md_merge(MD a, MD b) {
  const float M = fmaxf(a.m, b.m);
  // both identities (or a NaN-poisoned empty lane): keep d's poison
  if (M == kNegInf) return MD{kNegInf, a.d + b.d};
  return MD{M, a.d * exp_sub(a.m, M) + b.d * exp_sub(b.m, M)};
}

// XOR-butterfly over `width` lanes (power of two <= 32): every lane of the
// group ends with the group total.
template <int WIDTH>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int WIDTH>
__device__ __forceinline__ float group_min(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int WIDTH>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// (m, d) over a group: the max first, then each lane rescales its own d
// once (one ex2 per lane instead of two per butterfly step of a merge
// tree) and a plain sum -- the same poison rules as md_merge (an empty
// group keeps d's NaN; -inf lanes contribute 0; NaN / +inf poison d).
template <int WIDTH>
__device__ __forceinline__ MD md_group_reduce(MD s) {
  float M = s.m;
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float d = (M == kNegInf) ? s.d : s.d * exp_sub(s.m, M);
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  return MD{M, d};
}
template <int WIDTH>
__device__ __forceinline__ double group_sum_d(double v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// CTA-wide reductions for a CTA that owns exactly one row.  `scratch` must
// hold >= 2*NWARPS floats; the call ends with a __syncthreads so the
// scratch can be reused immediately.
template <int NWARPS>
__device__ __forceinline__ MD md_cta_reduce(MD s, float* scratch) {
  s = md_group_reduce<32>(s);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    scratch[w] = s.m;
    scratch[NWARPS + w] = s.d;
  }
  __syncthreads();
  MD t = md_identity();
  if (l < NWARPS) t = MD{scratch[l], scratch[NWARPS + l]};
  t = md_group_reduce<32>(t);
  __syncthreads();
  return t;
}
template <int NWARPS>
__device__ __forceinline__ float cta_max(float v, float* scratch) {
  v = group_max<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  float t = l < NWARPS ? scratch[l] : kNegInf;
  t = group_max<32>(t);
  __syncthreads();
  return t;
}
template <int NWARPS>
__device__ __forceinline__ float cta_min(float v, float* scratch) {
  v = group_min<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  float t = l < NWARPS ? scratch[l] : -kNegInf;
  t = group_min<32>(t);
  __syncthreads();
  return t;
}
template <int NWARPS>
__device__ __forceinline__ float cta_sum(float v, float* scratch) {
  v = group_sum<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  float t = l < NWARPS ? scratch[l] : 0.0f;
  t = group_sum<32>(t);
  __syncthreads();
  return t;
}
template <int NWARPS>
__device__ __forceinline__ double cta_sum_d(double v, double* scratch) {
  v = group_sum_d<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double t = l < NWARPS ? scratch[l] : 0.0;
  t = group_sum_d<32>(t);
  __syncthreads();
  return t;
}

// ------------------------------------------------------------ workspace --

// Every entry point takes a caller-owned device workspace whose first
// kWsHeader bytes are zero-initialised by osmx_workspace_init: this status
// header (osmx_check_status reads and re-zeroes it) and, from byte
// kWsTicketsOff, the per-row ticket counters of the one-launch wide-row
// top-K (topk_wide.cu; each counter is reset to 0 by the CTA that uses it).
struct WsHeader {
  unsigned long long bad;  // 0 = all rows finite, else (INT64_MAX - first bad row)
  long long row_base;      // added to flagged row ids (host pipeline blocks)
  unsigned long long chunk_ctr;  // dynamic chunk counter of the one-row TMA split (reset by its last CTA)
  unsigned long long pad[13];
};
constexpr int kWsTicketsOff = 128;
constexpr int kWsMaxTickets = 992;  // rows of one wide-row launch
constexpr int kWsHeader = kWsTicketsOff + 4 * kWsMaxTickets;  // 4096

__device__ __forceinline__ void flag_bad_row(void* ws, long long row) {
  WsHeader* h = reinterpret_cast<WsHeader*>(ws);
  atomicMax(&h->bad, static_cast<unsigned long long>(0x7fffffffffffffffLL - (row + h->row_base)));
}

// A row is non-finite iff its normalizer is not finite (NaN / +inf inputs
// poison d) or its minimum is -inf (the one case e^(x-m) hides).
__device__ __forceinline__ bool row_nonfinite(float m, float d, float mn) {
  return !(isfinite(d) && isfinite(m)) || mn == kNegInf;
}

// ---------------------------------------------------------------- top-K --

// Total order of the reference (topk.hpp:40-43 strict '<' bubble; oracle
// comparator oracle.cpp:48-51): a precedes b iff a.v > b.v, or equal values
// and a.i < b.i.  Float compares, so -0.0 == +0.0 as in the reference.
__device__ __forceinline__ bool before(float av, long long ai, float bv, long long bi) {
  return av > bv || (av == bv && ai < bi);
}

// Index order with the -1 sentinel last: compare as unsigned.
template <class I>
__device__ __forceinline__ bool idx_less(I a, I b) {
  using U = typename std::conditional<sizeof(I) == 8, unsigned long long, unsigned>::type;
  return static_cast<U>(a) < static_cast<U>(b);
}

// Per-thread sorted top list with capacity KC >= the runtime k.
//
// The k live slots are RIGHT-aligned: slots [0, KC-k) hold +inf blockers
// that never move, slots [KC-k, KC) hold the running top-k (sorted desc).
// The admission threshold is therefore always v[KC-1] -- a static register
// index (a runtime `v[k-1]` would force the list into local memory).
// normalize() shifts the live slots to the front before merging.
//
// offer(): a thread offers its own elements in increasing index order, so
// the strict '>' test keeps earlier indices ahead of later equal values --
// exactly the reference's insertion (topk.hpp:34-44).
// offer_ordered(): for merges, where candidates arrive in arbitrary index
// order, the full total order (value desc, index asc) decides.
// Live slots start at (-inf, -1) like topk_buffer's constructor
// (topk.hpp:27-28).
template <int KC, class I = int>
struct TopList {
  float v[KC];
  I i[KC];

  __device__ __forceinline__ void init(int k) {
#pragma unroll
    for (int s = 0; s < KC; ++s) {
      v[s] = (s < KC - k) ? -kNegInf : kNegInf;
      i[s] = I(-1);
    }
  }
  // left-aligned, all slots live (merge lists)
  __device__ __forceinline__ void init_empty() {
#pragma unroll
    for (int s = 0; s < KC; ++s) {
      v[s] = kNegInf;
      i[s] = I(-1);
    }
  }
  __device__ __forceinline__ float thr() const { return v[KC - 1]; }

  __device__ __forceinline__ void offer(float x, I j) {
    if (!(x > v[KC - 1])) return;
#pragma unroll
    for (int s = KC - 1; s > 0; --s) {
      if (x > v[s - 1]) {
        v[s] = v[s - 1];
        i[s] = i[s - 1];
      } else if (x > v[s]) {
        v[s] = x;
        i[s] = j;
      }
    }
    if (x > v[0]) {
      v[0] = x;
      i[0] = j;
    }
  }
  __device__ __forceinline__ void offer_ordered(float x, I j) {
    if (x < v[KC - 1]) return;
#pragma unroll
    for (int s = KC - 1; s > 0; --s) {
      if (before_(x, j, v[s - 1], i[s - 1])) {
        v[s] = v[s - 1];
        i[s] = i[s - 1];
      } else if (before_(x, j, v[s], i[s])) {
        v[s] = x;
        i[s] = j;
      }
    }
    if (before_(x, j, v[0], i[0])) {
      v[0] = x;
      i[0] = j;
    }
  }
  // Drop the front slot (taken by a merge round, or a blocker).
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int s = 0; s < KC - 1; ++s) {
      v[s] = v[s + 1];
      i[s] = i[s + 1];
    }
    v[KC - 1] = kNegInf;
    i[KC - 1] = I(-1);
  }
  // Move the k live slots to the front (KC-k pops of blockers).
  __device__ __forceinline__ void normalize(int k) {
#pragma unroll
    for (int step = 0; step < KC - 1; ++step)
      if (step < KC - k) pop();
  }
  __device__ __forceinline__ static bool before_(float av, I ai, float bv, I bi) {
    return av > bv || (av == bv && idx_less(ai, bi));
  }
};

// k rounds of a WIDTH-lane arg-max over the list heads, under (value desc,
// index asc, lane asc).  All lanes of the group receive winner r through
// sink(r, value, index); the winning lane pops its head.  Lanes of one
// group must hold indices in one coordinate system (same row / chunk base).
//
// WIDTH == 32: each round is a handful of warp-wide REDUX reductions (max of
// the ordered value key, then min of the index among the lanes holding it)
// instead of a 5-level shuffle butterfly carrying (value, index, lane):
// ~12 instructions and 3 dependent reductions per round instead of ~60.
// The key maps -0.0 to +0.0 (the reference's float compare ties them); the
// winner's own value is broadcast, so a -0.0 keeps its sign bit.
__device__ __forceinline__ int ord_key(float v) {
  const int i = __float_as_int(v + 0.0f);  // -0 -> +0 (round to nearest)
  return i ^ ((i >> 31) & 0x7fffffff);
}
template <int WIDTH, int KC, class I, class Sink>
__device__ __forceinline__ void group_merge(TopList<KC, I>& L, int k, Sink&& sink) {
  const int lane = (int)(threadIdx.x & 31u);
  if constexpr (WIDTH == 32) {
    for (int r = 0; r < k; ++r) {
      const int kv = ord_key(L.v[0]);
      const int mx = __reduce_max_sync(0xffffffffu, kv);
      const bool top = kv == mx;
      I bi;
      bool win;
      if constexpr (sizeof(I) == 8) {
        const unsigned long long u = top ? static_cast<unsigned long long>(L.i[0]) : ~0ull;
        const unsigned h = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(u >> 32));
        const unsigned l = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(u >> 32) == h
                                                              ? static_cast<unsigned>(u) : 0xffffffffu);
        const unsigned long long w = (static_cast<unsigned long long>(h) << 32) | l;
        bi = static_cast<I>(w);
        win = top && u == w;
      } else {
        const unsigned u = top ? static_cast<unsigned>(L.i[0]) : 0xffffffffu;
        const unsigned m = __reduce_min_sync(0xffffffffu, u);
        bi = static_cast<I>(m);
        win = top && u == m;
      }
      const int bl = __ffs(__ballot_sync(0xffffffffu, win)) - 1;  // lowest lane on a full tie
      const float bv = __shfl_sync(0xffffffffu, L.v[0], bl);
      if (lane == bl) L.pop();
      sink(r, bv, bi);
    }
  } else {
    for (int r = 0; r < k; ++r) {
      float bv = L.v[0];
      I bi = L.i[0];
      int bl = lane;
#pragma unroll
      for (int o = WIDTH / 2; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const I oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        const bool take = ov > bv || (ov == bv && (idx_less(oi, bi) || (oi == bi && ol < bl)));
        if (take) {
          bv = ov;
          bi = oi;
          bl = ol;
        }
      }
      if (lane == bl) L.pop();
      sink(r, bv, bi);
    }
  }
}

// Diagnostic builds only (make timeline, -DOSMX_TIMELINE): %globaltimer
// stamps at fixed points of the one-row combine (tools/c5_timeline.py).
#ifdef OSMX_TIMELINE
__device__ unsigned long long g_tl2[16];
#define OSMX_STAMP(i)                                                          \
  do {                                                                         \
    if ((threadIdx.x & 31) == 0) {                                             \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
      atomicMax(&g_tl2[(i)], t_);                                              \
    }                                                                          \
  } while (0)
#else
#define OSMX_STAMP(i) do { } while (0)
#endif

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while the previous kernel in the stream drains; it must call
// pdl_wait() before touching anything that kernel wrote (no-op when the
// kernel was launched normally).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace osmx_dev
