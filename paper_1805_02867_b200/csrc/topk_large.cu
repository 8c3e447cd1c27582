// topk_large.cu -- top-K for k above the register lists (k > OSMX_MAX_K):
// the reference accepts any 1 <= k <= V (kernels.hpp:28-30, topk.hpp:54-68).
//
// Per row (one 1024-thread CTA):
//   1. row statistics -- online (m, d) for the fused mode (Alg. 3 lines
//      1-6), max then sum for the safe mode (kernels.hpp:95-96), a finiteness
//      check for topk_of;
//   2. radix select of the k-th largest selection key tau (3 passes of 11 /
//      11 / 10 bits over order-preserving uint32 keys, shared-memory
//      histograms);
//   3. one ordered-compaction pass: every element with key > tau and the
//      (k - #>tau) lowest-index elements with key == tau, written in index
//      order (block scans);
// then a stable descending segmented radix sort of the k candidates per row
// (CUB; stability keeps equal keys in index order = the reference's
// tie-to-lower-index rule, topk.hpp:40-43) and an epilogue that writes the
// values (fused: e^(x - m) / d, kernels.hpp:122) and int64 indices.
//
// Selection keys: raw x (fused, kernels.hpp:116-118; topk_of), or the
// probability float(e^(x - M) / d) (safe fused, kernels.hpp:98).  -0.0 is
// keyed as +0.0 (the reference compares floats: -0.0 == +0.0).
#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.hpp"
#include "stream.cuh"

using namespace osmx_dev;

namespace {

// Block barrier after divergent code (per-lane atomics, predicated
// candidate appends): the non-.aligned barrier.sync, whose arrival is per
// thread -- the .aligned bar.sync that __syncthreads() emits requires a
// converged warp, and compute-sanitizer synccheck flagged this kernel's
// barriers after the candidate appends.
__device__ __forceinline__ void cta_sync() {
  __syncwarp();
  asm volatile("barrier.sync 0;" ::: "memory");
}

constexpr int kLT = 1024;  // threads per row
constexpr int kLW = kLT / 32;

__device__ __forceinline__ unsigned fkey(float f) {
  f = (f == 0.0f) ? 0.0f : f;
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Block-wide exclusive scan of two counters (all threads).
__device__ __forceinline__ void block_scan2(int a, int b, int& a_pre, int& b_pre, int& a_tot, int& b_tot,
                                            int* sm /* 2 * kLW */) {
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  int ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ta = __shfl_up_sync(0xffffffffu, ia, o), tb = __shfl_up_sync(0xffffffffu, ib, o);
    if (l >= o) ia += ta, ib += tb;
  }
  if (l == 31) sm[w] = ia, sm[kLW + w] = ib;
  cta_sync();
  if (w == 0) {
    int va = l < kLW ? sm[l] : 0, vb = l < kLW ? sm[kLW + l] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ta = __shfl_up_sync(0xffffffffu, va, o), tb = __shfl_up_sync(0xffffffffu, vb, o);
      if (l >= o) va += ta, vb += tb;
    }
    if (l < kLW) sm[l] = va, sm[kLW + l] = vb;  // inclusive over warps
  }
  cta_sync();
  a_tot = sm[kLW - 1];
  b_tot = sm[2 * kLW - 1];
  a_pre = (w ? sm[w - 1] : 0) + ia - a;
  b_pre = (w ? sm[kLW + w - 1] : 0) + ib - b;
  cta_sync();
}

// MODE: 0 fused online (key raw x, out e^(x-m)/d), 1 topk_of (raw), 2 safe (key p).
template <int MODE>
__global__ void __launch_bounds__(kLT, 1)
    k_topk_large_select(const float* __restrict__ x, long long ldx, long long V, int k, unsigned* __restrict__ ckey,
                        int* __restrict__ cidx, float* __restrict__ rowM, float* __restrict__ rowR, void* ws) {
  constexpr int U = 4;
  __shared__ float smf[2 * kLW];
  __shared__ int smi[2 * kLW];
  __shared__ unsigned hist[2048];
  __shared__ unsigned sel[2];  // chosen bucket, count above it
  const long long row = blockIdx.x;
  const int t = threadIdx.x;
  const float* xr = x + row * ldx;
  const Seg s = make_seg(xr, V);

  // 1. statistics
  __shared__ double smd[kLW];
  float M = 0.0f, R = 1.0f;  // R: the row normalizer d
  double D = 1.0;  // safe mode: the double normalizer
  bool bad = false;
  if constexpr (MODE == 0) {
    L2Acc acc;
    float mn = -kNegInf;
    stream_seg<kLT, U, 0>(
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
    const MD tot = md_cta_reduce<kLW>(acc.finish(), smf);
    mn = cta_min<kLW>(mn, smf);
    M = tot.m;
    R = tot.d;  // the epilogue divides by it in double (out_md)
    bad = !(tot.d == tot.d) || !isfinite(M) || mn == kNegInf;
  } else {
    float m = kNegInf, chk = 0.0f;
    stream_seg<kLT, U, 0>(
        s, t,
        [&](float v, long long) {
          m = fmaxf(m, v);
          chk = fmaf(v, 0.0f, chk);
        },
        [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            if (u < cnt) chk = fmaf(v[u].x, 0.0f, fmaf(v[u].y, 0.0f, fmaf(v[u].z, 0.0f, fmaf(v[u].w, 0.0f, chk))));
          }
        });
    chk = cta_sum<kLW>(chk, smf);
    bad = !(chk == chk);
    if constexpr (MODE == 2) {
      // d = sum exp(double(x) - m) in double (kernels.hpp:95-96)
      M = cta_max<kLW>(m, smf);
      __shared__ double tab[32];
      exp2_tab_init(tab);
      cta_sync();
      const double Md = (double)M;
      double d = 0.0;
      stream_seg<kLT, U, 0>(
          s, t, [&](float v, long long) { d += exp_neg_d((double)v - Md, tab); },
          [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (u < cnt)
                d += (exp_neg_d((double)v[u].x - Md, tab) + exp_neg_d((double)v[u].y - Md, tab)) +
                     (exp_neg_d((double)v[u].z - Md, tab) + exp_neg_d((double)v[u].w - Md, tab));
          });
      D = cta_sum_d<kLW>(d, smd);
      bad = bad || !(D == D) || !isfinite(M);
    }
  }
  if (t == 0) {
    rowM[row] = M;
    rowR[row] = R;
    if (bad) flag_bad_row(ws, row);
  }
  auto key = [&](float v) -> unsigned {
    if constexpr (MODE == 2)
      return fkey(safe_key_ref(v, M, D));  // the reference's p, bit for bit
    else
      return fkey(v);
  };

  // 2. radix select of the k-th largest key (digits 11 / 11 / 10 bits)
  unsigned prefix = 0, pmask = 0;
  int krem = k;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
#pragma unroll 1
  for (int p = 0; p < 3; ++p) {
    const int sh = shifts[p], nb = 1 << widths[p];
    for (int i = t; i < nb; i += kLT) hist[i] = 0u;
    cta_sync();
    auto add = [&](float v) {
      const unsigned u = key(v);
      if ((u & pmask) == prefix) atomicAdd(&hist[(u >> sh) & (nb - 1)], 1u);
    };
    stream_seg<kLT, U, 0>(
        s, t, [&](float v, long long) { add(v); },
        [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (u < cnt) add(v[u].x), add(v[u].y), add(v[u].z), add(v[u].w);
        });
    cta_sync();
    // suffix counts: thread t owns buckets [2t, 2t+1] of the reversed order
    const int r0 = 2 * t;  // reversed index: bucket nb-1-r
    unsigned c0 = r0 < nb ? hist[nb - 1 - r0] : 0u, c1 = r0 + 1 < nb ? hist[nb - 2 - r0] : 0u;
    int pre, dummy, tot, dtot;
    block_scan2((int)(c0 + c1), 0, pre, dummy, tot, dtot, smi);
    // count of keys with digit above bucket (nb-1-r0): pre
    if (r0 < nb) {
      if (pre < krem && pre + (int)c0 >= krem) {
        sel[0] = (unsigned)(nb - 1 - r0);
        sel[1] = (unsigned)pre;
      } else if (r0 + 1 < nb && pre + (int)c0 < krem && pre + (int)(c0 + c1) >= krem) {
        sel[0] = (unsigned)(nb - 2 - r0);
        sel[1] = (unsigned)(pre + c0);
      }
    }
    cta_sync();
    prefix |= sel[0] << sh;
    pmask |= (unsigned)(nb - 1) << sh;
    krem -= (int)sel[1];
    cta_sync();
  }
  const unsigned tau = prefix;
  const int need_eq = krem;  // elements equal to tau to take (lowest indices)

  // 3. ordered compaction: thread t takes elements [base + 4t, base + 4t + 4)
  unsigned* ok = ckey + row * (long long)k;
  int* oi = cidx + row * (long long)k;
  int gt_base = 0, eq_base = 0;
  for (long long base = 0; base < V; base += 4LL * kLT) {
    unsigned kk[4];
    int gt = 0, eq = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long e = base + 4LL * t + i;
      kk[i] = e < V ? key(ld_f1(xr + e)) : 0u;
      const bool in = e < V;
      gt += (in && kk[i] > tau);
      eq += (in && kk[i] == tau);
    }
    int gpre, epre, gtot, etot;
    block_scan2(gt, eq, gpre, epre, gtot, etot, smi);
    int gb = gt_base + gpre, ebf = eq_base + epre;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long e = base + 4LL * t + i;
      if (e >= V) break;
      if (kk[i] > tau) {
        const int pos = gb + min(ebf, need_eq);
        ok[pos] = kk[i];
        oi[pos] = (int)e;
        ++gb;
      } else if (kk[i] == tau) {
        if (ebf < need_eq) {
          const int pos = gb + ebf;
          ok[pos] = kk[i];
          oi[pos] = (int)e;
        }
        ++ebf;
      }
    }
    gt_base += gtot;
    eq_base += etot;
  }
}

// ------------------------------------------------------------ fast path --
// Fused online softmax + top-k and topk_of for 32 < k <= kFastK, two reads
// of the row instead of five, no global sort:
//   pass A  the row statistics (as above) and a 2048-bin histogram of the top
//           11 bits of every key (shared-memory atomics);
//   select  the bucket b* holding the k-th largest key (suffix scan);
//   pass B  every element whose bucket is >= b* -- a superset of the top k,
//           every tie at the k-th value included -- appended to shared
//           memory (key, index); at most kFastCap of them;
//   sort    a bitonic sort of the candidates under (key desc, index asc),
//           the reference's order (topk.hpp:37-43), in shared memory; the
//           first k are the answer, values re-read from x (so -0.0 keeps its
//           sign in topk_of).
// Rows whose boundary bucket is too full (heavy ties) take the radix path
// (passes 2-3 and the ordered compaction above) into the workspace, then the
// same shared-memory sort of their k candidates.
constexpr int kFastK = 4096;
constexpr int kFastCap = 8192;

// (key desc, index asc): a precedes b
__device__ __forceinline__ bool kbefore(unsigned ka, int ia, unsigned kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}
// Bitonic sort of P (a power of two <= kFastCap) entries, "before" first.
__device__ __forceinline__ void smem_bitonic(unsigned* ck, int* ci, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int ls = __ffs(size) - 2; ls >= 0; --ls) {  // stride = 2^ls (shifts, no integer division)
      const int stride = 1 << ls;
      for (int i = threadIdx.x; i < (P >> 1); i += kLT) {
        const int lo = ((i >> ls) << (ls + 1)) | (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;  // this block ends "before"-first
        const unsigned a = ck[lo], b = ck[hi];
        const int ai = ci[lo], bi = ci[hi];
        if (up ? kbefore(b, bi, a, ai) : kbefore(a, ai, b, bi)) {
          ck[lo] = b;
          ci[lo] = bi;
          ck[hi] = a;
          ci[hi] = ai;
        }
      }
      cta_sync();
    }
  }
}

// Suffix-scan bucket choice over nb buckets: sel[0] = the bucket holding
// the krem-th largest, sel[1] = keys in higher buckets.
__device__ __forceinline__ void pick_bucket(const unsigned* hist, int nb, int krem, unsigned* sel, int* smi) {
  const int t = threadIdx.x;
  const int r0 = 2 * t;  // reversed index: bucket nb-1-r
  const unsigned c0 = r0 < nb ? hist[nb - 1 - r0] : 0u, c1 = r0 + 1 < nb ? hist[nb - 2 - r0] : 0u;
  int pre, dummy, tot, dtot;
  block_scan2((int)(c0 + c1), 0, pre, dummy, tot, dtot, smi);
  if (r0 < nb) {
    if (pre < krem && pre + (int)c0 >= krem) {
      sel[0] = (unsigned)(nb - 1 - r0);
      sel[1] = (unsigned)pre;
    } else if (r0 + 1 < nb && pre + (int)c0 < krem && pre + (int)(c0 + c1) >= krem) {
      sel[0] = (unsigned)(nb - 2 - r0);
      sel[1] = (unsigned)(pre + c0);
    }
  }
  cta_sync();
}

// MODE: 0 fused online (key raw x, out e^(x-m)/d), 1 topk_of (raw).
template <int MODE>
__global__ void __launch_bounds__(kLT, 1)
    k_topk_large_fast(const float* __restrict__ x, long long ldx, long long V, int k, float* __restrict__ vals,
                      long long* __restrict__ idx, unsigned* __restrict__ ckey, int* __restrict__ cidx, void* ws) {
  constexpr int U = 4;
  extern __shared__ __align__(16) unsigned char fsm[];
  unsigned* hist = reinterpret_cast<unsigned*>(fsm);        // 2048
  unsigned* ck = hist + 2048;                                // kFastCap
  int* ci = reinterpret_cast<int*>(ck + kFastCap);           // kFastCap
  __shared__ float smf[2 * kLW];
  __shared__ int smi[2 * kLW];
  __shared__ unsigned sel[2];
  __shared__ int ncand;
  const long long row = blockIdx.x;
  const int t = threadIdx.x;
  const float* xr = x + row * ldx;
  const Seg s = make_seg(xr, V);
  for (int i = t; i < 2048; i += kLT) hist[i] = 0u;
  if (t == 0) ncand = 0;
  cta_sync();

  // pass A: statistics + top-11-bit histogram
  auto h = [&](float v) { atomicAdd(&hist[fkey(v) >> 21], 1u); };
  float M = 0.0f, R = 1.0f;
  bool bad = false;
  if constexpr (MODE == 0) {
    L2Acc acc;
    float mn = -kNegInf;
    stream_seg<kLT, U, 2>(
        s, t,
        [&](float v, long long) {
          mn = fminf(mn, v);
          acc.add1(v);
          h(v);
        },
        [&](float4 (&v)[U], long long, int cnt) {
          float bm = kNegInf, bn = -kNegInf;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            if (u < cnt) {
              bn = fminf(bn, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
              h(v[u].x), h(v[u].y), h(v[u].z), h(v[u].w);
            }
          }
          mn = fminf(mn, bn);
          acc.raise(bm);
          acc.add_batch<U>(v);
        });
    const MD tot = md_cta_reduce<kLW>(acc.finish(), smf);
    mn = cta_min<kLW>(mn, smf);
    M = tot.m;
    R = tot.d;
    bad = !(tot.d == tot.d) || !isfinite(M) || mn == kNegInf;
  } else {
    float chk = 0.0f;
    stream_seg<kLT, U, 2>(
        s, t,
        [&](float v, long long) {
          chk = fmaf(v, 0.0f, chk);
          h(v);
        },
        [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (u < cnt) {
              chk = fmaf(v[u].x, 0.0f, fmaf(v[u].y, 0.0f, fmaf(v[u].z, 0.0f, fmaf(v[u].w, 0.0f, chk))));
              h(v[u].x), h(v[u].y), h(v[u].z), h(v[u].w);
            }
        });
    chk = cta_sum<kLW>(chk, smf);
    bad = !(chk == chk);
  }
  if (t == 0 && bad) flag_bad_row(ws, row);
  cta_sync();  // histogram complete
  pick_bucket(hist, 2048, k, sel, smi);
  const unsigned bstar = sel[0];
  const int total = (int)sel[1] + (int)hist[bstar];

  int n;
  if (total <= kFastCap) {
    // pass B: the candidates (order of arrival is irrelevant: the sort uses
    // the full (key, index) order)
    auto take = [&](float v, long long j) {
      const unsigned u = fkey(v);
      if ((u >> 21) >= bstar) {
        const int p = atomicAdd(&ncand, 1);
        ck[p] = u;
        ci[p] = (int)j;
      }
    };
    stream_seg<kLT, U, 1>(
        s, t, take,
        [&](float4 (&v)[U], long long q0, int cnt) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (u >= cnt) break;
            const long long j = body_index(s, q0 + (long long)u * kLT, 0);
            if (((fkey(fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w))) >> 21) < bstar)) continue;
            take(v[u].x, j), take(v[u].y, j + 1), take(v[u].z, j + 2), take(v[u].w, j + 3);
          }
        });
    cta_sync();
    n = ncand;
    // Trim the candidates to (about) k before sorting: a radix select of the
    // k-th largest key over the shared-memory candidates (3 digits), then keep
    // every key > tau and every key == tau (ties, in any order; the sort
    // puts the lowest indices first).  Sorting ~k instead of ~3k entries.
    if (n > 2 * k) {
      unsigned prefix = 0, pmask = 0;
      int krem = k;
      const int shifts[3] = {21, 10, 0};
      const int widths[3] = {11, 11, 10};
#pragma unroll 1
      for (int p = 0; p < 3; ++p) {
        const int sh = shifts[p], nb = 1 << widths[p];
        for (int i = t; i < nb; i += kLT) hist[i] = 0u;
        cta_sync();
        for (int i = t; i < n; i += kLT) {
          const unsigned u = ck[i];
          if ((u & pmask) == prefix) atomicAdd(&hist[(u >> sh) & (nb - 1)], 1u);
        }
        cta_sync();
        pick_bucket(hist, nb, krem, sel, smi);
        prefix |= sel[0] << sh;
        pmask |= (unsigned)(nb - 1) << sh;
        krem -= (int)sel[1];
        cta_sync();
      }
      const unsigned tau = prefix;
      constexpr int kPer = kFastCap / kLT;  // entries per thread (8)
      unsigned kk[kPer];
      int ii[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int i = t + q * kLT;
        kk[q] = i < n ? ck[i] : 0u;
        ii[q] = i < n ? ci[i] : 0;
      }
      if (t == 0) ncand = 0;
      cta_sync();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (t + q * kLT < n && kk[q] >= tau) {
          const int pos = atomicAdd(&ncand, 1);
          ck[pos] = kk[q];
          ci[pos] = ii[q];
        }
      }
      cta_sync();
      n = ncand;
    }
  } else {
    // heavy ties at the boundary: exact radix select + ordered compaction of
    // the k candidates (index order) into the workspace, then sort them here
    unsigned* okey = ckey + row * (long long)k;
    int* oidx = cidx + row * (long long)k;
    unsigned prefix = 0, pmask = 0;
    int krem = k;
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
#pragma unroll 1
    for (int p = 0; p < 3; ++p) {
      const int sh = shifts[p], nb = 1 << widths[p];
      for (int i = t; i < nb; i += kLT) hist[i] = 0u;
      cta_sync();
      auto add = [&](float v) {
        const unsigned u = fkey(v);
        if ((u & pmask) == prefix) atomicAdd(&hist[(u >> sh) & (nb - 1)], 1u);
      };
      stream_seg<kLT, U, 0>(
          s, t, [&](float v, long long) { add(v); },
          [&](float4 (&v)[U], long long, int cnt) {
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (u < cnt) add(v[u].x), add(v[u].y), add(v[u].z), add(v[u].w);
          });
      cta_sync();
      pick_bucket(hist, nb, krem, sel, smi);
      prefix |= sel[0] << sh;
      pmask |= (unsigned)(nb - 1) << sh;
      krem -= (int)sel[1];
      cta_sync();
    }
    const unsigned tau = prefix;
    const int need_eq = krem;
    int gt_base = 0, eq_base = 0;
    for (long long base = 0; base < V; base += 4LL * kLT) {
      unsigned kk[4];
      int gt = 0, eq = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const long long e = base + 4LL * t + i;
        kk[i] = e < V ? fkey(ld_f1(xr + e)) : 0u;
        gt += (e < V && kk[i] > tau);
        eq += (e < V && kk[i] == tau);
      }
      int gpre, epre, gtot, etot;
      block_scan2(gt, eq, gpre, epre, gtot, etot, smi);
      int gb = gt_base + gpre, ebf = eq_base + epre;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const long long e = base + 4LL * t + i;
        if (e >= V) break;
        if (kk[i] > tau) {
          const int pos = gb + min(ebf, need_eq);
          okey[pos] = kk[i];
          oidx[pos] = (int)e;
          ++gb;
        } else if (kk[i] == tau) {
          if (ebf < need_eq) {
            const int pos = gb + ebf;
            okey[pos] = kk[i];
            oidx[pos] = (int)e;
          }
          ++ebf;
        }
      }
      gt_base += gtot;
      eq_base += etot;
    }
    cta_sync();
    for (int i = t; i < k; i += kLT) {
      ck[i] = okey[i];
      ci[i] = oidx[i];
    }
    n = k;
  }
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + t; i < P; i += kLT) {  // pads sort last
    ck[i] = 0u;
    ci[i] = 0x7fffffff;
  }
  cta_sync();
  smem_bitonic(ck, ci, P);
  const double rd = 1.0 / (double)R;
  for (int r = t; r < k; r += kLT) {
    const int j = ci[r];
    float v = ld_f1(xr + j);  // the element itself (keeps -0.0)
    if constexpr (MODE == 0) v = out_md(v, M, rd);  // kernels.hpp:122
    vals[row * (long long)k + r] = v;
    idx[row * (long long)k + r] = (long long)j;
  }
}

__global__ void k_topk_large_offsets(int* off, long long rows, int k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= rows; i += (long long)gridDim.x * blockDim.x)
    off[i] = (int)(i * k);
}

template <int MODE>
__global__ void k_topk_large_out(const unsigned* __restrict__ skey, const int* __restrict__ sidx,
                                 const float* __restrict__ rowM, const float* __restrict__ rowR, long long rows, int k,
                                 float* __restrict__ vals, long long* __restrict__ idx) {
  const long long n = rows * (long long)k;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / k;
    float v = fkey_inv(skey[i]);
    if constexpr (MODE == 0) v = out_md(v, rowM[r], 1.0 / (double)rowR[r]);  // kernels.hpp:122
    vals[i] = v;
    idx[i] = sidx[i];
  }
}

size_t al256(size_t b) { return (b + 255) / 256 * 256; }

struct LargeLayout {
  size_t key_in, key_out, idx_in, idx_out, off, rm, rr, temp, temp_bytes, total;
};

LargeLayout large_layout(long long rows, int k) {
  LargeLayout L{};
  const size_t n = (size_t)rows * (size_t)k;
  size_t temp_bytes = 0;
  cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, temp_bytes, (const unsigned*)nullptr,
                                                     (unsigned*)nullptr, (const int*)nullptr, (int*)nullptr,
                                                     (int)n, (int)rows, (const int*)nullptr, (const int*)nullptr);
  size_t o = 0;
  L.key_in = o, o += al256(n * 4);
  L.key_out = o, o += al256(n * 4);
  L.idx_in = o, o += al256(n * 4);
  L.idx_out = o, o += al256(n * 4);
  L.off = o, o += al256((size_t)(rows + 1) * 4);
  L.rm = o, o += al256((size_t)rows * 4);
  L.rr = o, o += al256((size_t)rows * 4);
  L.temp = o, o += al256(temp_bytes);
  L.temp_bytes = temp_bytes;
  L.total = o;
  return L;
}

template <int MODE>
cudaError_t run_large(const float* x, long long ldx, long long rows, long long V, int k, float* vals, long long* idx,
                      void* ws, char* region, cudaStream_t st) {
  const LargeLayout L = large_layout(rows, k);
  if constexpr (MODE != 2) {
    if (k <= kFastK && osmx_host::tuning().large_fast) {
      auto kern = k_topk_large_fast<MODE>;
      const size_t smem = (2048 + 2 * (size_t)kFastCap) * 4;
      if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      kern<<<(unsigned)rows, kLT, smem, st>>>(x, ldx, V, k, vals, idx, reinterpret_cast<unsigned*>(region + L.key_in),
                                              reinterpret_cast<int*>(region + L.idx_in), ws);
      osmx_host::count_launch();
      return cudaGetLastError();
    }
  }
  unsigned* key_in = reinterpret_cast<unsigned*>(region + L.key_in);
  unsigned* key_out = reinterpret_cast<unsigned*>(region + L.key_out);
  int* idx_in = reinterpret_cast<int*>(region + L.idx_in);
  int* idx_out = reinterpret_cast<int*>(region + L.idx_out);
  int* off = reinterpret_cast<int*>(region + L.off);
  float* rm = reinterpret_cast<float*>(region + L.rm);
  float* rr = reinterpret_cast<float*>(region + L.rr);
  k_topk_large_select<MODE><<<(unsigned)rows, kLT, 0, st>>>(x, ldx, V, k, key_in, idx_in, rm, rr, ws);
  osmx_host::count_launch();
  const int ob = (int)std::min<long long>((rows + 256) / 256, 4096);
  k_topk_large_offsets<<<ob, 256, 0, st>>>(off, rows, k);
  osmx_host::count_launch();
  size_t tb = L.temp_bytes;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairsDescending(
      region + L.temp, tb, key_in, key_out, idx_in, idx_out, (int)(rows * k), (int)rows, off, off + 1, 0, 32, st);
  osmx_host::count_launch();
  if (e != cudaSuccess) return e;
  const long long n = rows * (long long)k;
  const int gb = (int)std::min<long long>((n + 255) / 256, 8LL * osmx_host::num_sms() * 8);
  k_topk_large_out<MODE><<<gb, 256, 0, st>>>(key_out, idx_out, rm, rr, rows, k, vals, idx);
  osmx_host::count_launch();
  return cudaGetLastError();
}

}  // namespace

namespace osmx_host {

size_t topk_large_ws(long long rows, long long V, int k) {
  (void)V;
  if (k <= kMaxK || rows < 1) return 0;
  return large_layout(rows, k).total;
}

bool topk_large_supported(long long rows, long long V, int k) {
  return V < (1LL << 31) && (long long)rows * k < (1LL << 31);
}

cudaError_t launch_topk_large(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                              float* vals, long long* idx, void* ws, void* region, cudaStream_t st) {
  char* r = static_cast<char*>(region);
  switch (mode) {
    case 0: return run_large<0>(x, ldx, rows, V, k, vals, idx, ws, r, st);
    case 1: return run_large<1>(x, ldx, rows, V, k, vals, idx, ws, r, st);
    case 2: return run_large<2>(x, ldx, rows, V, k, vals, idx, ws, r, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace osmx_host
