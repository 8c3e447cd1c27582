// stream.cuh -- coalesced, 128-bit, unrolled streaming of one row segment by
// a group of G threads (G = a sub-warp, a warp, or the whole CTA).
//
// A segment [p, p+n) is split into
//   head : 0..3 scalar elements up to the first 16-byte boundary,
//   body : nvec float4s, group-strided (thread t takes t, t+G, ...), U in
//          flight per thread,
//   tail : 0..3 scalar elements.
// Each thread therefore sees its own elements in strictly increasing index
// order (head < body < tail), which is what the strict-'>' top-K insertion
// needs to reproduce the reference's tie order (topk.hpp:34-44).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace osmx_dev {

struct Seg {
  const float* p;
  long long n;
  int head;        // scalar elements before the first aligned float4
  long long nvec;  // aligned float4s
  int tail;        // scalar elements after the body
};

__device__ __forceinline__ Seg make_seg(const float* p, long long n) {
  Seg s;
  s.p = p;
  s.n = n;
  const unsigned mis = static_cast<unsigned>(reinterpret_cast<uintptr_t>(p) & 15u);
  long long h = mis ? (16 - mis) >> 2 : 0;  // float* is 4-byte aligned
  if (h > n) h = n;
  s.head = static_cast<int>(h);
  s.nvec = (n - h) >> 2;
  s.tail = static_cast<int>(n - h - 4 * s.nvec);
  return s;
}

// Bulk prefetch of [p, p + bytes) into L2 (no registers, no completion to
// wait for): p 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Element index of component c of body float4 q.
__device__ __forceinline__ long long body_index(const Seg& s, long long q, int c) {
  return s.head + 4 * q + c;
}

// Visit every element of the segment once:
//   f1(x, j)                    scalar element j
//   fb(v[U], q0, cnt)           cnt (<= U) float4s at body indices q0 + u*G
// LAST = 1 selects the evict-first load flavour (final read of the data),
// LAST = 2 the evict-last one (data re-read soon by the same CTA).
// pf > 0: thread 0 of the group keeps the group's body pf batches ahead in
// L2 with bulk prefetches, so the demand loads see L2 rather than DRAM
// latency without spending registers on more loads in flight.
template <int G, int U, int LAST, class F1, class FB>
__device__ __forceinline__ void stream_seg(const Seg& s, int t, F1&& f1, FB&& fb, int pf = 0) {
  auto L4 = [](const float* p) { return LAST == 1 ? ld_f4_last(p) : LAST == 2 ? ld_f4_keep(p) : ld_f4(p); };
  auto L1 = [](const float* p) { return LAST == 1 ? ld_f1_last(p) : LAST == 2 ? ld_f1_keep(p) : ld_f1(p); };
  if (t < s.head) f1(L1(s.p + t), (long long)t);
  const float* b = s.p + s.head;
  constexpr long long kB = (long long)U * G;  // float4s per batch of the group
  if (pf > 0 && t == 0 && s.nvec > 0) {
    const long long n = s.nvec < pf * kB ? s.nvec : pf * kB;
    prefetch_l2(b, (unsigned)(16 * n));
  }
  long long q = t;
  for (; q + (long long)(U - 1) * G < s.nvec; q += (long long)U * G) {
    if (pf > 0 && t == 0) {
      const long long qa = q + pf * kB;
      if (qa < s.nvec) prefetch_l2(b + 4 * qa, (unsigned)(16 * (s.nvec - qa < kB ? s.nvec - qa : kB)));
    }
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = L4(b + 4 * (q + (long long)u * G));
    fb(v, q, U);
  }
  if (q < s.nvec) {
    float4 v[U];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long qq = q + (long long)u * G;
      if (qq < s.nvec) {
        v[u] = L4(b + 4 * qq);
        cnt = u + 1;
      } else {
        v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      }
    }
    fb(v, q, cnt);
  }
  if (t < s.tail) {
    const long long j = s.head + 4 * s.nvec + t;
    f1(L1(s.p + j), j);
  }
}

// Same visit order as stream_seg for one warp (G = 32), but the body is
// software-pipelined through shared memory: each lane keeps NST - 1 batches
// of U float4s in flight with 16-byte cp.async (LDGSTS, L2 only) into its own
// slots of `wbuf` ([NST][U][32] float4s, private to the warp), so the loads
// of the next batches overlap the compute of this one without extra
// registers.  Each lane reads back only what it wrote: no barrier needed.
__device__ __forceinline__ void cp_async16(float4* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int U, int NST, class F1, class FB>
__device__ __forceinline__ void stream_seg_pipe(const Seg& s, int t, F1&& f1, FB&& fb, float4* wbuf) {
  if (t < s.head) f1(ld_f1(s.p + t), (long long)t);
  constexpr int kB = U * 32;                      // float4s per batch of the warp
  const int nvec = (int)s.nvec;                   // rows < 2^33 elements (host-checked)
  const int nfull = nvec / kB, nb = (nvec + kB - 1) / kB;
  const float* ip = s.p + s.head + 4 * t;         // this lane's float4 of the next batch to issue
  float4* const wl = wbuf + t;                    // this lane's slot of stage 0
  int issued = 0, is = 0;
  auto issue = [&]() {
    if (issued < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) cp_async16(wl + is * kB + u * 32, ip + u * 128);
    } else if (issued < nb) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (issued * kB + u * 32 + t < nvec) cp_async16(wl + is * kB + u * 32, ip + u * 128);
    }
    cp_async_commit();
    ip += 4 * kB;
    ++issued;
    is = is + 1 == NST ? 0 : is + 1;
  };
#pragma unroll
  for (int i = 0; i < NST - 1; ++i) issue();
  int cs = 0;
  for (int bi = 0; bi < nb; ++bi) {
    issue();
    cp_async_wait<NST - 1>();
    float4 v[U];
    int cnt = U;
    if (bi < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = wl[cs * kB + u * 32];
    } else {
      cnt = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (bi * kB + u * 32 + t < nvec) {
          v[u] = wl[cs * kB + u * 32];
          cnt = u + 1;
        } else {
          v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        }
      }
    }
    fb(v, (long long)(bi * kB + t), cnt);
    cs = cs + 1 == NST ? 0 : cs + 1;
  }
  if (t < s.tail) {
    const long long j = s.head + 4 * s.nvec + t;
    f1(ld_f1(s.p + j), j);
  }
}

// Same visit order as stream_seg (G threads, U float4s per batch per
// thread) with the body register-double-buffered: the loads of batch i+1 are
// issued before batch i is processed, so a warp keeps U float4s in flight
// while it computes instead of alternating load / compute (the one-wave
// regime where occupancy, not registers, limits the bytes in flight).
template <int G, int U, class F1, class FB>
__device__ __forceinline__ void stream_seg_db(const Seg& s, int t, F1&& f1, FB&& fb) {
  if (t < s.head) f1(ld_f1(s.p + t), (long long)t);
  const float* b = s.p + s.head;
  constexpr long long kB = (long long)U * G;
  const long long nfull = s.nvec / kB;  // full batches
  auto load = [&](float4 (&v)[U], long long bi) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_f4(b + 4 * (bi * kB + (long long)u * G + t));
  };
  float4 A[U], B[U];
  long long bi = 0;
  if (nfull > 0) load(A, 0);
  while (bi < nfull) {
    if (bi + 1 < nfull) load(B, bi + 1);
    fb(A, bi * kB + t, U);
    if (++bi >= nfull) break;
    if (bi + 1 < nfull) load(A, bi + 1);
    fb(B, bi * kB + t, U);
    ++bi;
  }
  // last partial batch
  const long long q0 = nfull * kB + t;
  if (nfull * kB < s.nvec) {
    float4 v[U];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long qq = q0 + (long long)u * G;
      if (qq < s.nvec) {
        v[u] = ld_f4(b + 4 * qq);
        cnt = u + 1;
      } else {
        v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      }
    }
    fb(v, q0, cnt);
  }
  if (t < s.tail) {
    const long long j = s.head + 4 * s.nvec + t;
    f1(ld_f1(s.p + j), j);
  }
}

// Same visit order as stream_seg for one warp (G = 32), the body streamed
// through a per-warp ring of NS shared-memory stages of U*32 float4s by 1-D
// bulk copies (cp.async.bulk, one instruction per 2 KB chunk, issued by lane
// 0, completing on the stage's mbarrier): NS chunks stay in flight without
// registers, and a chunk is refilled as soon as the warp has it in
// registers.  `g` is the warp's running chunk count (stage / parity across
// rows); ring = NS*U*32 float4s, bars = NS mbarriers, both private to the warp.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  unsigned done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

template <int U, int NS, class F1, class FB>
__device__ __forceinline__ void stream_seg_bulk(const Seg& s, int t, F1&& f1, FB&& fb, float4* ring, uint64_t* bars,
                                                long long& g) {
  if (t < s.head) f1(ld_f1(s.p + t), (long long)t);
  constexpr int kB = U * 32;  // float4s per chunk
  const long long nvec = s.nvec;
  const long long nch = (nvec + kB - 1) / kB;
  const float4* body = reinterpret_cast<const float4*>(s.p + s.head);
  const long long g0 = g;
  auto issue = [&](long long c) {  // lane 0: chunk c of this row into stage (g0 + c) % NS
    const int st = (int)((g0 + c) % NS);
    const long long q0 = c * kB;
    const unsigned bytes = (unsigned)(16 * (nvec - q0 < kB ? nvec - q0 : kB));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior reads of the stage before the async write
    bar_expect_tx(&bars[st], bytes);
    bulk_g2s(ring + st * kB, body + q0, bytes, &bars[st]);
  };
  if (t == 0)
    for (long long c = 0; c < nch && c < NS; ++c) issue(c);
  for (long long c = 0; c < nch; ++c) {
    const int st = (int)((g0 + c) % NS);
    bar_wait(&bars[st], (unsigned)(((g0 + c) / NS) & 1));
    const float4* sb = ring + st * kB;
    const long long q0 = c * kB + t;
    float4 v[U];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (q0 + u * 32 < nvec) {
        v[u] = sb[u * 32 + t];
        cnt = u + 1;
      } else {
        v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      }
    }
    __syncwarp();
    if (t == 0 && c + NS < nch) issue(c + NS);
    fb(v, q0, cnt);
  }
  g = g0 + nch;
  if (t < s.tail) {
    const long long j = s.head + 4 * s.nvec + t;
    f1(ld_f1(s.p + j), j);
  }
}

// Same traversal, writing one output per element (y has the same alignment
// phase as x only when ldx == ldy; the output pointer is aligned
// independently, falling back to scalar stores when phases differ).
//
// REV = true walks the body from its end: the final pass of a multi-pass
// kernel then starts with the lines the previous pass read last -- still in
// L2 when the row (or the grid's working set) is larger than L2.
template <int G, int U, class FMAP, bool REV = false>
__device__ __forceinline__ void map_seg(const Seg& s, float* __restrict__ y, int t, FMAP&& f,
                                        std::integral_constant<bool, REV> = {}) {
  const bool same_phase =
      ((reinterpret_cast<uintptr_t>(y) & 15u) == (reinterpret_cast<uintptr_t>(s.p) & 15u));
  if (t < s.head) st_f1(y + t, f(ld_f1_last(s.p + t)));
  const float* b = s.p + s.head;
  float* yb = y + s.head;
  if constexpr (REV) {
    // batches of U*G float4s from the last (possibly partial) one down
    constexpr long long kB = (long long)U * G;
    const long long nfull = s.nvec / kB;
    auto one = [&](long long q) {
      const float4 v = ld_f4_last(b + 4 * q);
      const float4 o = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
      float* dst = yb + 4 * q;
      if (same_phase) {
        st_f4(dst, o);
      } else {
        st_f1(dst, o.x);
        st_f1(dst + 1, o.y);
        st_f1(dst + 2, o.z);
        st_f1(dst + 3, o.w);
      }
    };
    for (long long q = nfull * kB + t; q < s.nvec; q += G) one(q);  // partial last batch
    for (long long bi = nfull - 1; bi >= 0; --bi) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_f4_last(b + 4 * (bi * kB + (long long)u * G + t));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long q = bi * kB + (long long)u * G + t;
        float4 o = make_float4(f(v[u].x), f(v[u].y), f(v[u].z), f(v[u].w));
        float* dst = yb + 4 * q;
        if (same_phase) {
          st_f4(dst, o);
        } else {
          st_f1(dst, o.x);
          st_f1(dst + 1, o.y);
          st_f1(dst + 2, o.z);
          st_f1(dst + 3, o.w);
        }
      }
    }
    if (t < s.tail) {
      const long long j = s.head + 4 * s.nvec + t;
      st_f1(y + j, f(ld_f1_last(s.p + j)));
    }
    return;
  }
  long long q = t;
  for (; q + (long long)(U - 1) * G < s.nvec; q += (long long)U * G) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_f4_last(b + 4 * (q + (long long)u * G));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 o = make_float4(f(v[u].x), f(v[u].y), f(v[u].z), f(v[u].w));
      float* dst = yb + 4 * (q + (long long)u * G);
      if (same_phase) {
        st_f4(dst, o);
      } else {
        st_f1(dst, o.x);
        st_f1(dst + 1, o.y);
        st_f1(dst + 2, o.z);
        st_f1(dst + 3, o.w);
      }
    }
  }
  for (; q < s.nvec; q += G) {
    float4 v = ld_f4_last(b + 4 * q);
    float4 o = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
    float* dst = yb + 4 * q;
    if (same_phase) {
      st_f4(dst, o);
    } else {
      st_f1(dst, o.x);
      st_f1(dst + 1, o.y);
      st_f1(dst + 2, o.z);
      st_f1(dst + 3, o.w);
    }
  }
  if (t < s.tail) {
    const long long j = s.head + 4 * s.nvec + t;
    st_f1(y + j, f(ld_f1_last(s.p + j)));
  }
}

}  // namespace osmx_dev
