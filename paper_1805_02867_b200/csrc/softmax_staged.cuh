// softmax_staged.cuh -- TMA-staged, shared-memory-resident batched softmax
// (naive / safe / online): every element crosses HBM exactly twice (one
// read, one write), both streams overlapped across rows.
//
// Same algorithms as softmax_impl.cuh (reference kernels.hpp:39-69).  A row
// is owned by a thread-block cluster of C CTAs (C = 1 for V <= 16K; up to 16
// for longer rows): CTA c of the cluster holds slice [c*Sv, (c+1)*Sv) of it
// (Sv a multiple of 4, so every slice keeps the row's 16-byte phase).
//
//   warp 0        producer: lane 0 copies the CTA's slice of each row into a
//                 D-slot shared-memory ring -- the 16-byte aligned body with
//                 one 1-D bulk copy (cp.async.bulk, UBLKCP) completing on the
//                 slot's "full" mbarrier; it runs up to D rows ahead.  The
//                 <= 3 + 3 edge elements are read from global memory by two
//                 consumer threads.
//   warps 1..     NG consumer groups of GW warps; group g takes the rows
//                 g, g+NG, ... of its cluster.  Every pass of the algorithm
//                 (online: (m, d) then scale; safe: max, sum, scale; naive:
//                 sum, scale) reads the slot with LDS.128; the group merges
//                 with shuffles (+ a named barrier when GW > 1).  With C > 1
//                 the group's 16-byte record goes to group g of every CTA of
//                 the cluster by st.async (distributed shared memory,
//                 completing on that CTA's record mbarrier -- no fence), and
//                 each CTA merges the C records in rank order, the
//                 reference's contiguous-chunk merge (normalizer.hpp:73-85);
//                 safe exchanges twice (max, then the sum against it).  The
//                 scale pass stores y straight to global memory with 128-bit
//                 streaming stores, then the group releases the slot.
//
// Slot layout: the slice is placed at float offset phase = (address/4) % 4,
// so slot float4 q holds slice elements 4q - phase .. 4q + 3 - phase; every
// interior float4 is aligned in shared and (when y has x's phase) global
// memory, whatever V and ld are.  The <= 2 edge float4s are masked.
//
// Ordering: D >= NG + 1 so a group never waits more than one phase ahead of
// a slot mbarrier; records are double-buffered per group by row parity --
// a peer writes a group's (k+2)-th record only after it has received this
// CTA's (k+1)-th, which this CTA sends after reading its k-th records.
#pragma once

#include "common.cuh"
#include "internal.hpp"
#include "tma.cuh"

namespace {

using namespace osmx_dev;

__device__ __forceinline__ void tma_load_1d_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Group-wide reductions: GW warps, named barrier `bar_id`, scratch `sm`
// (2 * GW floats / GW doubles, private to the group).
template <int GW>
struct SGrp {
  // (m, d) and the min together: one round of named barriers for both.
  __device__ static MD md_min(MD s, float& mn, float* sm, int bar_id, int lw) {
    s = md_group_reduce<32>(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if constexpr (GW == 1) {
      return s;
    } else {
      if ((threadIdx.x & 31) == 0) {
        sm[lw] = s.m;
        sm[GW + lw] = s.d;
        sm[2 * GW + lw] = mn;
      }
      named_sync(bar_id, GW * 32);
      MD t = MD{sm[0], sm[GW]};
      mn = sm[2 * GW];
#pragma unroll
      for (int i = 1; i < GW; ++i) {
        t = md_merge(t, MD{sm[i], sm[GW + i]});
        mn = fminf(mn, sm[2 * GW + i]);
      }
      named_sync(bar_id, GW * 32);
      return t;
    }
  }
  template <class T, class Op>
  __device__ static T red(T v, Op op, T* sm, int bar_id, int lw) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if constexpr (GW == 1) {
      return v;
    } else {
      if ((threadIdx.x & 31) == 0) sm[lw] = v;
      named_sync(bar_id, GW * 32);
      T t = sm[0];
#pragma unroll
      for (int i = 1; i < GW; ++i) t = op(t, sm[i]);
      named_sync(bar_id, GW * 32);
      return t;
    }
  }
};

struct SOpMax {
  __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};
struct SOpMin {
  __device__ float operator()(float a, float b) const { return fminf(a, b); }
};
struct SOpSum {
  __device__ float operator()(float a, float b) const { return a + b; }
};
struct SOpSumD {
  __device__ double operator()(double a, double b) const { return a + b; }
};

__host__ __device__ inline int staged_slot_floats(long long V) { return (int)((V + 3 + 3) / 4 * 4); }

struct SRecX {  // one slice's contribution, exchanged across the cluster (16 B)
  float m;      // max / running max
  float mn;     // min (-inf marks a non-finite element)
  double d;     // normalizer (naive: sum e^x; online: relative to m; safe round 1: relative to M)
};

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_count() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Asynchronous store of a record into CTA `rank`'s copy of `local`,
// completing 16 transaction bytes on that CTA's copy of `bar`.
__device__ __forceinline__ void st_async_rec(SRecX* local, uint64_t* bar, unsigned rank, const SRecX& r) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
  const unsigned long long db = (unsigned long long)__double_as_longlong(r.d);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
               "r"(__float_as_uint(r.m)), "r"(__float_as_uint(r.mn)), "r"((unsigned)(db & 0xffffffffu)),
               "r"((unsigned)(db >> 32)), "r"(rb)
               : "memory");
}

// Shared-memory layout (bytes):
//   0      full[64], empty[64] slot mbarriers
//   1024   record mbarriers [group][round][parity] (<= 31 groups)
//   2048   group reduce scratch (4 * GW floats per group)
//   2560   records [group][round][parity][C] (C > 1 only)
//   ...    slots (128-byte aligned)
constexpr int kStagedMaxD = 64;
__host__ __device__ inline size_t staged_recbar_off() { return 1024; }
__host__ __device__ inline size_t staged_scratch_off() { return 2048; }
__host__ __device__ inline size_t staged_recs_off() { return 2560; }
__host__ __device__ inline size_t staged_slots_off(int ng, int C) {
  const size_t recs = C > 1 ? (size_t)ng * 4 * C * sizeof(SRecX) : 0;
  return (staged_recs_off() + recs + 127) / 128 * 128;
}

// NG (runtime) consumer groups of GW warps; blockDim = 32 * (1 + GW * NG).
template <int GW, int ALG>
__global__ void __launch_bounds__(1024, 1)
    k_softmax_staged(const float* __restrict__ x, long long ldx, float* __restrict__ y, long long ldy,
                     long long rows, int V, int Sv, int D, void* ws) {
  constexpr int GT = GW * 32;
  const int NG = (blockDim.x / 32 - 1) / GW;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kStagedMaxD;
  uint64_t* recbar = reinterpret_cast<uint64_t*>(smem + staged_recbar_off());
  SRecX* recs = reinterpret_cast<SRecX*>(smem + staged_recs_off());
  const unsigned C = cl_size(), c = cl_rank();
  const long long ncl = cl_count(), cl = cl_id();
  const int slotf = staged_slot_floats(Sv);
  float* slots = reinterpret_cast<float*>(smem + staged_slots_off(NG, (int)C));
  const int s0 = (int)c * Sv;                                  // slice start (multiple of 4)
  const int n = V - s0 <= 0 ? 0 : (V - s0 < Sv ? V - s0 : Sv);  // slice length (may be 0)

  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&full[s], 1);    // the producer's expect_tx arrival
      mbar_init(&empty[s], GW);  // one arrival per consumer warp of the group
    }
    for (int b = 0; b < 4 * NG; ++b) mbar_init(&recbar[b], 1);  // local expect_tx; C x 16 B of st.async
    fence_mbar_init();
  }
  __syncthreads();
  if (C > 1) cl_sync();  // peers' barriers exist before any st.async reaches them

  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (w == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      long long j = 0;
      for (long long row = cl; row < rows; row += ncl, ++j) {
        const int s = (int)(j % D);
        if (j >= D) mbar_wait(&empty[s], (uint32_t)(((j / D) - 1) & 1));
        const float* xs = x + row * ldx + s0;
        const int phase = (int)((reinterpret_cast<uintptr_t>(xs) >> 2) & 3);
        int head = phase ? 4 - phase : 0;
        if (head > n) head = n;
        const int nvec = (n - head) >> 2;
        const int tail = n - head - 4 * nvec;
        float* sl = slots + (size_t)s * slotf + phase;  // sl[e] <- xs[e]
        (void)tail;  // the <= 3 + 3 edge elements are read from global memory by the consumers
        mbar_arrive_expect_tx(&full[s], (uint32_t)nvec * 16u);
        if (nvec > 0) tma_load_1d_nohint(sl + head, xs + head, (uint32_t)nvec * 16u, &full[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int g = (w - 1) / GW;   // group
    const int lw = (w - 1) % GW;  // warp within the group
    const int tg = lw * 32 + lane;
    const int bar_id = 1 + g;
    float* scr = reinterpret_cast<float*>(smem + staged_scratch_off()) + g * 4 * GW;  // 2*GW doubles
    double* scrd = reinterpret_cast<double*>(scr);

    long long j = g, k = 0;  // j: row sequence index in the cluster; k: this group's row count
    for (long long row = cl + (long long)g * ncl; row < rows; row += (long long)NG * ncl, j += NG, ++k) {
      const int s = (int)(j % D);
      const int par = (int)(k & 1);
      const float* xs = x + row * ldx + s0;
      float* ys = y + row * ldy + s0;
      const int phase = (int)((reinterpret_cast<uintptr_t>(xs) >> 2) & 3);
      const int nq = (phase + n + 3) >> 2;
      const float4* sl4 = reinterpret_cast<const float4*>(slots + (size_t)s * slotf);
      // Interior float4s [qa, qb) lie entirely inside the slice; the <= 2 edge
      // float4s (qe0 = 0 when phase > 0, qe1 = qb when the slice ends
      // mid-float4) are masked, one thread each.
      const int qa = phase ? 1 : 0;
      const int qb = (phase + n) >> 2 > qa ? (phase + n) >> 2 : qa;
      const int qe0 = (phase && n > 0) ? 0 : -1;
      const int qe1 = (qb < nq && qb != qe0) ? qb : -1;
      const int my_edge = tg == 0 ? qe0 : (tg == 1 ? qe1 : -1);
      // Edge float4s are not staged: their in-slice elements come from global
      // memory, loaded before the slot wait so the latency overlaps it.
      float4 ev = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (my_edge >= 0) {
        const int e0 = 4 * my_edge - phase;
        if (e0 + 0 >= 0 && e0 + 0 < n) ev.x = ld_f1(xs + e0 + 0);
        if (e0 + 1 >= 0 && e0 + 1 < n) ev.y = ld_f1(xs + e0 + 1);
        if (e0 + 2 >= 0 && e0 + 2 < n) ev.z = ld_f1(xs + e0 + 2);
        if (e0 + 3 >= 0 && e0 + 3 < n) ev.w = ld_f1(xs + e0 + 3);
      }
      mbar_wait(&full[s], (uint32_t)((j / D) & 1));
      auto masked = [&](int q, float fill) -> float4 {
        const int e0 = 4 * q - phase;
        float4 v;
        v.x = (e0 + 0 < 0 || e0 + 0 >= n) ? fill : ev.x;
        v.y = (e0 + 1 < 0 || e0 + 1 >= n) ? fill : ev.y;
        v.z = (e0 + 2 < 0 || e0 + 2 >= n) ? fill : ev.z;
        v.w = (e0 + 3 < 0 || e0 + 3 >= n) ? fill : ev.w;
        return v;
      };
      auto min4 = [](float a, const float4& v) { return fminf(fminf(a, fminf(v.x, v.y)), fminf(v.z, v.w)); };
      auto max4 = [](float a, const float4& v) { return fmaxf(fmaxf(a, fmaxf(v.x, v.y)), fmaxf(v.z, v.w)); };
      // Cluster exchange, round r: send this group's record to group g of every
      // CTA, wait for the C records of this row; returns them (rank order).
      auto exchange = [&](int r, const SRecX& mine) -> const SRecX* {
        const int b = (g * 2 + r) * 2 + par;
        SRecX* buf = recs + (size_t)b * C;
        if (tg == 0) {
          mbar_arrive_expect_tx(&recbar[b], 16u * C);
          for (unsigned q = 0; q < C; ++q) st_async_rec(&buf[c], &recbar[b], q, mine);
        }
        mbar_wait(&recbar[b], (uint32_t)((k >> 1) & 1));
        return buf;
      };

      float M = 0.0f;
      double rd = 0.0;
      Recip rc{0.0f, 0.0f};  // safe / online: 1/d as hi + lo
      bool bad;
      float mn = -kNegInf;
      if constexpr (ALG == osmx_host::kOnline) {
        // Alg. 3 lines 1-6: per thread, batch max first then one rescale.
        L2Acc acc;
        constexpr int U = 4;
        int q = qa + tg;
        for (; q + (U - 1) * GT < qb; q += U * GT) {
          float4 v[U];
          float bm = kNegInf;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            v[u] = sl4[q + u * GT];
            mn = min4(mn, v[u]);
            bm = max4(bm, v[u]);
          }
          acc.raise(bm);
          acc.add_batch<U>(v);
        }
        if (q < qb) {
          // last partial batch as one masked batch (one raise): the -inf fill
          // adds e^-inf = 0 terms (every batch is added: a NaN must poison d
          // even when the batch max, which fmaxf takes past NaN, is -inf)
          float4 v[U];
          float bm = kNegInf;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (q + u * GT < qb) {
              v[u] = sl4[q + u * GT];
              mn = min4(mn, v[u]);
            } else {
              v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
            }
            bm = max4(bm, v[u]);
          }
          acc.raise(bm);
          acc.add_batch<U>(v);
        }
        if (my_edge >= 0) {
          float4 v[1] = {masked(my_edge, kNegInf)};
          mn = min4(mn, masked(my_edge, -kNegInf));
          // always added: a NaN edge element must poison d (max4 and min4
          // both step past NaN); an all -inf batch on an empty accumulator
          // poisons it too, and such a row is non-finite anyway
          acc.raise(max4(kNegInf, v[0]));
          acc.add_batch<1>(v);
        }
        MD tot = SGrp<GW>::md_min(acc.finish(), mn, scr, bar_id, lw);
        if (C > 1) {
          const SRecX* rec = exchange(0, SRecX{tot.m, mn, (double)tot.d});
          tot = md_identity();
          mn = -kNegInf;
          for (unsigned q = 0; q < C; ++q) {
            tot = md_merge(tot, MD{rec[q].m, (float)rec[q].d});
            mn = fminf(mn, rec[q].mn);
          }
        }
        M = tot.m;
        rc = recip_of((double)tot.d);
        bad = !(tot.d == tot.d) || !isfinite(M) || mn == kNegInf;
      } else if constexpr (ALG == osmx_host::kSafe) {
        // kernels.hpp:54 max, :56 sum against it
        float m = kNegInf, chk = 0.0f;
        for (int q = qa + tg; q < qb; q += GT) {
          const float4 v = sl4[q];
          mn = min4(mn, v);
          m = max4(m, v);
          chk = fmaf(v.x, 0.0f, fmaf(v.y, 0.0f, fmaf(v.z, 0.0f, fmaf(v.w, 0.0f, chk))));  // NaN iff inf/NaN
        }
        if (my_edge >= 0) {
          m = max4(m, masked(my_edge, kNegInf));
          mn = min4(mn, masked(my_edge, -kNegInf));
          const float4 z = masked(my_edge, 0.0f);  // out-of-slice lanes must not poison chk
          chk = fmaf(z.x, 0.0f, fmaf(z.y, 0.0f, fmaf(z.z, 0.0f, fmaf(z.w, 0.0f, chk))));
        }
        if (!(chk == chk)) mn = kNegInf;  // -inf survives the fminf group reduce (NaN would not)
        M = SGrp<GW>::red(m, SOpMax(), scr, bar_id, lw);
        mn = SGrp<GW>::red(mn, SOpMin(), scr, bar_id, lw);
        if (C > 1) {
          const SRecX* rec = exchange(0, SRecX{M, mn, 0.0});
          M = kNegInf;
          mn = -kNegInf;
          for (unsigned q = 0; q < C; ++q) {
            M = fmaxf(M, rec[q].m);
            mn = fminf(mn, rec[q].mn);
          }
        }
        SafeAcc sacc;
        sacc.raise(M);
        for (int q = qa + tg; q < qb; q += GT) {
          float4 v[1] = {sl4[q]};
          sacc.add_batch<1>(v);
        }
        if (my_edge >= 0) {
          float4 v[1] = {masked(my_edge, kNegInf)};
          sacc.add_batch<1>(v);
        }
        double d = (M == kNegInf) ? 0.0 : sacc.d;
        d = SGrp<GW>::red(d, SOpSumD(), scrd, bar_id, lw);
        if (C > 1) {
          const SRecX* rec = exchange(1, SRecX{M, mn, d});
          d = 0.0;
          for (unsigned q = 0; q < C; ++q) d += rec[q].d;
        }
        rc = recip_of(d);
        bad = !(d == d) || !isfinite(M) || !(mn == mn) || mn == kNegInf;
      } else {
        // naive: d = sum double(expf(x)) (kernels.hpp:43-44), no max shift
        double d = 0.0;
        float mx = kNegInf;
        for (int q = qa + tg; q < qb; q += GT) {
          const float4 v = sl4[q];
          mn = min4(mn, v);
          mx = max4(mx, v);
          d += ((double)expf(v.x) + (double)expf(v.y)) + ((double)expf(v.z) + (double)expf(v.w));
        }
        if (my_edge >= 0) {
          const float4 v = masked(my_edge, kNegInf);  // expf(-inf) = 0
          mn = min4(mn, masked(my_edge, -kNegInf));
          mx = max4(mx, v);
          d += ((double)expf(v.x) + (double)expf(v.y)) + ((double)expf(v.z) + (double)expf(v.w));
        }
        d = SGrp<GW>::red(d, SOpSumD(), scrd, bar_id, lw);
        mx = SGrp<GW>::red(mx, SOpMax(), scr, bar_id, lw);
        mn = SGrp<GW>::red(mn, SOpMin(), scr, bar_id, lw);
        if (C > 1) {
          const SRecX* rec = exchange(0, SRecX{mx, mn, d});
          d = 0.0;
          mx = kNegInf;
          mn = -kNegInf;
          for (unsigned q = 0; q < C; ++q) {
            d += rec[q].d;
            mx = fmaxf(mx, rec[q].m);
            mn = fminf(mn, rec[q].mn);
          }
        }
        rd = 1.0 / d;
        bad = !(d == d) || !isfinite(mx) || mn == kNegInf;
      }
      if (bad && tg == 0 && c == 0) flag_bad_row(ws, row);

      // Final pass: y = e^(x - m) / d (kernels.hpp:57 / :68; naive :45).
      auto f = [&](float v) -> float {
        if constexpr (ALG == osmx_host::kNaive)
          return (float)((double)expf(v) * rd);
        else
          return out_soft<ALG == osmx_host::kSafe>(v, M, rc);
      };
      const bool same_phase = ((reinterpret_cast<uintptr_t>(ys) >> 2) & 3) == (uintptr_t)phase;
      float* yb = ys - phase;  // yb[4q + c] <-> slot float4 q component c
      if (same_phase) {
        constexpr int U2 = 4;
        int q = qa + tg;
        for (; q + (U2 - 1) * GT < qb; q += U2 * GT) {
          float4 v[U2];
#pragma unroll
          for (int u = 0; u < U2; ++u) v[u] = sl4[q + u * GT];
#pragma unroll
          for (int u = 0; u < U2; ++u)
            st_f4(yb + 4 * (q + u * GT), make_float4(f(v[u].x), f(v[u].y), f(v[u].z), f(v[u].w)));
        }
        for (; q < qb; q += GT) {
          const float4 v = sl4[q];
          st_f4(yb + 4 * q, make_float4(f(v.x), f(v.y), f(v.z), f(v.w)));
        }
      } else {
        for (int q = qa + tg; q < qb; q += GT) {
          const float4 v = sl4[q];
          float* d = yb + 4 * q;
          st_f1(d + 0, f(v.x));
          st_f1(d + 1, f(v.y));
          st_f1(d + 2, f(v.z));
          st_f1(d + 3, f(v.w));
        }
      }
      if (my_edge >= 0) {
        const float4 v = masked(my_edge, 0.0f);
        const int e0 = 4 * my_edge - phase;
        if (e0 + 0 >= 0 && e0 + 0 < n) st_f1(ys + e0 + 0, f(v.x));
        if (e0 + 1 >= 0 && e0 + 1 < n) st_f1(ys + e0 + 1, f(v.y));
        if (e0 + 2 >= 0 && e0 + 2 < n) st_f1(ys + e0 + 2, f(v.z));
        if (e0 + 3 >= 0 && e0 + 3 < n) st_f1(ys + e0 + 3, f(v.w));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncwarp();          // reconverge warp 0 (lane 0 ran the producer loop)
  if (C > 1) cl_sync();  // no CTA exits while a peer may still st.async into it
}

constexpr int kStagedSmemMax = 227 * 1024;
constexpr long long kStagedMaxV = 16384;   // one CTA per row up to here
constexpr long long kClusterSlice = 12288;  // slice per CTA of a 16-CTA cluster
// Cluster sizes that tile the B200's 18-SM GPCs (2, 3, 4, 6, 9) keep up to
// 144 SMs busy; a 16-CTA cluster fits once per GPC (112 SMs).  From
// tools/shape_sweep.py (4000 rows, cluster size x group width,
// profiles/r01s2_cluster_sweep.md): short slices (<= 7680 elements, 4-warp
// groups) on the smallest such cluster up to 9 x 7680; then 6 or 9 CTAs with
// 8-warp groups while the slice leaves three ring slots (150000: 0.80 vs 1.11
// ms at 16 CTAs; two slots: 165888 at 9 CTAs 1.35 ms); 16 CTAs above
// (177828: 1.19 vs 1.46 ms at 9).  The fp64-heavy naive softmax streams
// above 10 x 12288.
constexpr long long kClusterShortSlice = 7680;
constexpr int kClusterRingKB = 220;
constexpr long long kClusterMaxV = 16 * kClusterSlice;
template <int ALG>
constexpr long long cluster_max_v() {
  return ALG == osmx_host::kNaive ? 10 * kClusterSlice : 16 * kClusterSlice;
}

// Launch one (GW, NG, C) layout.  NG is clamped so that D >= NG + 1.
template <int GW, int ALG>
cudaError_t run_staged_cfg(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                           void* ws, cudaStream_t st, int ng, int ring_kb, int C) {
  const auto& tn = osmx_host::tuning();
  if (tn.staged_kb > 0) ring_kb = tn.staged_kb;
  if (tn.staged_ng > 0) ng = tn.staged_ng;
  const int Sv = (int)(((V + C - 1) / C + 3) / 4 * 4);
  const size_t slot = (size_t)staged_slot_floats(Sv) * 4;
  ng = std::min(ng, 31 / GW);
  int D = 0;
  // Ring depth vs groups of >= 4 warps: D >= NG + 2 once the ring has >= 5
  // slots.  With 4-warp groups, (D, NG) = (5, 4), (6, 5), (7, 6), (8, 7) and
  // once (7, 5) hung or faulted about once in 10^3-10^4 graph-replayed
  // launches on B200 (tools/runs/r2_aq.sh, r2_ar.sh, r2_at.sh: 4000 rows at
  // V = 7000-10000, including the previous defaults at 6500 < V <= 8192),
  // while (4, 3), (5, 3) and every 1- and 2-warp-group layout (e.g. (7, 6)
  // at V = 3162, thousands of sweep launches) ran clean.  The cause is not
  // understood -- the slot protocol (one full / one empty mbarrier per slot,
  // a group never more than one phase behind) checks out on paper, the
  // sanitizers are clean, and non-.aligned named barriers did not cure it
  // ((7, 6) still failed 1 run in 6 with the guard compiled out,
  // tools/runs/r2_bf.sh) -- so the defaults use 4-warp groups only with 3
  // groups (run_staged) and this guard covers the knobs.
  for (int it = 0; it < 3; ++it) {  // ng and the header size depend on each other (C > 1)
    const size_t avail = (size_t)std::min(ring_kb * 1024, kStagedSmemMax) - staged_slots_off(ng, C);
    D = (int)std::min<size_t>(avail / slot, kStagedMaxD);
    if (D >= 5 && GW >= 4) ng = std::min(ng, D - 2);
    else if (D >= 2) ng = std::min(ng, D - 1);
  }
  // One-CTA rows above 8K elements: no deeper than NG + 1 = 4 slots (4000 x
  // 10000: 0.0527 vs 0.0551 ms with 5 slots, tools/runs/r2_as.sh).
  if (C == 1 && Sv > 8192 && tn.staged_kb == 0) D = std::min(D, ng + 1);
  if (D < 1 || ng < 1 || D < ng) return cudaErrorInvalidValue;
  const size_t smem = staged_slots_off(ng, C) + (size_t)D * slot;
  auto kern = k_softmax_staged<GW, ALG>;
  if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kStagedSmemMax);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(32 * (1 + GW * ng));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;  // a plain launch without a cluster
  long long ncl;
  if (C == 1) {
    // resident CTAs per SM from registers, threads and shared memory together
    // (a smem-only estimate over-subscribes when registers allow fewer, and
    // the grid-strided rows of the second wave then start late)
    int ctas_per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, 32 * (1 + GW * ng), smem);
    ctas_per_sm = std::max(1, ctas_per_sm);
    ncl = std::min<long long>(rows, (long long)osmx_host::num_sms() * ctas_per_sm);
  } else {
    cfg.gridDim = dim3((unsigned)(C * osmx_host::num_sms()));
    int max_clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (max_clusters < 1) return cudaErrorInvalidConfiguration;
    ncl = std::min<long long>(rows, max_clusters);
  }
  cfg.gridDim = dim3((unsigned)(ncl * C));
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, x, ldx, y, ldy, rows, (int)V, Sv, D, ws);
  osmx_host::count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Cluster size for a row of V elements (1 up to kStagedMaxV).
inline int staged_cluster_size(long long V) {
  const int forced = osmx_host::tuning().cluster_size;
  if (forced > 0) return forced;
  if (V <= kStagedMaxV) return 1;
  for (int c : {2, 3, 4, 6, 9})
    if (V <= c * kClusterShortSlice) return c;
  for (int c : {6, 9}) {
    const size_t slot = (size_t)staged_slot_floats(((V + c - 1) / c + 3) / 4 * 4) * 4;
    if (staged_slots_off(3, c) + 3 * slot <= (size_t)kClusterRingKB * 1024) return c;
  }
  return 16;
}

template <int ALG>
cudaError_t run_staged(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                       void* ws, cudaStream_t st) {
  // Group width (warps per slice) and group count per slice length, from
  // tools/shape_sweep.py on B200 (4000 and 32768 rows, gw x ng grid,
  // profiles/r01s2_staged_sweep.md): 2-warp groups x 6 up to 4096, 4-warp
  // groups x 6 up to 8192, x 3 above; at least one slot stays in flight.
  const int C = staged_cluster_size(V);
  const long long Sv = (V + C - 1) / C;
  int gw = osmx_host::tuning().staged_gw;
  // two 100 KB CTAs per SM for short rows (4000 rows: 1778 -> 0.0156 vs 0.0205
  // ms, 3162 -> 0.0207 vs 0.0241), one 220 KB ring above
  const int kb = (C == 1 && Sv <= 4096) ? 100 : kClusterRingKB;
  // 4-warp groups only with <= 3 groups: six 4-warp groups (slices of
  // 4K-8K elements) hung or faulted now and then on B200 under long graph
  // replays (see run_staged_cfg); six 2-warp groups, the layout of the
  // shorter rows, run clean and as fast (4000 x 5623: 0.0316 vs 0.0312 ms).
  if (gw == 0) gw = Sv <= 1024 ? 1 : Sv <= 8192 ? 2 : (C > 1 && Sv > kClusterSlice) ? 8 : 4;
  const int ng = gw == 1 ? 16 : Sv <= 8192 ? 6 : 3;
  switch (gw) {
    case 1: return run_staged_cfg<1, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb, C);
    case 2: return run_staged_cfg<2, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb, C);
    case 4: return run_staged_cfg<4, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb, C);
    case 8: return run_staged_cfg<8, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb, C);
    default: return run_staged_cfg<16, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb, C);
  }
}

}  // namespace
