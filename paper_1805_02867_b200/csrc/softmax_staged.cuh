// softmax_staged.cuh -- TMA-staged, shared-memory-resident batched softmax
// (naive / safe / online) for rows that fit in shared memory.
//
// Same algorithms as softmax_impl.cuh (reference kernels.hpp:39-69), but
// each row crosses HBM exactly twice (one read, one write) with both streams
// overlapped across rows:
//
//   warp 0        producer: lane 0 copies whole rows into a D-slot
//                 shared-memory ring -- the 16-byte aligned body with one
//                 1-D bulk copy (cp.async.bulk, UBLKCP), the <= 3 + 3 head /
//                 tail elements with 4-byte cp.async -- completing on the
//                 slot's "full" mbarrier.  It runs up to D rows ahead.
//   warps 1..     NG consumer groups of GW warps; group g takes the CTA's
//                 rows g, g+NG, ...: every pass of the algorithm (online:
//                 (m, d) then scale; safe: max, sum, scale) reads the slot
//                 with LDS.128, the group merges with shuffles (+ a named
//                 barrier when GW > 1), and the scale pass stores y straight
//                 to global memory with 128-bit streaming stores.  The group
//                 then releases the slot ("empty" mbarrier).
//
// Row r is placed in its slot at float offset phase(r) = (address / 4) % 4,
// so slot float4 q holds row elements 4q - phase .. 4q + 3 - phase: every
// float4 of the slot is aligned both in shared memory and -- when y rows
// have x's alignment phase -- in global memory, and rows of any V or ld
// keep 128-bit accesses.  Out-of-row lanes of the first / last float4 are
// masked (-inf for reductions, not stored).
//
// Persistent: one CTA per SM, rows grid-strided; D * slot <= ~200 KB.
#pragma once

#include "common.cuh"
#include "internal.hpp"
#include "tma.cuh"

namespace {

using namespace osmx_dev;

__device__ __forceinline__ void cp_async_4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Arrive on `bar` once every cp.async this thread issued so far has landed
// (noinc: the arrival is one of the barrier's expected arrivals).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
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
  __device__ static MD md(MD s, float* sm, int bar_id, int lw) {
    s = md_group_reduce<32>(s);
    if constexpr (GW == 1) {
      return s;
    } else {
      if ((threadIdx.x & 31) == 0) {
        sm[lw] = s.m;
        sm[GW + lw] = s.d;
      }
      named_sync(bar_id, GW * 32);
      MD t = MD{sm[0], sm[GW]};
#pragma unroll
      for (int i = 1; i < GW; ++i) t = md_merge(t, MD{sm[i], sm[GW + i]});
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

// Shared-memory layout: [full D][empty D] mbarriers, group scratch, slots.
// Up to 64 slots and 31 consumer warps: a fixed 2 KB header.
constexpr int kStagedMaxD = 64;
__host__ __device__ inline size_t staged_scratch_off() { return (size_t)16 * kStagedMaxD; }
__host__ __device__ inline size_t staged_slots_off() { return 2048; }

// NG (runtime) consumer groups of GW warps; blockDim = 32 * (1 + GW * NG).
// Requires D >= NG: a group then never waits more than one phase ahead of a
// slot's mbarrier (its previous row, loaded before this one, is >= D rows
// back), so parity waits are unambiguous.
template <int GW, int ALG>
__global__ void __launch_bounds__(1024, 1)
    k_softmax_staged(const float* __restrict__ x, long long ldx, float* __restrict__ y, long long ldy,
                     long long rows, int V, int D, void* ws) {
  constexpr int GT = GW * 32;
  const int NG = (blockDim.x / 32 - 1) / GW;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + D;
  const int slotf = staged_slot_floats(V);
  float* slots = reinterpret_cast<float*>(smem + staged_slots_off());

  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&full[s], 2);    // expect_tx arrival + cp.async arrival
      mbar_init(&empty[s], GW);  // one arrival per consumer warp of the group
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (w == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      long long j = 0;
      for (long long row = blockIdx.x; row < rows; row += gridDim.x, ++j) {
        const int s = (int)(j % D);
        if (j >= D) mbar_wait(&empty[s], (uint32_t)(((j / D) - 1) & 1));
        const float* xr = x + row * ldx;
        const int phase = (int)((reinterpret_cast<uintptr_t>(xr) >> 2) & 3);
        int head = phase ? 4 - phase : 0;
        if (head > V) head = V;
        const int nvec = (V - head) >> 2;
        const int tail = V - head - 4 * nvec;
        float* sl = slots + (size_t)s * slotf + phase;  // sl[e] <- xr[e]
        for (int e = 0; e < head; ++e) cp_async_4(sl + e, xr + e);
        for (int e = V - tail; e < V; ++e) cp_async_4(sl + e, xr + e);
        cp_async_mbar_arrive(&full[s]);
        mbar_arrive_expect_tx(&full[s], (uint32_t)nvec * 16u);
        if (nvec > 0) tma_load_1d_nohint(sl + head, xr + head, (uint32_t)nvec * 16u, &full[s]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int g = (w - 1) / GW;   // group
  const int lw = (w - 1) % GW;  // warp within the group
  const int tg = lw * 32 + lane;
  const int bar_id = 1 + g;
  float* scr = reinterpret_cast<float*>(smem + staged_scratch_off()) + g * 4 * GW;  // 2*GW doubles
  double* scrd = reinterpret_cast<double*>(scr);

  long long j = g;
  for (long long row = blockIdx.x + (long long)g * gridDim.x; row < rows; row += (long long)NG * gridDim.x, j += NG) {
    const int s = (int)(j % D);
    mbar_wait(&full[s], (uint32_t)((j / D) & 1));
    const float* xr = x + row * ldx;
    float* yr = y + row * ldy;
    const int phase = (int)((reinterpret_cast<uintptr_t>(xr) >> 2) & 3);
    const int nq = (phase + V + 3) >> 2;
    const float4* sl4 = reinterpret_cast<const float4*>(slots + (size_t)s * slotf);
    // Slot float4 q holds elements 4q - phase .. 4q + 3 - phase.  Interior
    // float4s [qa, qb) are entirely inside the row and need no masking; the
    // <= 2 edge float4s (qe0 = 0 when phase > 0, qe1 = qb when the row ends
    // mid-float4) are masked, one thread each.
    const int qa = phase ? 1 : 0;
    const int qb = (phase + V) >> 2 > qa ? (phase + V) >> 2 : qa;
    const int qe0 = phase ? 0 : -1;
    const int qe1 = (qb < nq && qb != qe0) ? qb : -1;
    const int my_edge = tg == 0 ? qe0 : (tg == 1 ? qe1 : -1);
    auto masked = [&](int q, float fill) -> float4 {
      float4 v = sl4[q];
      const int e0 = 4 * q - phase;
      if (e0 + 0 < 0 || e0 + 0 >= V) v.x = fill;
      if (e0 + 1 < 0 || e0 + 1 >= V) v.y = fill;
      if (e0 + 2 < 0 || e0 + 2 >= V) v.z = fill;
      if (e0 + 3 < 0 || e0 + 3 >= V) v.w = fill;
      return v;
    };
    auto min4 = [](float a, const float4& v) { return fminf(fminf(a, fminf(v.x, v.y)), fminf(v.z, v.w)); };
    auto max4 = [](float a, const float4& v) { return fmaxf(fmaxf(a, fmaxf(v.x, v.y)), fmaxf(v.z, v.w)); };

    float M = 0.0f, r = 0.0f;
    double rd = 0.0;
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
      for (; q < qb; q += GT) {
        float4 v[1] = {sl4[q]};
        mn = min4(mn, v[0]);
        acc.raise(max4(kNegInf, v[0]));
        acc.add_batch<1>(v);
      }
      if (my_edge >= 0) {
        float4 v[1] = {masked(my_edge, kNegInf)};
        mn = min4(mn, masked(my_edge, -kNegInf));
        const float bm = max4(kNegInf, v[0]);
        acc.raise(bm);
        if (bm != kNegInf) acc.add_batch<1>(v);
      }
      const MD tot = SGrp<GW>::md(acc.finish(), scr, bar_id, lw);
      mn = SGrp<GW>::red(mn, SOpMin(), scr, bar_id, lw);
      M = tot.m;
      r = __frcp_rn(tot.d);
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
        const float4 v = masked(my_edge, kNegInf);
        m = max4(m, v);
        mn = min4(mn, masked(my_edge, -kNegInf));
        const float4 z = masked(my_edge, 0.0f);  // out-of-row lanes must not poison chk
        chk = fmaf(z.x, 0.0f, fmaf(z.y, 0.0f, fmaf(z.z, 0.0f, fmaf(z.w, 0.0f, chk))));
      }
      if (!(chk == chk)) mn = kNegInf;  // -inf survives the fminf group reduce (NaN would not)
      M = SGrp<GW>::red(m, SOpMax(), scr, bar_id, lw);
      mn = SGrp<GW>::red(mn, SOpMin(), scr, bar_id, lw);
      L2Acc sacc;
      sacc.raise(M);
      for (int q = qa + tg; q < qb; q += GT) {
        float4 v[1] = {sl4[q]};
        sacc.add_batch<1>(v);
      }
      if (my_edge >= 0) {
        float4 v[1] = {masked(my_edge, kNegInf)};
        sacc.add_batch<1>(v);
      }
      float d = (M == kNegInf) ? 0.0f : sacc.finish().d;
      d = SGrp<GW>::red(d, SOpSum(), scr, bar_id, lw);
      r = __frcp_rn(d);
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
      rd = 1.0 / d;
      bad = !(d == d) || !isfinite(mx) || mn == kNegInf;
    }
    if (bad && tg == 0) flag_bad_row(ws, row);

    // Final pass: y = e^(x - m) / d (kernels.hpp:57 / :68; naive :45).
    auto f = [&](float v) -> float {
      if constexpr (ALG == osmx_host::kNaive)
        return (float)((double)expf(v) * rd);
      else
        return expf(v - M) * r;
    };
    const bool same_phase = ((reinterpret_cast<uintptr_t>(yr) >> 2) & 3) == (uintptr_t)phase;
    float* yb = yr - phase;  // yb[4q + c] <-> slot float4 q component c
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
      const float4 v = sl4[my_edge];
      const int e0 = 4 * my_edge - phase;
      if (e0 + 0 >= 0 && e0 + 0 < V) st_f1(yr + e0 + 0, f(v.x));
      if (e0 + 1 >= 0 && e0 + 1 < V) st_f1(yr + e0 + 1, f(v.y));
      if (e0 + 2 >= 0 && e0 + 2 < V) st_f1(yr + e0 + 2, f(v.z));
      if (e0 + 3 >= 0 && e0 + 3 < V) st_f1(yr + e0 + 3, f(v.w));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Largest dynamic shared memory the staged kernels use per CTA.
constexpr int kStagedSmemMax = 227 * 1024;

template <int GW, int ALG>
cudaError_t run_staged_cfg(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                           void* ws, cudaStream_t st, int ng, int ring_kb) {
  const auto& tn = osmx_host::tuning();
  if (tn.staged_kb > 0) ring_kb = tn.staged_kb;
  if (tn.staged_ng > 0) ng = tn.staged_ng;
  const size_t slot = (size_t)staged_slot_floats(V) * 4;
  const size_t ring = std::min<size_t>((size_t)ring_kb * 1024, kStagedSmemMax) - staged_slots_off();
  int D = (int)std::min<size_t>(ring / slot, kStagedMaxD);
  ng = std::min(ng, std::min(D, 31 / GW));
  if (ng < 1) return cudaErrorInvalidValue;
  const int ctas_per_sm = std::max(1, (228 * 1024) / (ring_kb * 1024 + 1024));
  const size_t smem = staged_slots_off() + (size_t)D * slot;
  static bool attr_set = false;  // per instantiation; the attribute is per function
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_softmax_staged<GW, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kStagedSmemMax);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const long long grid = std::min<long long>(rows, (long long)osmx_host::num_sms() * ctas_per_sm);
  k_softmax_staged<GW, ALG><<<(unsigned)grid, 32 * (1 + GW * ng), smem, st>>>(x, ldx, y, ldy, rows, (int)V, D, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

// Largest V served by the staged family (3 slots of a 200 KB ring).
constexpr long long kStagedMaxV = 16384;

template <int ALG>
cudaError_t run_staged(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                       void* ws, cudaStream_t st) {
  // Group width (warps per row) and group count per V, from
  // tools/shape_sweep.py on B200 (4000 and 32768 rows, gw x ng grid,
  // profiles/r01s2_staged_sweep.md): 2-warp groups x 6 up to V = 4096,
  // 4-warp groups x 6 up to 8192, x 3 above; at least one slot stays in
  // flight (ng <= D - 1), which matters once only 3-5 rows fit the ring.
  int gw = osmx_host::tuning().staged_gw;
  const int kb = 220;
  if (gw == 0) gw = V <= 1024 ? 1 : V <= 4096 ? 2 : 4;
  int ng = gw == 1 ? 16 : V <= 8192 ? 6 : 3;
  {
    const size_t slot = (size_t)staged_slot_floats(V) * 4;
    const int D = (int)std::min<size_t>((size_t)(kb * 1024 - staged_slots_off()) / slot, kStagedMaxD);
    if (D >= 2) ng = std::min(ng, D - 1);
  }
  switch (gw) {
    case 1: return run_staged_cfg<1, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb);
    case 2: return run_staged_cfg<2, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb);
    case 4: return run_staged_cfg<4, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb);
    case 8: return run_staged_cfg<8, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb);
    default: return run_staged_cfg<16, ALG>(x, ldx, y, ldy, rows, V, ws, st, ng, kb);
  }
}

}  // namespace
