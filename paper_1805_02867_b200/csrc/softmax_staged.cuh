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
__host__ __device__ inline size_t staged_scratch_off(int D) { return (size_t)16 * D; }
template <int NG, int GW>
__host__ __device__ inline size_t staged_slots_off(int D) {
  return (staged_scratch_off(D) + (size_t)NG * 2 * GW * 8 + 127) / 128 * 128;
}

template <int GW, int NG, int ALG>
__global__ void __launch_bounds__(32 * (1 + GW * NG), 1)
    k_softmax_staged(const float* __restrict__ x, long long ldx, float* __restrict__ y, long long ldy,
                     long long rows, int V, int D, void* ws) {
  constexpr int GT = GW * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + D;
  const int slotf = staged_slot_floats(V);
  float* slots = reinterpret_cast<float*>(smem + staged_slots_off<NG, GW>(D));

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
  float* scr = reinterpret_cast<float*>(smem + staged_scratch_off(D)) + g * 4 * GW;  // 2*GW doubles
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
    // element index of component 0 of slot float4 q is 4q - phase
    auto masked = [&](int q) -> float4 {
      float4 v = sl4[q];
      const int e0 = 4 * q - phase;
      if (e0 < 0 || e0 + 4 > V) {
        if (e0 + 0 < 0 || e0 + 0 >= V) v.x = kNegInf;
        if (e0 + 1 < 0 || e0 + 1 >= V) v.y = kNegInf;
        if (e0 + 2 < 0 || e0 + 2 >= V) v.z = kNegInf;
        if (e0 + 3 < 0 || e0 + 3 >= V) v.w = kNegInf;
      }
      return v;
    };
    // min over the row's real elements (-inf detection); masked lanes -> +inf
    auto vmin = [&](float4 v, int q) -> float {
      const int e0 = 4 * q - phase;
      float a = (e0 + 0 >= 0 && e0 + 0 < V) ? v.x : -kNegInf;
      float b = (e0 + 1 >= 0 && e0 + 1 < V) ? v.y : -kNegInf;
      float c = (e0 + 2 >= 0 && e0 + 2 < V) ? v.z : -kNegInf;
      float d = (e0 + 3 >= 0 && e0 + 3 < V) ? v.w : -kNegInf;
      return fminf(fminf(a, b), fminf(c, d));
    };

    float M = 0.0f, r = 0.0f;
    double rd = 0.0;
    bool bad;
    float mn = -kNegInf;
    if constexpr (ALG == osmx_host::kOnline) {
      // Alg. 3 lines 1-6: per thread, batch max first then one rescale.
      L2Acc acc;
      constexpr int U = 4;
      int q = tg;
      for (; q + (U - 1) * GT < nq; q += U * GT) {
        float4 v[U];
        float bm = kNegInf;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          v[u] = masked(q + u * GT);
          mn = fminf(mn, vmin(v[u], q + u * GT));
          bm = fmaxf(bm, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
        }
        acc.raise(bm);
        if (bm != kNegInf) acc.add_batch<U>(v);
      }
      for (; q < nq; q += GT) {
        float4 v[1] = {masked(q)};
        mn = fminf(mn, vmin(v[0], q));
        const float bm = fmaxf(fmaxf(v[0].x, v[0].y), fmaxf(v[0].z, v[0].w));
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
      float m = kNegInf;
      for (int q = tg; q < nq; q += GT) {
        const float4 v = masked(q);
        mn = fminf(mn, vmin(v, q));
        m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        if (!(v.x == v.x && v.y == v.y && v.z == v.z && v.w == v.w)) mn = __int_as_float(0x7fffffff);
      }
      M = SGrp<GW>::red(m, SOpMax(), scr, bar_id, lw);
      mn = SGrp<GW>::red(mn, SOpMin(), scr, bar_id, lw);
      L2Acc sacc;
      sacc.raise(M);
      for (int q = tg; q < nq; q += GT) {
        float4 v[1] = {masked(q)};
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
      for (int q = tg; q < nq; q += GT) {
        const float4 v = masked(q);
        mn = fminf(mn, vmin(v, q));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
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
    for (int q = tg; q < nq; q += GT) {
      const float4 v = sl4[q];
      const float4 o = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
      const int e0 = 4 * q - phase;
      if (same_phase && e0 >= 0 && e0 + 4 <= V) {
        st_f4(yb + 4 * q, o);
      } else {
        if (e0 + 0 >= 0 && e0 + 0 < V) st_f1(yr + e0 + 0, o.x);
        if (e0 + 1 >= 0 && e0 + 1 < V) st_f1(yr + e0 + 1, o.y);
        if (e0 + 2 >= 0 && e0 + 2 < V) st_f1(yr + e0 + 2, o.z);
        if (e0 + 3 >= 0 && e0 + 3 < V) st_f1(yr + e0 + 3, o.w);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Largest dynamic shared memory the staged kernels use per CTA.
constexpr int kStagedSmem = 200 * 1024;

template <int GW, int NG, int ALG>
cudaError_t run_staged_cfg(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                           void* ws, cudaStream_t st) {
  const size_t slot = (size_t)staged_slot_floats(V) * 4;
  int D = (int)((kStagedSmem - 1024) / slot);
  D = D > 64 ? 64 : D;
  if (D < NG) return cudaErrorInvalidValue;
  const size_t smem = staged_slots_off<NG, GW>(D) + (size_t)D * slot;
  static bool attr_set = false;  // per instantiation; the attribute is per function
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_softmax_staged<GW, NG, ALG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kStagedSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const long long grid = std::min<long long>(rows, (long long)osmx_host::num_sms());
  k_softmax_staged<GW, NG, ALG><<<(unsigned)grid, 32 * (1 + GW * NG), smem, st>>>(x, ldx, y, ldy, rows, (int)V, D, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

// Largest V served by the staged family (3 slots of a 200 KB ring).
constexpr long long kStagedMaxV = 16384;

template <int ALG>
cudaError_t run_staged(const float* x, long long ldx, float* y, long long ldy, long long rows, long long V,
                       void* ws, cudaStream_t st) {
  if (V <= 1024) return run_staged_cfg<1, 16, ALG>(x, ldx, y, ldy, rows, V, ws, st);
  if (V <= 4096) return run_staged_cfg<2, 8, ALG>(x, ldx, y, ldy, rows, V, ws, st);
  if (V <= 8192) return run_staged_cfg<4, 4, ALG>(x, ldx, y, ldy, rows, V, ws, st);
  return run_staged_cfg<8, 2, ALG>(x, ldx, y, ldy, rows, V, ws, st);
}

}  // namespace
