// c5_lab.cu -- how fast can ONE launch read a 256 MB row (configs[4],
// V = 2^26 fp32) on this B200?  Pure-read kernels (max fold, no top-K) in
// several data-movement schemes, each launch on a cold buffer (4 x 256 MB
// rotation), CUDA-event timed, median of 30.
//   grid<U,B>   grid-stride LDG.128, U loads in flight per thread, B CTAs/SM
//   warp<U,B>   each warp owns one contiguous slice, lanes interleaved
//   tma<S,C,B>  each CTA owns one contiguous slice, S-stage ring of C-byte
//               1-D bulk copies (one producer lane), 8 consumer warps
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tools/c5_lab.cu -o build/c5_lab
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ float4 ldg4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float mx4(float4 v) { return fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)); }

template <int U>
__global__ void __launch_bounds__(256) k_grid(const float4* __restrict__ p, size_t n, float* out) {
  float m = -1e30f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg4(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) m = fmaxf(m, mx4(v[u]));
  }
  for (; i < n; i += stride) m = fmaxf(m, p[i].x);
  if (m == 12345.0f) *out = m;
}

template <int U>
__global__ void __launch_bounds__(256) k_warp(const float4* __restrict__ p, size_t n, float* out) {
  const size_t nw = (size_t)gridDim.x * 8, w = blockIdx.x * 8 + threadIdx.x / 32;
  const size_t per = (n + nw - 1) / nw;
  const size_t a = w * per, b = std::min(n, a + per);
  const int l = threadIdx.x & 31;
  float m = -1e30f;
  size_t i = a + l;
  for (; i + (U - 1) * 32 < b; i += U * 32) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg4(p + i + u * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) m = fmaxf(m, mx4(v[u]));
  }
  for (; i < b; i += 32) m = fmaxf(m, p[i].x);
  if (m == 12345.0f) *out = m;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int C>
__global__ void __launch_bounds__(288) k_tma(const float4* __restrict__ p, size_t n, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * C);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t per = ((n + gridDim.x - 1) / gridDim.x + (C / 16) - 1) / (C / 16) * (C / 16);
  const size_t a = blockIdx.x * per, b = std::min(n, a + per);
  const size_t bytes = b > a ? (b - a) * 16 : 0;
  const char* src = reinterpret_cast<const char*>(p + a);
  const int w = threadIdx.x / 32;
  if (w == 8) {
    if ((threadIdx.x & 31) == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (size_t off = 0; off < bytes; off += C) {
        const uint32_t nb = (uint32_t)std::min<size_t>(C, bytes - off);
        uint32_t done = 0;
        while (!done)
          asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                       : "=r"(done) : "r"(sa(&empty[s])), "r"(ph ^ 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(nb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + (size_t)s * C)), "l"(src + off), "r"(nb), "r"(sa(&full[s])) : "memory");
        if (++s == S) s = 0, ph ^= 1;
      }
    }
    return;
  }
  float m = -1e30f;
  int s = 0;
  uint32_t ph = 0;
  for (size_t off = 0; off < bytes; off += C) {
    const int n4 = (int)(std::min<size_t>(C, bytes - off) / 16);
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}"
                   : "=r"(done) : "r"(sa(&full[s])), "r"(ph) : "memory");
    const float4* sb = reinterpret_cast<const float4*>(sm + (size_t)s * C);
    for (int q = threadIdx.x; q < n4; q += 256) m = fmaxf(m, mx4(sb[q]));
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    if (++s == S) s = 0, ph ^= 1;
  }
  if (m == 12345.0f) *out = m;
}

int main() {
  const size_t bytes = 256ull << 20, n = bytes / 16;
  const int NB = 4;
  float4* buf[NB];
  float* o;
  for (int i = 0; i < NB; ++i) {
    CK(cudaMalloc(&buf[i], bytes));
    CK(cudaMemset(buf[i], 0, bytes));
  }
  CK(cudaMalloc(&o, 4));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    std::vector<float> ts;
    for (int r = 0; r < 34; ++r) {
      const float4* p = buf[r % NB];
      cudaEventRecord(e0);
      launch(p);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 4) ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    const float med = ts[ts.size() / 2];
    printf("%-28s %8.2f us  %7.1f GB/s  (min %.2f us)\n", name, med * 1e3, bytes / (med * 1e-3) / 1e9, ts[0] * 1e3);
  };
  for (int B : {2, 4, 8})
    for (int U : {4, 8, 16}) {
      char nm[64];
      snprintf(nm, sizeof nm, "grid U=%d B=%d", U, B);
      run(nm, [&](const float4* p) {
        if (U == 4) k_grid<4><<<sms * B, 256>>>(p, n, o);
        if (U == 8) k_grid<8><<<sms * B, 256>>>(p, n, o);
        if (U == 16) k_grid<16><<<sms * B, 256>>>(p, n, o);
      });
    }
  for (int B : {4, 8})
    for (int U : {4, 8, 16}) {
      char nm[64];
      snprintf(nm, sizeof nm, "warp U=%d B=%d", U, B);
      run(nm, [&](const float4* p) {
        if (U == 4) k_warp<4><<<sms * B, 256>>>(p, n, o);
        if (U == 8) k_warp<8><<<sms * B, 256>>>(p, n, o);
        if (U == 16) k_warp<16><<<sms * B, 256>>>(p, n, o);
      });
    }
  auto tma = [&](auto kern, int S, int C, int B, const char* nm) {
    const int smem = S * C + 2 * S * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run(nm, [&](const float4* p) { kern<<<sms * B, 288, smem>>>(p, n, o); });
  };
  tma(k_tma<4, 16384>, 4, 16384, 3, "tma S=4 C=16K B=3");
  tma(k_tma<6, 16384>, 6, 16384, 2, "tma S=6 C=16K B=2");
  tma(k_tma<12, 16384>, 12, 16384, 1, "tma S=12 C=16K B=1");
  tma(k_tma<6, 32768>, 6, 32768, 1, "tma S=6 C=32K B=1");
  tma(k_tma<3, 32768>, 3, 32768, 2, "tma S=3 C=32K B=2");
  tma(k_tma<8, 8192>, 8, 8192, 3, "tma S=8 C=8K B=3");
  tma(k_tma<2, 65536>, 2, 65536, 1, "tma S=2 C=64K B=1");
  tma(k_tma<3, 65536>, 3, 65536, 1, "tma S=3 C=64K B=1");
  return 0;
}
