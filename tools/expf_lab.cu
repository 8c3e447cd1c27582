// expf_lab.cu -- (1) how far is CUDA's expf from the reference's glibc expf
// (expf_ref, bit-exact replica) over every float in [-104, 88]; (2) what does
// the reference's output formula y = float(double(expf(x - m)) / d) cost in a
// streaming read+write pass, vs the fast y = expf(x - m) * rcp(d).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//      -Ipaper_1805_02867_b200/csrc tools/expf_lab.cu -o build/expf_lab
#include <algorithm>
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace osmx_dev;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k_ulps(unsigned lo, unsigned n, unsigned long long* hist, int* worst) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(lo + i);
    const float a = expf(x), b = expf_ref(x);
    int d = abs((int)__float_as_uint(a) - (int)__float_as_uint(b));
    atomicAdd(&hist[min(d, 7)], 1ULL);
    if (d) atomicMax(worst, d);
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_out(const float4* __restrict__ x, float4* __restrict__ y, size_t n, float m,
                                             float r, double rd) {
  __shared__ double tab[32];
  if (threadIdx.x < 32) tab[threadIdx.x] = __longlong_as_double((long long)kExpfTab[threadIdx.x]);
  __syncthreads();
  auto f = [&](float v) -> float {
    if (MODE == 0) return expf(v - m) * r;
    if (MODE == 1) return (float)((double)expf(v - m) * rd);
    // MODE 2: glibc expf with the table in shared memory, quotient in double
    const float xm = __fsub_rn(v, m);
    if (!(xm > -150.0f)) return 0.0f;
    const double z = __dmul_rn(0x1.71547652b82fep+5, (double)xm);
    double kd = __dadd_rn(z, 0x1.8p+52);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, 0x1.8p+52);
    const double rr = __dsub_rn(z, kd);
    const unsigned long long t = (unsigned long long)__double_as_longlong(tab[ki & 31]) + (ki << 47);
    const double sc = __longlong_as_double((long long)t);
    const double q = __fma_rn(0x1.c6af84b912394p-20, rr, 0x1.ebfce50fac4f3p-13);
    double yy = __fma_rn(0x1.62e42ff0c52d6p-6, rr, 1.0);
    yy = __fma_rn(q, __dmul_rn(rr, rr), yy);
    const float e = __double2float_rn(__dmul_rn(yy, sc));
    return __double2float_rn(__dmul_rn((double)e, rd));
  };
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    y[i] = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
  }
}

int main() {
  unsigned long long* hist;
  int* worst;
  CK(cudaMalloc(&hist, 8 * 8));
  CK(cudaMalloc(&worst, 4));
  CK(cudaMemset(hist, 0, 64));
  CK(cudaMemset(worst, 0, 4));
  // negative floats from -0 down to -104 (bit patterns 0x80000000..), and 0..88
  const unsigned neg_lo = 0x80000000u, neg_n = __builtin_bit_cast(unsigned, -104.0f) - 0x80000000u;
  k_ulps<<<148 * 8, 256>>>(neg_lo, neg_n, hist, worst);
  k_ulps<<<148 * 8, 256>>>(0u, __builtin_bit_cast(unsigned, 88.0f), hist, worst);
  CK(cudaDeviceSynchronize());
  unsigned long long h[8];
  int w;
  CK(cudaMemcpy(h, hist, 64, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&w, worst, 4, cudaMemcpyDeviceToHost));
  printf("CUDA expf vs glibc expf (ulps): 0:%llu 1:%llu 2:%llu 3:%llu 4:%llu 5:%llu 6:%llu >=7:%llu  worst %d\n", h[0],
         h[1], h[2], h[3], h[4], h[5], h[6], h[7], w);

  const size_t bytes = 1ull << 30, n = bytes / 16;
  float4 *x, *y;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&y, bytes));
  CK(cudaMemset(x, 0, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* nm, auto launch) {
    std::vector<float> ts;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    printf("%-34s %8.3f ms  %7.1f GB/s (read+write)\n", nm, ts[ts.size() / 2], 2.0 * bytes / (ts[ts.size() / 2] * 1e-3) / 1e9);
  };
  for (int B : {4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "fast expf*rcp   B=%d", B);
    run(nm, [&] { k_out<0><<<sms * B, 256>>>(x, y, n, 0.5f, 0.25f, 0.25); });
    snprintf(nm, sizeof nm, "cuda expf, dmul B=%d", B);
    run(nm, [&] { k_out<1><<<sms * B, 256>>>(x, y, n, 0.5f, 0.25f, 0.25); });
    snprintf(nm, sizeof nm, "glibc expf, dmul B=%d", B);
    run(nm, [&] { k_out<2><<<sms * B, 256>>>(x, y, n, 0.5f, 0.25f, 0.25); });
  }
  return 0;
}
