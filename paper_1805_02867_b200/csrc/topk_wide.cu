// topk_wide.cu -- one-launch fused online softmax + top-K (and topk_of) for
// a few very long rows: configs[4] (one row of 2^26) and the V-split slice
// records of the cross-GPU path.
//
// Reference semantics: online_softmax_topk_kernel (kernels.hpp:108-125) on
// each row, evaluated as the chunked normalizer of normalizer.hpp:74-85 --
// per-CTA partial states merged with the paper's operator (Eq. 4,
// normalizer.hpp:52-58) in a fixed order, and per-CTA top-K lists merged
// under (value desc, index asc) (topk.hpp:37-43, oracle.cpp:48-51).
//
// Layout: `cpr` CTAs per row (the whole device's resident CTAs divided among
// the rows).  CTA c of a row reads the row's aligned float4 body grid-stride
// -- float4 q belongs to CTA (q / 256) % cpr, thread q % 256 -- with U
// independent 128-bit loads in flight per thread, so at every instant the
// whole device streams one contiguous window of the row (measured fastest
// of the one-launch read schemes for a 256 MB row, tools/c5_lab.cu: 43.7 us
// vs 46.6 us for a TMA ring of per-CTA pieces).  Every thread still sees its
// elements in increasing index order, so its strict-'>' list insertion keeps
// the reference's tie rule.
//
// The combine is fused: each CTA writes its record (m, d, min, k
// candidates with global indices) to the workspace, then takes a ticket
// (one counter per row in the workspace header area, zeroed by
// osmx_workspace_init and reset by its user); the CTA that takes the last
// ticket merges the row's cpr records IN CTA ORDER (deterministic, whatever
// the arrival order) and writes the outputs -- no second launch, no idle
// gap between the pieces and the combine.
#include "topk_impl.cuh"

namespace {

constexpr int kWideThreads = 256;
constexpr int kWideNW = kWideThreads / 32;

template <int KC, int MODE, int U, int MINB>
__global__ void __launch_bounds__(kWideThreads, MINB)
    k_topk_wide(const float* __restrict__ x, long long ldx, long long rows, long long V, int k, int cpr,
                float* __restrict__ vals, long long* __restrict__ idx, char* __restrict__ rec,
                unsigned* __restrict__ tickets, void* ws, long long col0, char* __restrict__ out_rec) {
  __shared__ float smf[2 * kWideNW];
  __shared__ float sv[kWideNW * KC];
  __shared__ int si[kWideNW * KC];
  __shared__ int tsh;
  __shared__ int s_last;
  __shared__ CombineSmem<KC, kWideThreads> csm;
  const long long row = blockIdx.x / cpr;
  const int slot = (int)(blockIdx.x % cpr);
  const int t = threadIdx.x;
  if (t == 0) tsh = Pass<KC, U, MODE, kWideThreads>::f2o(kNegInf);
  __syncthreads();

  const Seg s = make_seg(x + row * ldx, V);
  Pass<KC, U, MODE, kWideThreads> P;
  P.L.init(k);
  P.kk = k;
  P.Tsh = &tsh;
  // head scalars (before the first aligned float4) go to CTA 0's first
  // threads, ahead of their body elements (increasing index per thread)
  if (slot == 0 && t < s.head) P.scalar(ld_f1(s.p + t), t, k);
  const float* body = s.p + s.head;
  const long long S = (long long)cpr * kWideThreads;  // float4 stride between a thread's elements
  const long long nvec = s.nvec;
  // the warp's first float4 of this round decides the (warp-uniform) loop
  const long long wq0 = (long long)slot * kWideThreads + (t & ~31);
  long long q0 = (long long)slot * kWideThreads + t;
  for (long long wq = wq0; wq < nvec; wq += U * S, q0 += U * S) {
    float4 v[U];
    int cnt = 0;
    if (wq + (U - 1) * S + 31 < nvec) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_f4(body + 4 * (q0 + u * S));
      cnt = U;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (q0 + u * S < nvec) {
          v[u] = ld_f4(body + 4 * (q0 + u * S));
          cnt = u + 1;
        } else {
          v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        }
      }
    }
    P.batch_j(v, cnt, s.head + (int)(4 * q0), (int)(4 * S));
  }
  if (slot == cpr - 1 && t < s.tail) {
    const int j = s.head + (int)(4 * nvec) + t;
    P.scalar(ld_f1(s.p + j), j, k);
  }

  // ---- this CTA's record
  RecHdr hdr{kNegInf, 0.0f, 0.0f, k};
  if constexpr (MODE == kModeFused) {
    const MD tot = md_cta_reduce<kWideNW>(P.acc.finish(), smf);
    const float mn = cta_min<kWideNW>(P.mn, smf);
    hdr = RecHdr{tot.m, tot.d, mn, k};
  } else {
    const float c = cta_sum<kWideNW>(P.chk, smf);
    hdr.mn = (c == c) ? 0.0f : c;
  }
  const size_t rb = rec_bytes_(k);
  char* my = rec + ((size_t)row * cpr + slot) * rb;
  cta_merge<kWideNW>(P.L, k, sv, si, [&](int r, float v, int i) {
    if ((int)(threadIdx.x & 31) == (r & 31)) {
      reinterpret_cast<float*>(my + rec_vals_off())[r] = v;
      reinterpret_cast<long long*>(my + rec_idx_off(k))[r] = i < 0 ? -1LL : (long long)i + col0;
    }
  });
  if (t == 0) *reinterpret_cast<RecHdr*>(my) = hdr;

  // ---- ticket: the last CTA of the row merges the row's records
  __threadfence();  // this thread's record stores, device-wide, before the ticket
  __syncthreads();
  if (t == 0) {
    const unsigned tk = atomicAdd(&tickets[row], 1u);
    s_last = tk == (unsigned)(cpr - 1);
    if (s_last) tickets[row] = 0u;  // every other CTA of the row has taken its ticket
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();  // acquire side: the other CTAs' records (read L2-coherent below)
  combine_records_cta<KC, kWideThreads, true>(rec + (size_t)row * cpr * rb, cpr, k, MODE,
                                              out_rec ? out_rec + (size_t)row * rb : nullptr,
                                              vals ? vals + row * k : nullptr, vals ? idx + row * k : nullptr, ws,
                                              row, true, csm);
}

constexpr int kWideU = 8;
constexpr int kWideMinB = 4;

template <int KC, int MODE>
int wide_per_sm() {
  static int per_sm = 0;  // per instantiation (same on every sm_100 device)
  if (per_sm == 0) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_topk_wide<KC, MODE, kWideU, kWideMinB>, kWideThreads, 0);
    per_sm = n < 1 ? 1 : n;
  }
  return per_sm;
}

template <int KC, int MODE>
cudaError_t run_wide(const float* x, long long ldx, long long rows, long long V, int k, float* vals, long long* idx,
                     void* ws, cudaStream_t st, long long col0, char* out_rec) {
  const long long slots = (long long)wide_per_sm<KC, MODE>() * osmx_host::num_sms();
  const int cpr = (int)std::max<long long>(1, slots / rows);
  char* base = static_cast<char*>(ws);
  unsigned* tickets = reinterpret_cast<unsigned*>(base + kWsTicketsOff);
  char* rec = base + kWsHeader;
  k_topk_wide<KC, MODE, kWideU, kWideMinB><<<(unsigned)(rows * cpr), kWideThreads, 0, st>>>(
      x, ldx, rows, V, k, cpr, vals, idx, rec, tickets, ws, col0, out_rec);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_wide(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                          long long* idx, void* ws, cudaStream_t st, long long col0, char* out_rec) {
#define OSMX_WIDE_CASE(KC) return run_wide<KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, col0, out_rec)
  if (k <= 1) OSMX_WIDE_CASE(1);
  if (k <= 5) OSMX_WIDE_CASE(5);
  if (k <= 8) OSMX_WIDE_CASE(8);
  if (k <= 16) OSMX_WIDE_CASE(16);
  OSMX_WIDE_CASE(32);
#undef OSMX_WIDE_CASE
}

}  // namespace

namespace osmx_host {
long long topk_wide_slots(int k) {
  const int per_sm = k <= 1 ? wide_per_sm<1, kModeFused>() : k <= 5 ? wide_per_sm<5, kModeFused>()
                     : k <= 8 ? wide_per_sm<8, kModeFused>() : k <= 16 ? wide_per_sm<16, kModeFused>()
                     : wide_per_sm<32, kModeFused>();
  return (long long)per_sm * num_sms();
}
// mode 0: fused online softmax + top-K; 1: topk_of.  Records go to the
// split region (ws + kWsHeader), rows * cpr of them.
cudaError_t launch_topk_wide(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                             float* vals, long long* idx, void* ws, cudaStream_t st, long long col0, char* out_rec) {
  if (mode == kModeFused) return dispatch_wide<kModeFused>(x, ldx, rows, V, k, vals, idx, ws, st, col0, out_rec);
  return dispatch_wide<kModeTopkOf>(x, ldx, rows, V, k, vals, idx, ws, st, col0, out_rec);
}
}  // namespace osmx_host
