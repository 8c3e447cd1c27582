// topk_tma.cu -- persistent, TMA-fed fused online softmax + top-K
// (Alg. 4, reference online_softmax_topk_kernel kernels.hpp:108-125) and
// topk_of (kernels.hpp:72-83) for many rows of large V.
//
// Structure (one CTA per SM slot, rows visited grid-stride):
//   warp NCW      producer: lane 0 streams every row's 16-byte aligned body
//                 through a STAGES x CHUNK shared-memory ring with 1-D bulk
//                 copies (cp.async.bulk, evict-first), one mbarrier pair per
//                 stage.  It runs ahead across row boundaries, so the next
//                 row is already in flight while consumers merge this one.
//   warps 0..NCW-1 consumers: per stage, each thread takes U float4s
//                 (LDS.128), updates its online (m, d) with a batch-max-first
//                 rescale and offers batch survivors to its register top-K
//                 list; at row end a named-barrier CTA reduce (Eq. 4 merge)
//                 and a k-round list merge under (value desc, index asc).
// Head / tail elements outside the aligned body (V % 4 or unaligned rows)
// are read directly from global memory by the first consumer threads, first
// and last respectively, so every thread still sees its elements in
// increasing index order (the reference's tie rule, topk.hpp:37-43).
#include "topk_impl.cuh"
#include "tma.cuh"

namespace {

constexpr int kChunk = 16384;  // bytes per stage (4096 floats)
constexpr int kTmaMinBlocks = 3;  // 3 CTAs (24 consumer warps) per SM: <= 72 registers

// Consumer-group reductions over NC threads using named barrier 1.
template <int NCW>
__device__ __forceinline__ MD md_group_cta(MD s, float* sm) {
  s = md_group_reduce<32>(s);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sm[w] = s.m;
    sm[NCW + w] = s.d;
  }
  named_sync(1, NCW * 32);
  MD t = md_identity();
  if (l < NCW) t = MD{sm[l], sm[NCW + l]};
  t = md_group_reduce<32>(t);
  named_sync(1, NCW * 32);
  return t;
}
template <int NCW, class Op>
__device__ __forceinline__ float red_group_cta(float v, float init, Op op, float* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  named_sync(1, NCW * 32);
  float t = l < NCW ? sm[l] : init;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = op(t, __shfl_xor_sync(0xffffffffu, t, o));
  named_sync(1, NCW * 32);
  return t;
}

template <int NCW, int KC, class Sink>
__device__ __forceinline__ void merge_group_cta(TopList<KC>& L, int k, float* sv, int* si, Sink&& sink) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  L.normalize(k);
  group_merge<32>(L, k, [&](int r, float v, int i) {
    if (l == 0) {
      sv[w * KC + r] = v;
      si[w * KC + r] = i;
    }
  });
  named_sync(1, NCW * 32);
  if (w == 0) {
    TopList<KC> M;
    M.init_empty();
    if (l < NCW) {
#pragma unroll
      for (int r = 0; r < KC; ++r)
        if (r < k) {
          M.v[r] = sv[l * KC + r];
          M.i[r] = si[l * KC + r];
        }
    }
    group_merge<32>(M, k, sink);
  }
  named_sync(1, NCW * 32);
}

struct MinOp {
  __device__ float operator()(float a, float b) const { return fminf(a, b); }
};
struct SumOp {
  __device__ float operator()(float a, float b) const { return a + b; }
};

template <int NCW, int STAGES, int KC, int MODE>
__global__ void __launch_bounds__((NCW + 1) * 32, kTmaMinBlocks)
    k_topk_tma(const float* __restrict__ x, long long ldx, long long rows, long long V, int k,
               float* __restrict__ vals, long long* __restrict__ idx, void* ws, int R = 0, long long chunk = 0,
               long long col0 = 0, char* __restrict__ rec = nullptr, unsigned* __restrict__ tickets = nullptr,
               char* __restrict__ out_rec = nullptr) {
  constexpr int NC = NCW * 32;
  constexpr int U = kChunk / 16 / NC;  // float4s per consumer thread per stage
  static_assert(U >= 1 && U * NC * 16 == kChunk, "chunk must split evenly");
  extern __shared__ __align__(128) unsigned char smem[];
  float4* ring = reinterpret_cast<float4*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kChunk);
  uint64_t* empty = full + STAGES;
  float* smf = reinterpret_cast<float*>(empty + STAGES);  // 2*NCW
  float* sv = smf + 2 * NCW;                              // NCW*KC
  int* si = reinterpret_cast<int*>(sv + NCW * KC);        // NCW*KC
  int* tsh = si + NCW * KC;                               // 2 (row parity) + the last-piece flag
  // Record mode with tickets: the consumer group of the CTA that finishes a
  // row's last piece merges the row's R records (in piece order) and writes
  // the row's outputs -- the split combine fused into this launch.
  __shared__ CombineSmem<KC, NCW * 32> csm;

  // Record mode (rec != nullptr): "row" p is piece p % R of input row p / R,
  // columns [r * chunk, min(V, (r + 1) * chunk)), and writes a split record
  // like k_topk_rows' record mode.
  auto seg_of = [&](long long row, long long& piece0) {
    if (rec) {
      piece0 = (row % R) * chunk;
      return make_seg(x + (row / R) * ldx + piece0, V - piece0 < chunk ? V - piece0 : chunk);
    }
    piece0 = 0;
    return make_seg(x + row * ldx, V);
  };
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
    tsh[0] = tsh[1] = Pass<KC, 1, MODE, NCW * 32>::f2o(kNegInf);
  }
  __syncthreads();

  if (w == NCW) {
    // ------------------------------------------------------- producer
    if ((threadIdx.x & 31) == 0) {
      const uint64_t pol = pol_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        long long piece0;
        const Seg sg = seg_of(row, piece0);
        const char* b = reinterpret_cast<const char*>(sg.p + sg.head);
        const long long bytes = sg.nvec * 16;
        for (long long off = 0; off < bytes; off += kChunk) {
          const uint32_t n = (uint32_t)(bytes - off < kChunk ? bytes - off : kChunk);
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], n);
          tma_load_1d(reinterpret_cast<char*>(ring) + (size_t)s * kChunk, b + off, n, &full[s], pol);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  // --------------------------------------------------------- consumers
  const int t = threadIdx.x;
  int s = 0;
  uint32_t ph = 0;
  int it = 0;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x, ++it) {
    long long piece0;
    const Seg sg = seg_of(row, piece0);
    if (t == 0) tsh[(it + 1) & 1] = Pass<KC, U, MODE, NC>::f2o(kNegInf);
    Pass<KC, U, MODE, NC> P;
    P.L.init(k);
    P.kk = k;
    P.Tsh = &tsh[it & 1];
    if (t < sg.head) P.scalar(ld_f1(sg.p + t), t, k);
    const long long bytes = sg.nvec * 16;
    for (long long off = 0; off < bytes; off += kChunk) {
      const int n4 = (int)((bytes - off < kChunk ? bytes - off : kChunk) >> 4);
      mbar_wait(&full[s], ph);
      const float4* sb = ring + (size_t)s * (kChunk / 16);
      const int j0 = sg.head + (int)(off >> 2) + 4 * t;
      float4 v[U];
      if (n4 == kChunk / 16) {
        // full stage (every stage but a piece's last): no bounds checks, and
        // batch_j inlines with a constant count (no per-u masking)
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = sb[t + u * NC];
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&empty[s]);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
        P.batch_j(v, U, j0, 4 * NC);
        continue;
      }
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = t + u * NC;
        if (q < n4) {
          v[u] = sb[q];
          cnt = u + 1;
        } else {
          v[u] = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
      P.batch_j(v, cnt, j0, 4 * NC);  // warp-uniform call
    }
    if (t < sg.tail) {
      const int j = sg.head + (int)(4 * sg.nvec) + t;
      P.scalar(ld_f1(sg.p + j), j, k);
    }
    // ---- row epilogue (consumers only)
    float outM = 0.0f;
    double outR = 1.0;
    bool bad;
    RecHdr hdr{kNegInf, 0.0f, 0.0f, k};
    if constexpr (MODE == kModeFused) {
      const MD tot = md_group_cta<NCW>(P.acc.finish(), smf);
      const float mn = red_group_cta<NCW>(P.mn, -kNegInf, MinOp(), smf);
      outM = tot.m;
      outR = 1.0 / (double)tot.d;
      bad = !(tot.d == tot.d) || !isfinite(tot.m) || mn == kNegInf;
      hdr = RecHdr{tot.m, tot.d, mn, k};
    } else {
      const float c = red_group_cta<NCW>(P.chk, 0.0f, SumOp(), smf);
      bad = !(c == c);
      hdr.mn = (c == c) ? 0.0f : c;
    }
    char* my = rec ? rec + (size_t)row * rec_bytes_(k) : nullptr;
    merge_group_cta<NCW>(P.L, k, sv, si, [&](int r, float v, int i) {
      if ((int)(threadIdx.x & 31) == (r & 31)) {
        if (my) {
          reinterpret_cast<float*>(my + rec_vals_off())[r] = v;
          reinterpret_cast<long long*>(my + rec_idx_off(k))[r] = i < 0 ? -1LL : (long long)i + piece0 + col0;
          return;
        }
        float out = v;
        if constexpr (MODE == kModeFused) out = out_md(v, outM, outR);  // kernels.hpp:122
        vals[row * k + r] = out;
        idx[row * k + r] = (long long)i;
      }
    });
    if (my) {
      if (t == 0) *reinterpret_cast<RecHdr*>(my) = hdr;  // non-finite pieces: flagged by the combine
      if (tickets) {
        const long long ir = row / R;
        __threadfence();  // this thread's record stores, device-wide, before the ticket
        named_sync(1, NC);
        if (t == 0) {
          const unsigned tk = atomicAdd(&tickets[ir], 1u);
          tsh[2] = tk == (unsigned)(R - 1);
          if (tk == (unsigned)(R - 1)) tickets[ir] = 0u;  // every other piece of the row has its ticket
        }
        named_sync(1, NC);
        if (tsh[2]) {
          __threadfence();
          const size_t rb = rec_bytes_(k);
          combine_records_cta<KC, NCW * 32, true>(rec + (size_t)ir * R * rb, R, k, MODE,
                                                  out_rec ? out_rec + (size_t)ir * rb : nullptr,
                                                  vals ? vals + ir * k : nullptr, vals ? idx + ir * k : nullptr, ws,
                                                  ir, true, csm, [] { named_sync(1, NCW * 32); });
        }
      }
    } else if (bad && t == 0) {
      flag_bad_row(ws, row);
    }
  }
}

constexpr int kNCW = 8;
constexpr int kStages = 4;  // 3 x 4 x 16 KB of ring per SM

template <int KC, int MODE>
size_t tma_smem() {
  return (size_t)kStages * kChunk + 2 * kStages * sizeof(uint64_t) + 2 * kNCW * sizeof(float) +
         (size_t)kNCW * KC * (sizeof(float) + sizeof(int)) + 3 * sizeof(int);
}
template <int KC, int MODE>
int tma_per_sm() {
  static int per_sm = 0;  // per instantiation (same on every sm_100 device)
  if (per_sm == 0) {
    auto kern = k_topk_tma<kNCW, kStages, KC, MODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<KC, MODE>());
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (kNCW + 1) * 32, tma_smem<KC, MODE>());
    per_sm = n < 1 ? 1 : n;
  }
  return per_sm;
}

template <int KC, int MODE>
cudaError_t run_tma(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                    long long* idx, void* ws, cudaStream_t st, int R = 0, long long chunk = 0, long long col0 = 0,
                    char* rec = nullptr, unsigned* tickets = nullptr, char* out_rec = nullptr) {
  auto kern = k_topk_tma<kNCW, kStages, KC, MODE>;
  const size_t smem = tma_smem<KC, MODE>();
  const int per_sm = tma_per_sm<KC, MODE>();
  if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long grid = std::min<long long>(rows, (long long)per_sm * osmx_host::num_sms());
  kern<<<(unsigned)grid, (kNCW + 1) * 32, smem, st>>>(x, ldx, rows, V, k, vals, idx, ws, R, chunk, col0, rec, tickets,
                                                     out_rec);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_tma(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                         long long* idx, void* ws, cudaStream_t st, int R = 0, long long chunk = 0,
                         long long col0 = 0, char* rec = nullptr, unsigned* tickets = nullptr,
                         char* out_rec = nullptr) {
#define OSMX_TMA_CASE(KC) \
  return run_tma<KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec)
  if (k <= 1) OSMX_TMA_CASE(1);
  if (k <= 5) OSMX_TMA_CASE(5);
  if (k <= 8) OSMX_TMA_CASE(8);
  if (k <= 16) OSMX_TMA_CASE(16);
  OSMX_TMA_CASE(32);
#undef OSMX_TMA_CASE
}

}  // namespace

namespace osmx_host {
// mode 0: fused online softmax + top-K; mode 1: topk_of.
cudaError_t launch_topk_tma(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                            float* vals, long long* idx, void* ws, cudaStream_t st) {
  if (mode == kModeFused) return dispatch_tma<kModeFused>(x, ldx, rows, V, k, vals, idx, ws, st);
  return dispatch_tma<kModeTopkOf>(x, ldx, rows, V, k, vals, idx, ws, st);
}
long long topk_tma_slots(int k) {
  const int per_sm = k <= 1 ? tma_per_sm<1, kModeFused>() : k <= 5 ? tma_per_sm<5, kModeFused>()
                     : k <= 8 ? tma_per_sm<8, kModeFused>() : k <= 16 ? tma_per_sm<16, kModeFused>()
                     : tma_per_sm<32, kModeFused>();
  return (long long)per_sm * num_sms();
}
cudaError_t launch_topk_tma_records(int mode, const float* x, long long ldx, long long pieces, long long V, int k,
                                    void* ws, cudaStream_t st, int R, long long chunk, long long col0, char* rec,
                                    float* vals, long long* idx, char* out_rec) {
  // vals / out_rec given: the last piece of each row merges its records
  // (ticket counters in the workspace header area), no combine launch
  unsigned* tickets = (vals || out_rec) ? reinterpret_cast<unsigned*>(static_cast<char*>(ws) + kWsTicketsOff) : nullptr;
  if (mode == kModeFused)
    return dispatch_tma<kModeFused>(x, ldx, pieces, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec);
  return dispatch_tma<kModeTopkOf>(x, ldx, pieces, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec);
}
}  // namespace osmx_host
