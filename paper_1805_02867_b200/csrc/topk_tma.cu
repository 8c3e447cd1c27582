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

// CTAs per SM the ring leaves room for: 3 x 64 KB (<= 72 registers), 2 x 96 KB
constexpr int tma_min_blocks(int ring_bytes) { return ring_bytes > 65536 ? 2 : 3; }

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

template <int NCW, int STAGES, int kChunk, int KC, int MODE>
__global__ void __launch_bounds__((NCW + 1) * 32, tma_min_blocks(STAGES * kChunk))
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

// ------------------------------------------------- one row, dynamic chunks --
// configs[4] (one row of 2^26) and the V-split slices: every resident CTA
// streams the row through its ring, but the producer CLAIMS stage-sized
// chunks from a device-wide counter (atomicAdd, issued one chunk ahead so
// its latency hides behind the empty-slot wait) instead of owning a fixed
// piece: SMs whose DRAM path is faster take more chunks, and every CTA
// runs out of work within one chunk of the others.  (Static pieces: ncu
// shows per-SM active cycles spread 86K..99K -- the slowest SMs set the
// time.)  A CTA's chunk ids only increase, and each thread walks its chunk
// offsets in order, so every thread still sees its elements in increasing
// index order (the strict '>' tie rule, topk.hpp:37-43); the CTA writes one
// record, and the last CTA to finish (ticket) merges the records in CTA
// order under (value desc, index asc) -- indices are exact and
// deterministic; d sums per-thread partials whose composition follows the
// dynamic assignment (fp32 rounding, like every other d here).
#ifdef OSMX_TIMELINE
// Diagnostic build only (make timeline): per CTA %globaltimer at entry,
// end of streaming, ticket, combine end (last CTA), and chunks consumed.
__device__ unsigned long long g_tl[1024 * 5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define OSMX_TL(slot, val) \
  do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_tl[blockIdx.x * 5 + (slot)] = (val); } while (0)
#else
#define OSMX_TL(slot, val) do { } while (0)
#endif

template <int NCW, int STAGES, int kChunk, int KC, int MODE>
__global__ void __launch_bounds__((NCW + 1) * 32, tma_min_blocks(STAGES * kChunk))
    k_topk_tma_dyn(const float* __restrict__ x, long long V, int k, float* __restrict__ vals,
                   long long* __restrict__ idx, void* ws, long long col0, char* __restrict__ rec,
                   char* __restrict__ out_rec) {
  constexpr int NC = NCW * 32;
  constexpr int U = kChunk / 16 / NC;
  static_assert(U >= 1 && U * NC * 16 == kChunk, "chunk must split evenly");
  extern __shared__ __align__(128) unsigned char smem[];
  float4* ring = reinterpret_cast<float4*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kChunk);
  uint64_t* empty = full + STAGES;
  float* smf = reinterpret_cast<float*>(empty + STAGES);  // 2*NCW
  __shared__ long long chunk_of[STAGES];                  // claimed chunk per stage (-1: no more)
  __shared__ int tsh;
  __shared__ int s_last;
  __shared__ CombineSmem<KC, NC> csm;
  __shared__ float sv[NCW * KC];
  __shared__ int si[NCW * KC];
  WsHeader* hdr_ws = reinterpret_cast<WsHeader*>(ws);
  unsigned* ticket = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + kWsTicketsOff);

#ifdef OSMX_TIMELINE
  OSMX_TL(0, gtimer());
  int tl_chunks = 0;
#endif
  const Seg sg = make_seg(x, V);
  const long long bytes = sg.nvec * 16;
  const long long nch = (bytes + kChunk - 1) / kChunk;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
    tsh = Pass<KC, U, MODE, NC>::f2o(kNegInf);
  }
  __syncthreads();

  if (w == NCW) {
    // ------------------------------------------------------- producer
    if ((threadIdx.x & 31) == 0) {
      const uint64_t pol = pol_evict_first();
      const char* b = reinterpret_cast<const char*>(sg.p + sg.head);
      int s = 0;
      uint32_t ph = 0;
      long long next = (long long)atomicAdd(&hdr_ws->chunk_ctr, 1ull);
      for (;;) {
        const long long c = next;
        if (c >= nch) break;
        next = (long long)atomicAdd(&hdr_ws->chunk_ctr, 1ull);  // in flight during the wait below
        const long long off = c * kChunk;
        const uint32_t n = (uint32_t)(bytes - off < kChunk ? bytes - off : kChunk);
        mbar_wait(&empty[s], ph ^ 1);
        chunk_of[s] = c;
        mbar_arrive_expect_tx(&full[s], n);
        tma_load_1d(reinterpret_cast<char*>(ring) + (size_t)s * kChunk, b + off, n, &full[s], pol);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      mbar_wait(&empty[s], ph ^ 1);
      chunk_of[s] = -1;
      mbar_arrive(&full[s]);  // completes the phase with no bytes: "no more chunks"
    }
    return;
  }

  // --------------------------------------------------------- consumers
  const int t = threadIdx.x;
  Pass<KC, U, MODE, NC> P;
  P.L.init(k);
  P.kk = k;
  P.Tsh = &tsh;
  // head scalars precede every body element: CTA 0's first threads, first
  if (blockIdx.x == 0 && t < sg.head) P.scalar(ld_f1(sg.p + t), t, k);
  int s = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full[s], ph);
    const long long c = *reinterpret_cast<volatile long long*>(&chunk_of[s]);
    if (c < 0) break;
#ifdef OSMX_TIMELINE
    ++tl_chunks;
#endif
    const long long off = c * kChunk;
    const int n4 = (int)((bytes - off < kChunk ? bytes - off : kChunk) >> 4);
    const float4* sb = ring + (size_t)s * (kChunk / 16);
    const int j0 = sg.head + (int)(off >> 2) + 4 * t;
    float4 v[U];
    int cnt = U;
    if (n4 == kChunk / 16) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = sb[t + u * NC];
    } else {
      cnt = 0;
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
    }
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(&empty[s]);
    if (++s == STAGES) {
      s = 0;
      ph ^= 1;
    }
    if (cnt == U)
      P.batch_j(v, U, j0, 4 * NC);
    else
      P.batch_j(v, cnt, j0, 4 * NC);
  }
#ifdef OSMX_TIMELINE
  OSMX_TL(1, gtimer());
  OSMX_TL(4, (unsigned long long)tl_chunks);
#endif
  // tail scalars follow every body element: CTA 0's first threads, last
  if (blockIdx.x == 0 && t < sg.tail) {
    const int j = sg.head + (int)(4 * sg.nvec) + t;
    P.scalar(ld_f1(sg.p + j), j, k);
  }

  // ---- this CTA's record, then the ticket: two barrier rounds.  Each warp
  // reduces its (m, d, min) and merges its lanes' lists; warp 0 reduces the
  // NCW warp results, writes the record, fences it and takes the ticket.
  const int l = t & 31;
  {
    MD tot = md_identity();
    float mn = -kNegInf;
    if constexpr (MODE == kModeFused) {
      tot = md_group_reduce<32>(P.acc.finish());
      mn = group_min<32>(P.mn);
    } else {
      mn = group_sum<32>(P.chk);  // NaN iff some element was inf / NaN
    }
    P.L.normalize(k);
    group_merge<32>(P.L, k, [&](int r, float v, int i) {
      if (l == 0) {
        sv[w * KC + r] = v;
        si[w * KC + r] = i;
      }
    });
    if (l == 0) {
      smf[w] = tot.m;
      smf[NCW + w] = tot.d;
      csm.sm_mn[w] = mn;
    }
  }
  named_sync(1, NC);
  if (w == 0) {
    MD tot = l < NCW ? MD{smf[l], smf[NCW + l]} : md_identity();
    float mn = l < NCW ? csm.sm_mn[l] : (MODE == kModeFused ? -kNegInf : 0.0f);
    RecHdr hdr{kNegInf, 0.0f, 0.0f, k};
    if constexpr (MODE == kModeFused) {
      tot = md_group_reduce<32>(tot);
      mn = group_min<32>(mn);
      hdr = RecHdr{tot.m, tot.d, mn, k};
    } else {
      mn = group_sum<32>(mn);
      hdr.mn = (mn == mn) ? 0.0f : mn;
    }
    const size_t rb = rec_bytes_(k);
    char* my = rec + (size_t)blockIdx.x * rb;
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
    group_merge<32>(M, k, [&](int r, float v, int i) {
      if (l == (r & 31)) {
        reinterpret_cast<float*>(my + rec_vals_off())[r] = v;
        reinterpret_cast<long long*>(my + rec_idx_off(k))[r] = i < 0 ? -1LL : (long long)i + col0;
      }
    });
    if (l == 0) *reinterpret_cast<RecHdr*>(my) = hdr;
    __threadfence();  // the record, device-wide, before the ticket
    __syncwarp();
    if (l == 0) {
      const unsigned tk = atomicAdd(ticket, 1u);
      s_last = tk == gridDim.x - 1;
#ifdef OSMX_TIMELINE
      OSMX_TL(2, gtimer());
#endif
      if (s_last) {  // every CTA has claimed its last chunk and taken its ticket
        ticket[0] = 0u;
        hdr_ws->chunk_ctr = 0ull;
      }
    }
  }
  named_sync(1, NC);
  if (!s_last) return;
  OSMX_STAMP(5);
  __threadfence();
  OSMX_STAMP(6);
  auto sync = [] { named_sync(1, NCW * 32); };
  combine_records_cta<KC, NC, true, decltype(sync), false>(rec, (int)gridDim.x, k, MODE, out_rec, vals, idx, ws, 0,
                                                           true, csm, sync);
#ifdef OSMX_TIMELINE
  OSMX_TL(3, gtimer());
#endif
}

// Ring layouts (knob tma_cfg): consumer warps x stages x stage bytes.
//   0: 8 x 4 x 16 KB, 3 CTAs per SM, 4 float4s per thread per stage
//   1: 8 x 3 x 32 KB, 2 CTAs per SM, 8 float4s per thread per stage
//   2: 4 x 4 x 16 KB, 3 CTAs per SM, 8 float4s per thread per stage
template <int CFG> struct TmaCfg;
template <> struct TmaCfg<0> { static constexpr int NCW = 8, STAGES = 4, CH = 16384; };
template <> struct TmaCfg<1> { static constexpr int NCW = 8, STAGES = 3, CH = 32768; };
template <> struct TmaCfg<2> { static constexpr int NCW = 4, STAGES = 4, CH = 16384; };

template <int CFG, int KC, int MODE>
size_t tma_smem() {
  using C = TmaCfg<CFG>;
  return (size_t)C::STAGES * C::CH + 2 * C::STAGES * sizeof(uint64_t) + 2 * C::NCW * sizeof(float) +
         (size_t)C::NCW * KC * (sizeof(float) + sizeof(int)) + 3 * sizeof(int);
}
template <int CFG, int KC, int MODE>
int tma_per_sm() {
  static int per_sm = 0;  // per instantiation (same on every sm_100 device)
  if (per_sm == 0) {
    using C = TmaCfg<CFG>;
    auto kern = k_topk_tma<C::NCW, C::STAGES, C::CH, KC, MODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem<CFG, KC, MODE>());
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (C::NCW + 1) * 32, tma_smem<CFG, KC, MODE>());
    per_sm = n < 1 ? 1 : n;
  }
  return per_sm;
}

template <int CFG, int KC, int MODE>
cudaError_t run_tma(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                    long long* idx, void* ws, cudaStream_t st, int R = 0, long long chunk = 0, long long col0 = 0,
                    char* rec = nullptr, unsigned* tickets = nullptr, char* out_rec = nullptr) {
  using C = TmaCfg<CFG>;
  auto kern = k_topk_tma<C::NCW, C::STAGES, C::CH, KC, MODE>;
  const size_t smem = tma_smem<CFG, KC, MODE>();
  const int per_sm = tma_per_sm<CFG, KC, MODE>();
  if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long grid = std::min<long long>(rows, (long long)per_sm * osmx_host::num_sms());
  kern<<<(unsigned)grid, (C::NCW + 1) * 32, smem, st>>>(x, ldx, rows, V, k, vals, idx, ws, R, chunk, col0, rec,
                                                        tickets, out_rec);
  osmx_host::count_launch();
  return cudaGetLastError();
}

template <int CFG, int KC, int MODE>
cudaError_t run_tma_dyn(const float* x, long long V, int k, float* vals, long long* idx, void* ws, cudaStream_t st,
                        long long col0, char* rec, char* out_rec) {
  using C = TmaCfg<CFG>;
  auto kern = k_topk_tma_dyn<C::NCW, C::STAGES, C::CH, KC, MODE>;
  const size_t smem = (size_t)C::STAGES * C::CH + 2 * C::STAGES * sizeof(uint64_t) + 2 * C::NCW * sizeof(float);
  static int per_sm = 0;
  if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (per_sm == 0) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (C::NCW + 1) * 32, smem);
    per_sm = n < 1 ? 1 : n;
  }
  // <= the records the split workspace holds (topk_split_ws: wide slots)
  const int grid = (int)std::min<long long>((long long)per_sm * osmx_host::num_sms(), osmx_host::topk_wide_slots(k));
  kern<<<(unsigned)grid, (C::NCW + 1) * 32, smem, st>>>(x, V, k, vals, idx, ws, col0, rec, out_rec);
  osmx_host::count_launch();
  return cudaGetLastError();
}

// The layout in force: the alternatives are built for the fused k <= 5 case
// (configs[4] and the V-split slices) only.
// Auto (-1): 8 x 3 x 32 KB for the one-row dynamic-chunk path (configs[4]:
// 0.0521 vs 0.0528 ms for layout 0, 0.0558 for layout 2; tools/runs/r2_s.sh),
// 8 x 4 x 16 KB for the static pieces (its one-wave piece count needs 3 CTAs
// per SM).
inline int tma_cfg_for(int k, int mode, bool dyn = false) {
  int c = osmx_host::tuning().tma_cfg;
  if (c < 0) c = dyn ? 1 : 0;
  return (mode == kModeFused && k > 1 && k <= 5) ? c : 0;
}

template <int KC, int MODE>
cudaError_t run_tma_cfg(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                        long long* idx, void* ws, cudaStream_t st, int R, long long chunk, long long col0, char* rec,
                        unsigned* tickets, char* out_rec) {
  if constexpr (KC == 5 && MODE == kModeFused) {
    const int c = tma_cfg_for(k, MODE);
    if (c == 1) return run_tma<1, KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec);
    if (c == 2) return run_tma<2, KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec);
  }
  return run_tma<0, KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec);
}

template <int MODE>
cudaError_t dispatch_tma(const float* x, long long ldx, long long rows, long long V, int k, float* vals,
                         long long* idx, void* ws, cudaStream_t st, int R = 0, long long chunk = 0,
                         long long col0 = 0, char* rec = nullptr, unsigned* tickets = nullptr,
                         char* out_rec = nullptr) {
#define OSMX_TMA_CASE(KC) \
  return run_tma_cfg<KC, MODE>(x, ldx, rows, V, k, vals, idx, ws, st, R, chunk, col0, rec, tickets, out_rec)
  if (k <= 1) OSMX_TMA_CASE(1);
  if (k <= 5) OSMX_TMA_CASE(5);
  if (k <= 8) OSMX_TMA_CASE(8);
  if (k <= 16) OSMX_TMA_CASE(16);
  OSMX_TMA_CASE(32);
#undef OSMX_TMA_CASE
}

}  // namespace

#ifdef OSMX_TIMELINE
extern "C" int osmx_diag_timeline_clear() {
  static unsigned long long zero[1024 * 5];
  cudaMemcpyToSymbol(g_tl2, zero, sizeof(unsigned long long) * 16);
  return (int)cudaMemcpyToSymbol(g_tl, zero, sizeof(zero));
}
extern "C" int osmx_diag_timeline2(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_tl2, sizeof(unsigned long long) * 16);
}
extern "C" int osmx_diag_timeline(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_tl, sizeof(unsigned long long) * (size_t)(n < 5120 ? n : 5120));
}
#endif

namespace osmx_host {
// mode 0: fused online softmax + top-K; mode 1: topk_of.
cudaError_t launch_topk_tma(int mode, const float* x, long long ldx, long long rows, long long V, int k,
                            float* vals, long long* idx, void* ws, cudaStream_t st) {
  if (mode == kModeFused) return dispatch_tma<kModeFused>(x, ldx, rows, V, k, vals, idx, ws, st);
  return dispatch_tma<kModeTopkOf>(x, ldx, rows, V, k, vals, idx, ws, st);
}
long long topk_tma_slots(int k) {
  const int c = tma_cfg_for(k, kModeFused);
  const int per_sm = k <= 1 ? tma_per_sm<0, 1, kModeFused>()
                     : k <= 5 ? (c == 1 ? tma_per_sm<1, 5, kModeFused>()
                                : c == 2 ? tma_per_sm<2, 5, kModeFused>() : tma_per_sm<0, 5, kModeFused>())
                     : k <= 8 ? tma_per_sm<0, 8, kModeFused>() : k <= 16 ? tma_per_sm<0, 16, kModeFused>()
                     : tma_per_sm<0, 32, kModeFused>();
  return (long long)per_sm * num_sms();
}
// One row, dynamic chunks, combine fused (records: one per resident CTA).
cudaError_t launch_topk_tma_dyn(int mode, const float* x, long long V, int k, float* vals, long long* idx, void* ws,
                                cudaStream_t st, long long col0, char* rec, char* out_rec) {
  const int c = tma_cfg_for(k, mode, true);
#define OSMX_DYN(CFG, KC, MD) return run_tma_dyn<CFG, KC, MD>(x, V, k, vals, idx, ws, st, col0, rec, out_rec)
  if (mode == kModeFused) {
    if (k <= 1) OSMX_DYN(0, 1, kModeFused);
    if (k <= 5) {
      if (c == 1) OSMX_DYN(1, 5, kModeFused);
      if (c == 2) OSMX_DYN(2, 5, kModeFused);
      OSMX_DYN(0, 5, kModeFused);
    }
    if (k <= 8) OSMX_DYN(0, 8, kModeFused);
    if (k <= 16) OSMX_DYN(0, 16, kModeFused);
    OSMX_DYN(0, 32, kModeFused);
  }
  if (k <= 1) OSMX_DYN(0, 1, kModeTopkOf);
  if (k <= 5) OSMX_DYN(0, 5, kModeTopkOf);
  if (k <= 8) OSMX_DYN(0, 8, kModeTopkOf);
  if (k <= 16) OSMX_DYN(0, 16, kModeTopkOf);
  OSMX_DYN(0, 32, kModeTopkOf);
#undef OSMX_DYN
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
