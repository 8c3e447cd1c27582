// proj_topk.cu -- the projection layer fused with the online softmax + top-K
// (SURVEY.md sec.8f item 4): logits Z = H W^T (H rows x D, W V x
// D, bf16, fp32 accumulation) are never written to HBM.  Each CTA computes a
// 128 x 256 tile of Z on the 5th-generation tensor cores and its epilogue
// reduces every row of the tile to one split record -- the online normalizer
// (m, d) of the 256 logits (Alg. 3 lines 1-6) and their top-K (topk.hpp:34-44,
// strict '>' over increasing column) -- which k_topk_combine_cta merges per
// row (Eq. 4 merge, (value desc, index asc) list merge) into the final
// e^(z - m)/d values and column indices, as for any split row.
//
// Per CTA (one 128 x 256 tile, 192 KB ring of 4 K-stages of 64 bf16):
//   warp 0 (one lane)  TMA producer: cp.async.bulk.tensor.2d of the H tile
//                      (128 x 64) and the W tile (256 x 64), 128-byte swizzle,
//                      onto the stage's "full" mbarrier (complete_tx);
//   warp 1 (one lane)  MMA issuer: per stage 4 x tcgen05.mma.cta_group::1.
//                      kind::f16 (M 128, N 256, K 16) into a 256-column TMEM
//                      accumulator, tcgen05.commit -> the stage's "empty"
//                      mbarrier; after the last stage, commit -> "accum";
//   warp 2             TMEM allocation / deallocation;
//   warps 4..7         epilogue: tcgen05.ld 32x32b.x32 (thread = TMEM lane =
//                      tile row), online (m, d) + register top-K list over the
//                      row's 256 columns, one record per (row, tile).
// Out-of-range rows / columns (TMA zero fill) are masked to -inf.
#include <cuda.h>

#include "common.cuh"
#include "internal.hpp"
#include "tma.cuh"
#include "topk_impl.cuh"

using namespace osmx_dev;

namespace {

constexpr int kBM = 128, kBK = 64;  // row tile, K-stage (64 bf16 = one 128-byte swizzle row)
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kProjThreads = 256;
// BN (vocabulary tile) = 256, 224 (whole waves of tiles over the SMs when
// there are few row tiles), or 128 (forced only)
template <int BN>
struct ProjCfg {
  static constexpr int kStages = BN == 128 ? 6 : 4;  // ~176-192 KB ring
  // TMEM columns for the two accumulators (allocation: a power of two)
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr size_t kSmem = 1024 /* align slack */ + (size_t)kStages * kStageBytes + 256;
};
constexpr int kBNMax = 256;

// Bounded mbarrier wait: a protocol bug traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_b(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  for (long long it = 0; it < (1LL << 24); ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128-byte
// atoms stacked along M/N at 1024 bytes (SBO), LBO unused (1), version 1
// (cute/arch/mma_sm100_desc.hpp SmemDescriptor; make_umma_desc<Major::K>).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address  [0,14)
  d |= (uint64_t)1 << 16;                         // LBO            [16,30)
  d |= (uint64_t)(1024 >> 4) << 32;               // SBO            [32,46)
  d |= (uint64_t)1 << 46;                         // version        [46,48)
  d |= (uint64_t)2 << 61;                         // SWIZZLE_128B   [61,64)
  return d;
}

// Instruction descriptor: BF16 x BF16 -> F32, both K-major, M 128, N = BN
// (cute/arch/mma_sm100_desc.hpp InstrDescriptor).
template <int BN>
constexpr uint32_t idesc_bf16() {
  return (1u << 4)                        // c_format F32
         | (1u << 7)                      // a_format BF16
         | (1u << 10)                     // b_format BF16
         | ((uint32_t)(BN >> 3) << 17)    // n_dim
         | ((uint32_t)(kBM >> 4) << 24);  // m_dim
}

template <int BN>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_c, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_c),
      "l"(adesc), "l"(bdesc), "r"(idesc_bf16<BN>()), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Persistent: one CTA per SM walks the (row tile, vocabulary tile) grid,
// row tiles fastest (the CTAs in flight cover every row tile of a few
// vocabulary tiles, so each W tile is read from HBM once and shared through
// L2; H stays L2-resident).  Two 256-column TMEM accumulators: the MMA warp
// fills one while the epilogue warps drain the other, and the TMA producer
// runs ahead across tile boundaries -- the epilogue and the pipeline fill
// are hidden behind the tensor-core mainloop.
template <int KC, int BN>
__global__ void __launch_bounds__(kProjThreads, 1)
    k_proj_topk(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w, int rows,
                int D, int V, int k, char* __restrict__ rec, int MT, int NT) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kBN = BN;
  constexpr int kStageBytes = ProjCfg<BN>::kStageBytes;
  constexpr int kStages = ProjCfg<BN>::kStages;
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* afull = empty + kStages;  // [2] accumulator ready (MMA commit)
  uint64_t* aempty = afull + 2;       // [2] accumulator drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (D + kBK - 1) / kBK;
  const int ntiles = MT * NT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 1);
      mbar_init(&aempty[b], 4);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_h) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_w) : "memory");
  }
  if (warp == 2) {  // TMEM: 2 x 256 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(ProjCfg<BN>::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer
    long long g = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m0 = (t % MT) * kBM, n0 = (t / MT) * kBN;
      for (int kc = 0; kc < nk; ++kc, ++g) {
        const int s = (int)(g % kStages);
        if (g >= kStages) mbar_wait_b(&empty[s], (uint32_t)(((g / kStages) - 1) & 1));
        unsigned char* a = smem + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], (uint32_t)kStageBytes);
        tma_load_2d(a, &tmap_h, kc * kBK, m0, &full[s]);
        tma_load_2d(a + kABytes, &tmap_w, kc * kBK, n0, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------- MMA issuer
    long long g = 0;
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      if (i >= 2) mbar_wait_b(&aempty[b], (uint32_t)(((i >> 1) - 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc_t = tmem + (uint32_t)(b * kBN);
      for (int kc = 0; kc < nk; ++kc, ++g) {
        const int s = (int)(g % kStages);
        mbar_wait_b(&full[s], (uint32_t)((g / kStages) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = smem_u32(smem + s * kStageBytes);
        const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(a + kABytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)  // K 16 per MMA = 32 bytes along the swizzled row
          umma_bf16<BN>(acc_t, ad + (uint64_t)((kk * 32) >> 4), bd + (uint64_t)((kk * 32) >> 4), (kc | kk) != 0);
        umma_commit(&empty[s]);  // stage free once these MMAs have read it
      }
      umma_commit(&afull[b]);  // accumulator b complete
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;       // TMEM lane quadrant of this warp
    const int r = q * 32 + lane;  // tile row = TMEM lane
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      const int m0 = (t % MT) * kBM, nt = t / MT, n0 = nt * kBN;
      const int row = m0 + r;
      mbar_wait_b(&afull[b], (uint32_t)((i >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      L2Acc acc;
      TopList<KC> L;
      L.init(k);
      float mn = -kNegInf;
#pragma unroll 1
      for (int c = 0; c < kBN; c += 32) {
        uint32_t u[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
              "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]),
              "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]),
              "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]),
              "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
            : "r"(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kBN + c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[j] = make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]), __uint_as_float(u[4 * j + 2]),
                             __uint_as_float(u[4 * j + 3]));
        if (n0 + c + 32 > V) {  // the vocabulary ends inside this chunk: mask (TMA zero fill)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int col = n0 + c + 4 * j;
            if (col + 0 >= V) v[j].x = kNegInf;
            if (col + 1 >= V) v[j].y = kNegInf;
            if (col + 2 >= V) v[j].z = kNegInf;
            if (col + 3 >= V) v[j].w = kNegInf;
          }
        }
        float bm = kNegInf, bn = -kNegInf;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          bm = fmaxf(bm, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
          // masked lanes are -inf; min over real columns only matters for
          // the non-finite check, and real logits are finite or NaN
          if (n0 + c + 4 * j + 3 < V) bn = fminf(bn, fminf(fminf(v[j].x, v[j].y), fminf(v[j].z, v[j].w)));
        }
        mn = fminf(mn, bn);
        if (n0 + c < V) {  // any real column: added even when the max is -inf, so NaN logits poison d
          acc.raise(bm);
          acc.add_batch<8>(v);
        }
        // columns in increasing order: strict '>' keeps ties on the lower column
        if (bm > L.thr()) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (!(fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)) > L.thr())) continue;
            const int col = c + 4 * j;
            L.offer(v[j].x, col);
            L.offer(v[j].y, col + 1);
            L.offer(v[j].z, col + 2);
            L.offer(v[j].w, col + 3);
          }
        }
      }
      // accumulator b is in registers now: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&aempty[b]);
      if (row < rows) {
        const MD md = acc.finish();
        char* my = rec + ((size_t)row * NT + nt) * rec_bytes_(k);
        *reinterpret_cast<RecHdr*>(my) = RecHdr{md.m, md.d, mn, k};
        float* rv = reinterpret_cast<float*>(my + rec_vals_off());
        long long* ri = reinterpret_cast<long long*>(my + rec_idx_off(k));
        L.normalize(k);
#pragma unroll
        for (int s2 = 0; s2 < KC; ++s2)
          if (s2 < k) {
            rv[s2] = L.v[s2];
            ri[s2] = L.i[s2] < 0 ? -1LL : (long long)(n0 + L.i[s2]);
          }
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ProjCfg<BN>::kTmemCols) : "memory");
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 tensor map of a row-major [outer x inner] matrix, box [box_outer x 64].
bool make_map(CUtensorMap* m, const void* base, long long inner, long long outer, int box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KC, int BN>
cudaError_t run_proj_bn(const void* h, long long rows, long long D, const void* w, long long V, int k, float* vals,
                        long long* idx, void* ws, cudaStream_t st) {
  constexpr size_t smem = ProjCfg<BN>::kSmem;
  CUtensorMap mh, mw;
  if (!make_map(&mh, h, D, rows, kBM) || !make_map(&mw, w, D, V, BN)) return cudaErrorInvalidValue;
  auto kern = k_proj_topk<KC, BN>;
  if (osmx_host::first_use_on_device(reinterpret_cast<const void*>(kern))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int MT = (int)((rows + kBM - 1) / kBM), nt = (int)((V + BN - 1) / BN);
  char* rec = static_cast<char*>(ws) + kWsHeader;
  const long long tiles = (long long)MT * nt;
  const int grid = (int)std::min<long long>(tiles, osmx_host::num_sms());
  kern<<<grid, kProjThreads, smem, st>>>(mh, mw, (int)rows, (int)D, (int)V, k, rec, MT, nt);
  osmx_host::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (nt >= 64)
    launch_pdl(k_topk_combine_cta<KC, 256>, dim3((unsigned)rows), dim3(256), 0, st, (const char*)rec, nt, k,
               (int)kModeFused, (char*)nullptr, vals, idx, 0LL, ws);
  else
    launch_pdl(k_topk_combine<KC>, dim3((unsigned)rows), dim3(32), 0, st, (const char*)rec, nt, k, (int)kModeFused,
               (char*)nullptr, vals, idx, 0LL, ws);
  osmx_host::count_launch();
  return cudaGetLastError();
}

// Vocabulary tile: 256 columns, or 224 when that fills the last wave of the
// persistent grid clearly better (> 3% shorter waves x width; few row
// tiles: 128 x 4096 x 131072 has 512 tiles of 256 = 3.46 waves over 148
// SMs, 586 of 224 = 3.96).  128
// only when forced: measured slower at every tested shape, 32..4096 rows,
// tools/proj_bench.py -- the finer load balance does not pay for twice the
// per-tile epilogues and records.
inline long long proj_span(long long rows, long long V, int bn) {  // waves x tile width
  const long long sms = osmx_host::num_sms();
  const long long tiles = ((rows + kBM - 1) / kBM) * ((V + bn - 1) / bn);
  return (tiles + sms - 1) / sms * bn;
}
inline int proj_bn(long long rows, long long V) {
  const int forced = osmx_host::tuning().proj_bn;
  if (forced) return forced;
  return proj_span(rows, V, 224) * 103 < proj_span(rows, V, 256) * 100 ? 224 : 256;
}

template <int KC>
cudaError_t run_proj(const void* h, long long rows, long long D, const void* w, long long V, int k, float* vals,
                     long long* idx, void* ws, cudaStream_t st) {
  const int bn = proj_bn(rows, V);
  if (bn == 128) return run_proj_bn<KC, 128>(h, rows, D, w, V, k, vals, idx, ws, st);
  if (bn == 224) return run_proj_bn<KC, 224>(h, rows, D, w, V, k, vals, idx, ws, st);
  return run_proj_bn<KC, 256>(h, rows, D, w, V, k, vals, idx, ws, st);
}

}  // namespace

namespace osmx_host {

size_t proj_topk_ws(long long rows, long long V, int k) {
  const long long nt = (V + 128 - 1) / 128;  // the finer of the two tile widths
  return (size_t)(rows * nt) * rec_bytes_(k);
}

cudaError_t launch_proj_topk(const void* h, long long rows, long long D, const void* w, long long V, int k,
                             float* vals, long long* idx, void* ws, cudaStream_t st) {
  if (k <= 1) return run_proj<1>(h, rows, D, w, V, k, vals, idx, ws, st);
  if (k <= 5) return run_proj<5>(h, rows, D, w, V, k, vals, idx, ws, st);
  if (k <= 8) return run_proj<8>(h, rows, D, w, V, k, vals, idx, ws, st);
  if (k <= 16) return run_proj<16>(h, rows, D, w, V, k, vals, idx, ws, st);
  return run_proj<32>(h, rows, D, w, V, k, vals, idx, ws, st);
}

}  // namespace osmx_host
