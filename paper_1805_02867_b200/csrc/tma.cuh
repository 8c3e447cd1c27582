// tma.cuh -- Blackwell bulk-copy (TMA, cp.async.bulk) + mbarrier helpers for
// the shared-memory staged streaming kernels.
//
// A CTA owns a ring of STAGES shared-memory buffers.  One producer thread
// issues 1-D bulk copies global -> shared (UBLKCP in SASS) that complete on
// the stage's "full" mbarrier with a transaction byte count; consumer warps
// wait on "full", read the stage with LDS.128, and arrive on the stage's
// "empty" mbarrier so the producer can refill it.  The bytes in flight per
// SM are set by the ring size, not by registers, and the producer keeps
// streaming the next row while consumers reduce / merge the current one.
#pragma once

#include <cstdint>

namespace osmx_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Make the barrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
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

// 1-D bulk copy global -> shared, completing `bytes` transactions on `bar`.
// src, dst 16-byte aligned, bytes a multiple of 16.  Evict-first L2 policy:
// every input line is read exactly once.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Named barrier over the consumer warps only (the producer warp never joins).
// The non-.aligned barrier.sync: arrival is per thread, so a warp that is
// still diverged from a lane-0-only store or an mbarrier wait loop is
// counted correctly (bar.sync = barrier.sync.aligned requires a converged
// warp; the compiler need not reconverge before it).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace osmx_dev
