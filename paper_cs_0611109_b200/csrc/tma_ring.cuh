// tma_ring.cuh -- the PTX pieces of the TMA producer/consumer ring shared by the fast kernel
// (zp_fast.cuh) and the TMA-staged generic kernel (zp_generic.cuh): mbarriers, 1-D bulk copies
// global <-> shared (cp.async.bulk), bulk groups, proxy fences, named barriers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace zp {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: the waiting thread sleeps in the barrier unit until the
// phase completes (or the hint expires) instead of re-polling -- fewer issued instructions on
// the consumers' waits for TMA data.
#ifndef ZP_NO_WAIT_HINT
#define ZP_TRY_WAIT "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 0x989680;\n\t"
#else  // A/B control: plain try_wait polling
#define ZP_TRY_WAIT "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "ZP_WAIT_%=:\n\t" ZP_TRY_WAIT
      "@!P1 bra ZP_WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// The same on a precomputed shared-space address (the consumers' per-row wait and release: no
// generic-to-shared conversion per row).
__device__ __forceinline__ void mbar_wait_sa(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "ZP_WAITS_%=:\n\t" ZP_TRY_WAIT
      "@!P1 bra ZP_WAITS_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_sa(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_row(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// Consumer side of a TMA stage release: this thread's generic-proxy reads of the stage (LDS) are
// ordered before the async-proxy write (the producer's next cp.async.bulk into the stage) by a
// proxy fence -- a write-after-read across proxies; the LDS results are otherwise free to land
// after the arrive, and the compiler may schedule their consumers after it (a long bench run
// of the r02 fold once came back with 3 KB rebuilt wrong).  __syncwarp then gathers the lanes
// and lane 0 arrives on the stage's `empty` barrier (count = consumer warps).
__device__ __forceinline__ void consumer_release(uint32_t empty_bar_sa, int lane) {
#ifndef ZP_NO_RELEASE_FENCE  // (negative control only)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
  __syncwarp();
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty_bar_sa) : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace zp
