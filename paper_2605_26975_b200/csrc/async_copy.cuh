// Shared-memory / asynchronous-copy helpers for sm_100a: mbarriers, TMA bulk copies
// (cp.async.bulk, SASS UBLKCP), L2 bulk prefetch and Ampere-style cp.async (LDGSTS).
#pragma once
#include <cstdio>
// Device-side bounds / protocol checks of a debug build (-DPLP_DEBUG_CHECKS; tools/tune_edge.py
// variant `checked`): compute-sanitizer is unavailable on the GPU pool, so the kernels' shared-
// memory indexing and copy sizes are asserted in-kernel instead.  Free in the product build.
#ifdef PLP_DEBUG_CHECKS
#define PLP_DCHECK(cond, what)                                                                  \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("PLP_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define PLP_DCHECK(cond, what) do {} while (0)
#endif
#include <cstdint>

namespace plp {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  // try_wait with a suspend-time hint: the warp sleeps in hardware until the phase completes (or
  // the hint expires) instead of spinning, so waiting warps do not take issue slots from the
  // computing warps of their SM sub-partition
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// Polling wait with a sleep between polls: for a producer warp that has slack, so that its spinning
// does not take issue slots from the compute warps of its SM sub-partition.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity, unsigned ns) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* src, unsigned bytes) {  // bytes % 16 == 0
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// L2 prefetch of an arbitrary byte range [src, src + bytes): widened to 16-byte alignment (the
// bulk prefetch requires it; the arrays are padded, and a prefetch never faults the kernel's data)
__device__ __forceinline__ void l2_prefetch_range(const void* src, size_t bytes) {
  const uintptr_t a = (uintptr_t)src & ~(uintptr_t)15;
  const uintptr_t e = ((uintptr_t)src + bytes + 15) & ~(uintptr_t)15;
  if (e > a) l2_prefetch(reinterpret_cast<const void*>(a), (unsigned)(e - a));
}
// TMA row gather (sm_100 tile::gather4): rows r0..r3, columns [c0, c0 + box width) of the 2-D
// tensor described by `tmap` (a __grid_constant__ CUtensorMap) land densely at dst (128-byte
// aligned); completion counts bytes on `bar`.  One instruction, one thread, no LSU traffic.
__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrives on `bar` once all of this thread's prior cp.async copies have completed (no pending-count
// increment: the arrival counts against the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_staged() {  // all but the most recent group
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {  // at most N of this thread's groups pending
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace plp
