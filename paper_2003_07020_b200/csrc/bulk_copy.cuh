// bulk_copy.cuh -- Blackwell bulk-copy staging (cp.async.bulk, SASS UBLKCP) with mbarrier
// completion, for the warp-owned row kernels: one lane of a group issues the copy of a whole row
// (or a 16-byte aligned superset of it) from global into shared memory; the group's lanes wait on
// the mbarrier's phase and then read their transform inputs from shared memory.  One memory round
// trip per row, issued by the copy engine instead of 16..48 register loads per lane.
#pragma once
#include <cstdint>

namespace fpc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make the initialised barrier visible to the async (copy-engine) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// generic-proxy shared-memory accesses before a later bulk copy into the same bytes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// global -> shared bulk copy; dst, src and bytes must be 16-byte multiples / aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Per-thread asynchronous copies (cp.async, SASS LDGSTS) for staging column tiles: a thread issues
// its whole share of a tile, then waits once (cp_async_wait_all), so everything it copies is in flight
// together instead of a register-limited batch.  ok = false writes zeros (rows / columns past the
// edge) without reading src; src must still be a valid address.
__device__ __forceinline__ void cp_async8_zfill(void* smem_dst, const void* src, bool ok) {
  const int bytes = ok ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem_dst)), "l"(src), "r"(bytes)
               : "memory");
}
// dst and src 16-byte aligned
__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* src, bool ok) {
  const int bytes = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

}  // namespace fpc
