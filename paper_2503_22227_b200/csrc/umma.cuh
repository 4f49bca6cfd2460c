// Inline-PTX wrappers for the 5th-generation tensor cores (tcgen05) on
// sm_100a: TMEM allocation, shared-memory matrix descriptors, the u8 x u8 ->
// s32 MMA (kind::i8) with the accumulator in TMEM, commit to an mbarrier,
// and TMEM -> register loads for the epilogue.
//
// Operand layout (both A = M x K and B = N x K, K-major, no swizzle): the
// canonical "interleaved" core-matrix layout -- a core matrix is 8 rows x 16
// bytes stored contiguously (128 B); core matrices adjacent in M/N are SBO
// bytes apart, those adjacent in K (the two 16-byte halves of one K = 32
// byte MMA step) LBO bytes apart.  Here a tile with G row groups of 8 rows
// is stored [k16 chunk][row group][8 rows][16 B], so SBO = 128 and
// LBO = 128 G, and K step j starts 2 j chunks in.
#pragma once
#include <cstdint>

__device__ __forceinline__ unsigned umma_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start
// address, LBO and SBO in 16-byte units; bits 46-47 = 1 (sm_100 version);
// base offset 0, legacy LBO mode, layout type 0 = no swizzle
__device__ __forceinline__ uint64_t umma_desc(unsigned saddr, unsigned lbo, unsigned sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A and B u8 (format
// 0), both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr unsigned umma_idesc_u8(int m, int n) {
  return (2u << 4) | ((unsigned)(n >> 3) << 17) | ((unsigned)(m >> 4) << 24);
}

__device__ __forceinline__ void tmem_alloc(unsigned* dst_smem, unsigned ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   umma_smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned taddr, unsigned ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void umma_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D[tmem] (+)= A[adesc] * B[bdesc]^T, one K = 32 byte step
__device__ __forceinline__ void umma_u8(unsigned tmem_d, uint64_t adesc, uint64_t bdesc,
                                        unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier once every MMA issued so far by this thread is done
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          umma_smem_u32(bar))
      : "memory");
}

// lane (32 (warp % 4) + laneid) of TMEM, 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld8(unsigned taddr, unsigned (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void umma_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma_smem_u32(bar)), "r"(count));
}
// try_wait with a suspend-time hint: the waiting thread sleeps until the
// phase completes (or the hint expires) instead of spinning on the barrier
#ifndef FHE_UMMA_WAIT_HINT
#define FHE_UMMA_WAIT_HINT 0x989680
#endif
__device__ __forceinline__ void umma_mbar_wait(uint64_t* bar, unsigned phase) {
#if FHE_UMMA_WAIT_HINT
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "UMMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra UMMA_WAIT_%=;\n\t}" ::"r"(umma_smem_u32(bar)),
      "r"(phase), "n"(FHE_UMMA_WAIT_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "UMMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra UMMA_WAIT_%=;\n\t}" ::"r"(umma_smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}
__device__ __forceinline__ void umma_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma_smem_u32(bar)) : "memory");
}
