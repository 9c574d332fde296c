// tcgen05.cuh -- PTX wrappers for the 5th-generation tensor core path
// (tcgen05.mma kind::i8 with accumulators in tensor memory) used by the
// split-integer contraction (split.cuh).
//
// Descriptor encodings (sm_100a):
//   * shared-memory matrix descriptor, 64 bit: start address >> 4 [0,14),
//     leading-byte-offset >> 4 [16,30), stride-byte-offset >> 4 [32,46),
//     version = 1 [46,48), base offset [49,52), layout type [61,64)
//     (0 none, 2 = 128B swizzle, 4 = 64B, 6 = 32B);
//   * instruction descriptor, 32 bit: D format [4,6) (2 = s32), A format
//     [7,10) and B format [10,13) (1 = signed 8-bit), A/B major [15]/[16]
//     (0 = K-major), N >> 3 [17,23), M >> 4 [24,29).
// Operands here are always K-major with the 32-byte swizzle: a row holds 32
// int8 (one MMA K step), 8-row atoms of 256 B, atoms packed back to back
// (SBO = 256 B) -- exactly what a TMA box {32 B, rows} with
// CU_TENSOR_MAP_SWIZZLE_32B writes.
#pragma once

#include <cstdint>

namespace pcc {

__device__ __forceinline__ uint64_t umma_desc_k_sw32(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;           // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;                    // SWIZZLE_32B
  return d;
}

// K-major, 64-byte swizzle: rows of 64 bytes (two int8 MMA K steps), 8-row
// atoms of 512 B packed back to back (SBO = 512 B) -- what a TMA box
// {64 B, rows} with CU_TENSOR_MAP_SWIZZLE_64B writes; the second K step of a
// row starts 32 B further (the swizzle is a function of the address bits).
__device__ __forceinline__ uint64_t umma_desc_k_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;           // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                    // SWIZZLE_64B
  return d;
}

template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_i8_s32() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, one elected thread issues.
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// Whole warp: allocate `cols` TMEM columns, base address written to smem.
__device__ __forceinline__ void tmem_alloc(uint32_t smem_dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_dst), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols) : "memory");
}

// Warp-collective: lane i of the warp reads TMEM lane (taddr.lane + i),
// 16 consecutive 32-bit columns starting at taddr.col.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

}  // namespace pcc
