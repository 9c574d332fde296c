// common.cuh -- shared device helpers: the job-id <-> coordinate bijection
// and the PTX wrappers (cp.async, FP64 mma.sync) the kernels use.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace pcc {

// Cells (or tiles) strictly above row y of the upper triangle of an m x m
// matrix: F(y) = y(2m - y + 1)/2 (indexing.py:55-64).  Unsigned 64-bit: the
// product y(2m-y+1) stays below 2^64 for m < 2^32 (indexing.py:40 MAX_N).
__host__ __device__ __forceinline__ uint64_t row_prefix(uint64_t m, uint64_t y) {
  return y * (2 * m - y + 1) / 2;
}

// Row of tile/job `id` in the m x m upper triangle: the reference's closed
// form y = ceil(m - 0.5 - sqrt(m^2 + m + 0.25 - 2(id+1))) evaluated in FP64,
// clamped, then walked to the exact row by integer bracket checks
// (_kernels.py:301-319, indexing.py:97-109).
__host__ __device__ __forceinline__ uint64_t tile_row(uint64_t m, uint64_t id) {
  double mf = (double)m;
  double disc = mf * mf + mf + 0.25 - 2.0 * ((double)id + 1.0);
  int64_t y = disc >= 0.0 ? (int64_t)ceil(mf - 0.5 - sqrt(disc)) : (int64_t)m - 1;
  if (y < 0) y = 0;
  if (y > (int64_t)m - 1) y = (int64_t)m - 1;
  while (y > 0 && id < row_prefix(m, (uint64_t)y)) --y;
  while (id >= row_prefix(m, (uint64_t)y + 1)) ++y;
  return (uint64_t)y;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte global -> shared asynchronous copy (LDGSTS), L2-only caching.
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D(8x8) += A(8x4) * B(4x8), FP64 on the tensor pipe (SASS DMMA.8x8x4).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// {c0, c1} = C[lane/4][2*(lane%4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void dmma_8x8x4_v(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) primitives ---------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 2-D TMA tile load global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int32_t c0, int32_t c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace pcc
