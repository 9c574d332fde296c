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

// Processing order of a contiguous tile-id range [tb, te) (the partition
// unit).  The SET of tiles is fixed by the bijection; only the order in
// which a persistent grid visits them is chosen for L2 locality:
//   head  [tb, head_end)          partial first tile row, id order
//   body  full rows [body_lo, body_hi) in groups of `group` rows, each group
//         walked column by column (rows of a column consecutive), so a wave
//         of concurrent CTAs shares ~group A bands and ~wave/group B bands
//   tail  [tail_begin, te)        partial last tile row, id order
// Every cell's arithmetic is independent of the order (no split-K), so the
// result is bitwise identical to the plain id order.
struct TileOrder {
  uint64_t tb, head_end, body_lo, body_hi, body_count, tail_begin, te, total;
  uint32_t group;
};

__host__ __device__ inline TileOrder make_tile_order(uint64_t m, uint64_t tb, uint64_t te, uint32_t group) {
  TileOrder o{};
  o.tb = tb;
  o.te = te;
  o.total = te > tb ? te - tb : 0;
  o.group = group < 1 ? 1 : group;
  o.head_end = tb;
  o.body_lo = o.body_hi = 0;
  o.body_count = 0;
  o.tail_begin = te;
  if (te <= tb) return o;
  const uint64_t y0 = tile_row(m, tb), y1 = tile_row(m, te - 1);
  if (y0 == y1) {
    o.head_end = te;
    return o;
  }
  const bool head_full = tb == row_prefix(m, y0);
  const bool tail_full = te == row_prefix(m, y1 + 1);
  o.head_end = head_full ? tb : row_prefix(m, y0 + 1);
  o.body_lo = head_full ? y0 : y0 + 1;
  o.body_hi = tail_full ? y1 + 1 : y1;
  o.tail_begin = tail_full ? te : row_prefix(m, y1);
  o.body_count = o.body_hi > o.body_lo ? row_prefix(m, o.body_hi) - row_prefix(m, o.body_lo) : 0;
  return o;
}

// Schedule index s in [0, o.total) -> tile coordinate (Y, X).
__host__ __device__ inline void tile_at(const TileOrder &o, uint64_t m, uint64_t s, uint64_t &Y, uint64_t &X) {
  const uint64_t head = o.head_end - o.tb;
  uint64_t J;
  if (s < head) {
    J = o.tb + s;
  } else if (s - head < o.body_count) {
    uint64_t r = s - head;
    uint64_t ya = o.body_lo;
    uint64_t g = 0;
    for (;;) {
      g = o.body_hi - ya < o.group ? o.body_hi - ya : o.group;
      const uint64_t size = g * (m - ya) - g * (g - 1) / 2;
      if (r < size) break;
      r -= size;
      ya += g;
    }
    const uint64_t corner = g * (g - 1) / 2;  // columns ya .. ya+g-2 hold 1 .. g-1 tiles
    if (r < corner) {
      // column q (0-based from ya) holds q+1 tiles; triangular-number inverse
      uint64_t q = (uint64_t)((sqrt(8.0 * (double)r + 1.0) - 1.0) * 0.5);
      while (q * (q + 1) / 2 > r) --q;
      while ((q + 1) * (q + 2) / 2 <= r) ++q;
      X = ya + q;
      Y = ya + (r - q * (q + 1) / 2);
    } else {
      const uint64_t r2 = r - corner;
      X = ya + g - 1 + r2 / g;
      Y = ya + r2 % g;
    }
    return;
  } else {
    J = o.tail_begin + (s - head - o.body_count);
  }
  Y = tile_row(m, J);
  X = J + Y - row_prefix(m, Y);
}

// Split-mode digits (split.cuh): the 7 balanced radix-128 digits of v in
// (-128, 128), d_i = rint(128^i r_i) with r_0 = v, r_{i+1} = r_i - d_i 128^-i
// (round to nearest, ties to even; every step exact).  Written with the shift
// constants C_i = 1.5 * 2^(52 - 7i): t = RN(r + C_i) rounds r to a multiple of
// 128^-i, so the digit is the low byte of t's bit pattern and t - C_i is
// d_i 128^-i exactly -- three FP64 operations per digit.  Digit i of
// element j (0..3) goes to byte j of packed[i].
__device__ __forceinline__ void split_digits7(double v, int j, uint32_t packed[7]) {
  constexpr double C[7] = {0x1.8p52, 0x1.8p45, 0x1.8p38, 0x1.8p31, 0x1.8p24, 0x1.8p17, 0x1.8p10};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    const double t = __dadd_rn(v, C[i]);
    v = __dsub_rn(v, __dsub_rn(t, C[i]));
    packed[i] |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * j);
  }
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
