// normalize.cuh -- K1: per-variable z-normalisation, bit-exact to the
// reference's _kernels.normalize_rows (_kernels.py:226-252).
//
// Arithmetic contract (what makes it bit-exact):
//   * sum8 / ssd8 (_kernels.py:71-165): lane j (0..7) accumulates elements
//     k = j (mod 8) in increasing k, then ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)).
//     Here each row is owned by an 8-thread group; thread j of the group IS
//     reference lane j and runs its chain sequentially; the tree is three
//     xor-shuffles (1, 2, 4), which pair lanes exactly as the tree does
//     (IEEE addition is commutative, so a+b and b+a are the same bits).
//   * every multiply/add is __dmul_rn/__dadd_rn/__dsub_rn: the compiler may
//     not contract them into FMA (the reference never fuses).
//   * mean = sum / l, scale = sqrt(ssd), u = (x - mean) / scale are IEEE
//     round-to-nearest division / sqrt (__ddiv_rn, __dsqrt_rn).
//   * zero variance: exact all-equal-to-first test (_kernels.py:209-223)
//     folded into the sum pass, plus the ssd == 0.0 guard (:244-247).
//
// Memory: one warp = 4 rows x 8 lanes; each load instruction reads 64
// contiguous bytes per row (full 32-byte sectors).  The row is read twice
// (sum, ssd) and once more to write U; the re-reads are served by L1/L2.
// Algorithmic traffic is 1 read of X + 1 write of U (HBM-bound kernel).
#pragma once

#include "common.cuh"

namespace pcc {

constexpr int kNormThreads = 256;
constexpr int kNormRowsPerCta = kNormThreads / 8;

__global__ void __launch_bounds__(kNormThreads)
normalize_rows_kernel(const double *__restrict__ x, int64_t ldx, double *__restrict__ u, int64_t ldu,
                      uint8_t *__restrict__ zero_variance, int64_t l, int64_t row_lo, int64_t row_hi) {
  const int lane8 = threadIdx.x & 7;
  const int64_t row = row_lo + (int64_t)blockIdx.x * kNormRowsPerCta + (threadIdx.x >> 3);
  const bool active = row < row_hi;
  // Shuffles below use the full warp; inactive groups compute on row_lo's
  // data (valid memory) and never store.
  const int64_t r = active ? row : row_lo;
  const double *xr = x + r * ldx;
  double *ur = u + r * ldu;

  // Pass 1: lane sum (sum8 order) + exact constancy test.
  const double first = xr[0];
  double s = 0.0;
  bool varies = false;
  int64_t k = lane8;
#pragma unroll 4
  for (; k < l; k += 8) {
    double v = __ldg(xr + k);
    s = __dadd_rn(s, v);
    varies |= (v != first);
  }
  // Tree ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)) inside each 8-lane group.
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  const unsigned vb = __ballot_sync(0xffffffffu, varies);
  const unsigned group_mask = 0xffu << (threadIdx.x & 24);
  const bool constant = (vb & group_mask) == 0u;

  double ssd = 0.0, mean = 0.0;
  if (!constant) {  // uniform within the 8-lane group
    mean = __ddiv_rn(s, (double)l);
    double q = 0.0;
    for (k = lane8; k < l; k += 8) {
      double d = __dsub_rn(__ldg(xr + k), mean);
      q = __dadd_rn(q, __dmul_rn(d, d));
    }
    ssd = q;
  }
  // Every lane of the warp reaches this point (constant groups carry 0.0).
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 1));
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 2));
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 4));

  if (!active) return;
  const bool zero = constant || ssd == 0.0;
  if (lane8 == 0) zero_variance[row] = zero ? 1 : 0;
  if (zero) {
    for (k = lane8; k < ldu; k += 8) ur[k] = 0.0;
    return;
  }
  const double scale = __dsqrt_rn(ssd);
  for (k = lane8; k < l; k += 8) ur[k] = __ddiv_rn(__dsub_rn(__ldg(xr + k), mean), scale);
  for (k = l + lane8; k < ldu; k += 8) ur[k] = 0.0;
}

// ---------------------------------------------------------------------------
// Shared-memory-staged variant (the default when R >= 1 rows of l doubles
// fit the per-CTA budget): X is read from HBM exactly once.
//   1. all 256 threads stream R rows into shared memory with 8-byte
//      cp.async (any l / ldx alignment), many copies in flight per thread;
//   2. 8 threads per row run the reference's lane chains (sum + constancy,
//      then ssd) out of shared memory and finish with the shuffle tree;
//   3. all threads write u = (x - mean) / scale (or the zero row) back with
//      coalesced stores, plus the zero K padding up to ldu.
// Two CTAs per SM (<= ~100 KB each) overlap one CTA's chains with the
// other's copies.  Same arithmetic as normalize_rows_kernel, bit for bit.
constexpr int kNormSmemBudget = 100 * 1024;

__device__ __forceinline__ void cp_async_8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
}

__global__ void __launch_bounds__(kNormThreads)
normalize_rows_smem_kernel(const double *__restrict__ x, int64_t ldx, double *__restrict__ u, int64_t ldu,
                           uint8_t *__restrict__ zero_variance, int64_t l, int64_t row_lo, int64_t row_hi,
                           int rows_per_cta) {
  extern __shared__ __align__(16) double srow[];  // [rows_per_cta][l]
  __shared__ double s_mean[kNormRowsPerCta], s_scale[kNormRowsPerCta];
  __shared__ int s_zero[kNormRowsPerCta];
  const int tid = threadIdx.x;
  const int64_t r0 = row_lo + (int64_t)blockIdx.x * rows_per_cta;
  const int rows = (int)((row_hi - r0) < (int64_t)rows_per_cta ? (row_hi - r0) : (int64_t)rows_per_cta);
  const uint32_t sbase = smem_u32(srow);

  // 1. stage the rows
  for (int r = 0; r < rows; ++r) {
    const double *xr = x + (r0 + r) * ldx;
    const uint32_t sr = sbase + (uint32_t)(r * l * sizeof(double));
    for (int64_t k = tid; k < l; k += kNormThreads) cp_async_8(sr + (uint32_t)(k * sizeof(double)), xr + k);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // 2. lane chains: thread (row = tid / 8, lane8 = tid % 8)
  const int lane8 = tid & 7;
  const int row = tid >> 3;
  const bool active = row < rows;
  const double *sr = srow + (int64_t)(active ? row : 0) * l;
  const double first = sr[0];
  double s = 0.0;
  bool varies = false;
  int64_t k = lane8;
#pragma unroll 8
  for (; k < l; k += 8) {
    const double v = sr[k];
    s = __dadd_rn(s, v);
    varies |= (v != first);
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  const unsigned vb = __ballot_sync(0xffffffffu, varies);
  const bool constant = (vb & (0xffu << (tid & 24))) == 0u;
  double mean = 0.0, ssd = 0.0;
  if (!constant) {
    mean = __ddiv_rn(s, (double)l);
    double q = 0.0;
#pragma unroll 8
    for (k = lane8; k < l; k += 8) {
      const double d = __dsub_rn(sr[k], mean);
      q = __dadd_rn(q, __dmul_rn(d, d));
    }
    ssd = q;
  }
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 1));
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 2));
  ssd = __dadd_rn(ssd, __shfl_xor_sync(0xffffffffu, ssd, 4));
  if (active && lane8 == 0) {
    const bool zero = constant || ssd == 0.0;
    s_zero[row] = zero;
    s_mean[row] = mean;
    s_scale[row] = zero ? 0.0 : __dsqrt_rn(ssd);
    zero_variance[r0 + row] = zero ? 1 : 0;
  }
  __syncthreads();

  // 3. write U rows (coalesced), zero rows for zero variance, zero K padding
  for (int r = 0; r < rows; ++r) {
    double *ur = u + (r0 + r) * ldu;
    const double *xs = srow + (int64_t)r * l;
    if (s_zero[r]) {
      for (k = tid; k < ldu; k += kNormThreads) ur[k] = 0.0;
    } else {
      const double m = s_mean[r], sc = s_scale[r];
      for (k = tid; k < l; k += kNormThreads) ur[k] = __ddiv_rn(__dsub_rn(xs[k], m), sc);
      for (k = l + tid; k < ldu; k += kNormThreads) ur[k] = 0.0;
    }
  }
}

}  // namespace pcc
