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

}  // namespace pcc
