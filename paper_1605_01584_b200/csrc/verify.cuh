// verify.cuh -- GPU restatement of the reference's brute-force oracle
// (Eq. (1) of the paper): _kernels.pcc_naive_pair / naive_allpairs_packed /
// constant_row_flags (_kernels.py:255-298), bit for bit.
//
// The reference recomputes both rows' statistics for every pair; the values
// it computes per row (is_constant, mean = sum8/l, ssd = ssd8(x, mean)) do
// not depend on the partner, so they are computed once per row here
// (row_stats_kernel) and reused -- the per-pair arithmetic and its order are
// unchanged: covar8 lanes, the fixed tree, then
//   0.0 if either row is constant or either ssd == 0.0,
//   else covar / (sqrt(ssd_a) * sqrt(ssd_b))        (IEEE, no FMA).
// This is the product's `verify` (fileio.py:314-367) at GPU speed; it shares
// no code path with the normalise + contraction engine it checks.
#pragma once

#include "normalize.cuh"

namespace pcc {

// Per-row is_constant, mean and ssd in the reference's order.
__global__ void __launch_bounds__(256)
row_stats_kernel(const double *__restrict__ x, int64_t ldx, int64_t l, int64_t n, double *__restrict__ mean,
                 double *__restrict__ ssd, uint8_t *__restrict__ constant) {
  const int lane8 = threadIdx.x & 7;
  const int64_t row = (int64_t)blockIdx.x * 32 + (threadIdx.x >> 3);
  const bool active = row < n;
  const double *xr = x + (active ? row : 0) * ldx;
  const int64_t nsteps = (l - lane8 + 7) >> 3;
  bool varies = false;
  double s = lane_chain<false, 16>(xr + lane8, nsteps, xr[0], varies);
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  const unsigned vb = __ballot_sync(0xffffffffu, varies);
  const bool cst = (vb & (0xffu << (threadIdx.x & 24))) == 0u;
  // the reference computes mean/ssd only for non-constant rows; the values of
  // a constant row are never used (the pair returns 0.0 first)
  const double m = __ddiv_rn(s, (double)l);
  bool unused = false;
  double q = lane_chain<true, 16>(xr + lane8, nsteps, m, unused);
  q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 1));
  q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 2));
  q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 4));
  if (active && lane8 == 0) {
    mean[row] = m;
    ssd[row] = q;
    constant[row] = cst ? 1 : 0;
  }
}

// pcc_naive_pair for packed job ids [id_lo, id_hi) of the n x n triangle;
// one 8-lane group per pair (lane j = reference lane j of covar8).
__global__ void __launch_bounds__(256)
naive_pairs_kernel(const double *__restrict__ x, int64_t ldx, int64_t l, int64_t n,
                   const double *__restrict__ mean, const double *__restrict__ ssd,
                   const uint8_t *__restrict__ constant, uint64_t id_lo, uint64_t id_hi, double *__restrict__ out) {
  const int lane8 = threadIdx.x & 7;
  const int group = (threadIdx.x & 31) >> 3;  // 4 pairs per warp
  const uint64_t warp = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t count = id_hi - id_lo;
  for (uint64_t base = warp * 4; base < count; base += warps * 4) {  // warp-uniform
    const uint64_t rel = base + group;
    const bool active = rel < count;
    const uint64_t id = id_lo + (active ? rel : 0);
    const uint64_t y = tile_row((uint64_t)n, id);
    const uint64_t xc = id + y - row_prefix((uint64_t)n, y);
    const double *a = x + (int64_t)y * ldx;
    const double *b = x + (int64_t)xc * ldx;
    const double ma = mean[y], mb = mean[xc];
    double s = 0.0;
    for (int64_t k = lane8; k < l; k += 8) {
      const double p = __dmul_rn(__dsub_rn(a[k], ma), __dsub_rn(b[k], mb));
      s = __dadd_rn(s, p);
    }
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    if (active && lane8 == 0) {
      double r;
      if (constant[y] || constant[xc]) {
        r = 0.0;
      } else {
        const double sa = ssd[y], sb = ssd[xc];
        r = (sa == 0.0 || sb == 0.0) ? 0.0 : __ddiv_rn(s, __dmul_rn(__dsqrt_rn(sa), __dsqrt_rn(sb)));
      }
      out[rel] = r;
    }
  }
}

}  // namespace pcc
