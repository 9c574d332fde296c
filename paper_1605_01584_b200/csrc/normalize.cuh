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

// ---------------------------------------------------------------------------
// One reference reduction lane, software-pipelined: the next PF elements of
// the lane (stride 8) are loaded while the current PF are added, so the
// dependent add chain -- which the reference's order makes inherently
// sequential -- runs at FP64-add latency instead of load latency.
// SSD = false: sum8 lane + constancy test against `ref` (= x[0]);
// SSD = true:  ssd8 lane with `ref` = mean.
template <bool SSD, int PF, bool DMAX = false>
__device__ __forceinline__ double lane_chain(const double *p, int64_t nsteps64, double ref, bool &varies,
                                             double *dmax = nullptr) {
  const int nsteps = (int)nsteps64;
  const int full = (nsteps / PF) * PF;
  double s = 0.0;
  double nxt[PF];
  if (full > 0) {
#pragma unroll
    for (int i = 0; i < PF; ++i) nxt[i] = p[8 * i];
  }
  int t = 0;
  for (; t < full; t += PF) {
    double cur[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) cur[i] = nxt[i];
    if (t + PF < full) {
#pragma unroll
      for (int i = 0; i < PF; ++i) nxt[i] = p[8 * (t + PF + i)];
    }
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      if (SSD) {
        const double d = __dsub_rn(cur[i], ref);
        s = __dadd_rn(s, __dmul_rn(d, d));
        if (DMAX) *dmax = fmax(*dmax, fabs(d));
      } else {
        s = __dadd_rn(s, cur[i]);
        varies |= (cur[i] != ref);
      }
    }
  }
  for (; t < nsteps; ++t) {
    const double v = p[8 * t];
    if (SSD) {
      const double d = __dsub_rn(v, ref);
      s = __dadd_rn(s, __dmul_rn(d, d));
      if (DMAX) *dmax = fmax(*dmax, fabs(d));
    } else {
      s = __dadd_rn(s, v);
      varies |= (v != ref);
    }
  }
  return s;
}

// Pure lane chains over already-prepared values (stride 8): SQUARE = false
// sums v, SQUARE = true sums RN(v*v) -- the sum8 / ssd8 lane accumulations
// once the constancy test and the centring (d = x - mean) have been done by
// all threads in parallel.  One FP64 add (and one multiply) per step on the
// dependent chain; loads run PF steps ahead.
template <bool SQUARE, int PF>
__device__ __forceinline__ double lane_sum(const double *p, int nsteps) {
  const int full = (nsteps / PF) * PF;
  double s = 0.0;
  double nxt[PF];
  if (full > 0) {
#pragma unroll
    for (int i = 0; i < PF; ++i) nxt[i] = p[8 * i];
  }
  int t = 0;
  for (; t < full; t += PF) {
    double cur[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) cur[i] = nxt[i];
    if (t + PF < full) {
#pragma unroll
      for (int i = 0; i < PF; ++i) nxt[i] = p[8 * (t + PF + i)];
    }
#pragma unroll
    for (int i = 0; i < PF; ++i) s = __dadd_rn(s, SQUARE ? __dmul_rn(cur[i], cur[i]) : cur[i]);
  }
  for (; t < nsteps; ++t) {
    const double v = p[8 * t];
    s = __dadd_rn(s, SQUARE ? __dmul_rn(v, v) : v);
  }
  return s;
}

// One reference lane chain over a whole shared-memory row (stride 8),
// straight-line in 64-step blocks with the loads two 8-step batches ahead of
// the dependent adds (~14.7 cycles per step on B200 vs ~17 for the
// software-pipelined loop above, tools/k1s2_probe.cu EXP 9):
//   SSD = false: s += x (sum8 lane);  SSD = true: d = x - ref (the mean),
//   s += RN(d * d) (ssd8 lane).  The constancy test is not on this chain.
template <bool SSD, bool CONST = false>
__device__ __forceinline__ void chain64(double &s, const double *p, double ref, bool &varies) {
  double v[3][8];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[b][i] = p[8 * (8 * b + i)];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    if (b + 2 < 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[(b + 2) % 3][i] = p[8 * (8 * (b + 2) + i)];
    }
    const double *cur = v[b % 3];
    if (SSD) {
      double d[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = __dsub_rn(cur[i], ref);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __dadd_rn(s, __dmul_rn(d[i], d[i]));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s = __dadd_rn(s, cur[i]);
        if (CONST) varies |= cur[i] != ref;
      }
    }
  }
}
// CONST (sum chain only): also the exact constancy test x != ref (= x[0]).
template <bool SSD, bool CONST = false>
__device__ __forceinline__ double row_chain(const double *p, int nsteps, double ref, bool &varies) {
  double s = 0.0;
  int t = 0;
  for (; t + 64 <= nsteps; t += 64) chain64<SSD, CONST>(s, p + 8 * t, ref, varies);
  for (; t < nsteps; ++t) {
    const double v = p[8 * t];
    if (SSD) {
      const double d = __dsub_rn(v, ref);
      s = __dadd_rn(s, __dmul_rn(d, d));
    } else {
      s = __dadd_rn(s, v);
      if (CONST) varies |= v != ref;
    }
  }
  return s;
}

// The same lane chain continued from s over nsteps more elements (chunked
// kernel: a row's chain runs across shared-memory chunks).
template <bool SSD, bool CONST = false>
__device__ __forceinline__ void row_chain_more(double &s, const double *p, int nsteps, double ref, bool &varies) {
  int t = 0;
  for (; t + 64 <= nsteps; t += 64) chain64<SSD, CONST>(s, p + 8 * t, ref, varies);
  for (; t < nsteps; ++t) {
    const double v = p[8 * t];
    if (SSD) {
      const double d = __dsub_rn(v, ref);
      s = __dadd_rn(s, __dmul_rn(d, d));
    } else {
      s = __dadd_rn(s, v);
      if (CONST) varies |= v != ref;
    }
  }
}

// u = a / b bit-identical to IEEE division (__ddiv_rn), one FMA correction
// instead of a full division per element: with y = RN(1/b) (one __drcp_rn
// per row) and q0 = RN(a y), q = RN(q0 + (a - b q0) y) is the correctly rounded
// quotient (Markstein's correction step; a - b q0 is exact by FMA) as long as
// no intermediate underflows -- guarded here to |a| >= 2^-520 and b in
// [2^-500, 2^500]; everything else (zeros, huge or tiny values) takes
// __ddiv_rn.  tools/div_check.cu compares the two on 3e10 random pairs.
struct RowDiv {
  double b, y;
  bool fast;
};
__device__ __forceinline__ RowDiv row_div(double b) {
  return RowDiv{b, __drcp_rn(b), b >= 0x1p-500 && b <= 0x1p500};
}
__device__ __forceinline__ double div_rn(double a, const RowDiv &d) {
  if (d.fast && fabs(a) >= 0x1p-520) {
    const double q0 = __dmul_rn(a, d.y);
    return __fma_rn(__fma_rn(-q0, d.b, a), d.y, q0);
  }
  return __ddiv_rn(a, d.b);
}
// The same quotient without the per-element branch (the branch and the
// inlined IEEE fallback made the output loops ~2.5x slower, tools/
// k1c_probe.cu): the guard is tested on the bits of a and collected in
// `bad` -- +0 is exact here, -0 and |a| < 2^-520 (subnormals included) are
// not -- and a caller whose `bad` is set anywhere writes its block again with
// __ddiv_rn.  Rows whose scale fails the range test (!d.fast) take __ddiv_rn
// throughout.
__device__ __forceinline__ double div_fast(double a, const RowDiv &d, bool &bad) {
  const double q0 = __dmul_rn(a, d.y);
  const int hi = __double2hiint(a), lo = __double2loint(a);
  bad |= ((hi & 0x7fffffff) < ((1023 - 520) << 20)) & ((hi | lo) != 0);
  return __fma_rn(__fma_rn(-q0, d.b, a), d.y, q0);
}

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
  const int64_t nsteps = (l - lane8 + 7) >> 3;
  bool varies = false;
  double s = lane_chain<false, 16>(xr + lane8, nsteps, xr[0], varies);
  int64_t k;
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
    bool unused = false;
    ssd = lane_chain<true, 16>(xr + lane8, nsteps, mean, unused);
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
  const RowDiv dv = row_div(scale);
  for (k = lane8; k < l; k += 8) ur[k] = div_rn(__dsub_rn(__ldg(xr + k), mean), dv);
  for (k = l + lane8; k < ldu; k += 8) ur[k] = 0.0;
}

// Shared-memory-staged variant (default whenever a row fits): X is read from
// HBM exactly once.
//   1. the CTA stages its R rows into shared memory with one bulk copy per
//      row (any l / ldx alignment: the 16-byte-aligned interior by TMA, an
//      unaligned first / last element by plain loads);
//   2. 8 threads per row run the reference's lane chains (sum + constancy,
//      then ssd) out of shared memory and finish with the shuffle tree;
//   3. all threads write u = (x - mean) / scale (or the zero row) back with
//      coalesced stores, plus the zero K padding up to ldu.
// Small CTAs (64 threads, R <= 8 rows) so several CTAs share an SM and one
// CTA's chains overlap the others' copies.  Same arithmetic as
// normalize_rows_kernel, bit for bit.
constexpr int kNormSmemMaxRows = 8;  // rows per CTA (one 8-lane group each; 64 or 128 threads)


#ifdef PCC_K1_PHASES
// tools/k1_phases.cu: per-phase clock totals of normalize_rows_smem_kernel
__device__ unsigned long long g_k1_phase[8];
#define K1_MARK(i)                                                              \
  do {                                                                          \
    if (threadIdx.x == 0) {                                                     \
      const long long now_ = clock64();                                         \
      atomicAdd(&g_k1_phase[i], (unsigned long long)(now_ - k1_t_));            \
      k1_t_ = now_;                                                             \
    }                                                                           \
  } while (0)
#else
#define K1_MARK(i) \
  do {             \
  } while (0)
#endif

// Extra destinations of the broadcast variant: each U row (and flag) is
// stored to every listed buffer -- peer GPUs' U over NVLink (CUDA IPC
// mappings) in the multi-GPU exchange, so normalisation and the all-gather
// of U are one kernel.
constexpr int kMaxNormDests = 16;
struct NormDests {
  double *u[kMaxNormDests];
  uint8_t *flags[kMaxNormDests];
  int n;
  // kNormDigits mode (split mode, csrc/split.cuh): the normalised rows go
  // straight into int8 radix-128 digit planes [KB][7][rows_total][64] and
  // a power-of-two scale per row -- U itself is never written
  int8_t *slices;
  double *scale;
  int64_t rows_total;
};
constexpr int kNormLocal = 0, kNormBcast = 1, kNormDigits = 2;

__device__ __forceinline__ void bulk_copy_row(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int kNormSmemThreads, int MODE = kNormLocal>
__global__ void __launch_bounds__(kNormSmemThreads)
normalize_rows_smem_kernel(const double *__restrict__ x, int64_t ldx, double *__restrict__ u, int64_t ldu,
                           uint8_t *__restrict__ zero_variance, int64_t l, int64_t row_lo, int64_t row_hi,
                           int rows_per_cta, int64_t lds, NormDests dests) {
  extern __shared__ __align__(16) double srow[];  // [rows_per_cta][lds]
  __shared__ double s_mean[kNormSmemMaxRows], s_scale[kNormSmemMaxRows];
  __shared__ int s_zero[kNormSmemMaxRows];
  __shared__ int64_t s_base[kNormSmemMaxRows];  // row r's element 0 is srow[s_base[r]]
  const int tid = threadIdx.x;
  const int64_t r0 = row_lo + (int64_t)blockIdx.x * rows_per_cta;
  const int rows = (int)((row_hi - r0) < (int64_t)rows_per_cta ? (row_hi - r0) : (int64_t)rows_per_cta);
  const uint32_t sbase = smem_u32(srow);
#ifdef PCC_K1_PHASES
  long long k1_t_ = clock64();
#endif

  // 1. stage the rows: per row one 1-D bulk copy (cp.async.bulk, byte-counted
  //    mbarrier) of its 16-byte-aligned interior, issued by its own thread
  //    (bulk copies issued by one thread complete one after another,
  //    tools/bulk_bw.cu), plus plain loads of an unaligned first and last
  //    element -- any l and ldx, and nothing outside the rows is read.  The
  //    smem row starts 8 bytes into its slot when the row's first element is
  //    misaligned, so the interior lands 16-byte aligned (slot stride lds).
  __shared__ __align__(8) uint64_t s_bar;
  const uint32_t bar = smem_u32(&s_bar);
  if (tid == 0) {
    mbar_init(bar, (uint32_t)rows);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid < rows) {
    const double *xr = x + (r0 + tid) * ldx;
    const int pre = (int)((reinterpret_cast<uintptr_t>(xr) >> 3) & 1);  // first element misaligned
    const int64_t base = (int64_t)tid * lds + pre;
    s_base[tid] = base;
    const int64_t body = (l - pre) & ~(int64_t)1;  // aligned interior [pre, pre + body)
    if (pre) srow[base] = xr[0];
    if (pre + body < l) srow[base + l - 1] = xr[l - 1];
    if (body > 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)(body * sizeof(double)));
      bulk_copy_row(sbase + (uint32_t)((base + pre) * sizeof(double)), xr + pre, (uint32_t)(body * sizeof(double)),
                    bar);
    } else {
      mbar_arrive(bar);
    }
  }
  if (tid == 0) mbar_wait(bar, 0);
  __syncthreads();
  K1_MARK(0);

  // 2. the 8 lanes of each row run the reference's chains back to back out
  //    of shared memory: sum8, the mean, then ssd8 with the centring d = x -
  //    mean inline (the subtract and square are off the dependent add chain).
  //    The reference's exact constancy test (every x == x[0],
  //    _kernels.py:209-223) is row min == row max, and the row's min and max
  //    -- order-free -- are taken by the warps that run no lane chains while
  //    the chains run (after them, by every thread, when every warp runs
  //    chains).  Digit planes need them too: max |x - mean| = max(RN(xmax -
  //    mean), RN(mean - xmin)) (RN is monotone and odd).
  constexpr int kWarps = kNormSmemThreads / 32;
  __shared__ double s_min[kWarps][kNormSmemMaxRows], s_max[kWarps][kNormSmemMaxRows];
  const int chain_warps = (rows * 8 + 31) / 32;
  const int nfw = kWarps - chain_warps;
  auto row_minmax = [&](int w, int nw) {  // this warp is w of nw warps sharing the rows
    for (int r = 0; r < rows; ++r) {
      const double *ds = srow + s_base[r];
      double lo = ds[0], hi = ds[0];
      for (int64_t k = w * 32 + (tid & 31); k < l; k += nw * 32) {
        lo = fmin(lo, ds[k]);
        hi = fmax(hi, ds[k]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if ((tid & 31) == 0) {
        s_min[tid >> 5][r] = lo;
        s_max[tid >> 5][r] = hi;
      }
    }
  };
  // U modes: the constancy test rides on the sum chain (x != x[0]); digit
  // planes: it is row min == row max, the min / max the digits need anyway,
  // taken by the warps that run no chains while the chains run
  constexpr bool kMinMax = MODE == kNormDigits;
  if (kMinMax && (tid >> 5) >= chain_warps) row_minmax((tid >> 5) - chain_warps, nfw);
  const int lane8 = tid & 7;
  const int row = tid >> 3;
  const bool active = row < rows;
  if ((tid >> 5) < chain_warps) {
    const double *sr = srow + s_base[active ? row : 0];
    const int nsteps = (int)((l - lane8 + 7) >> 3);
    bool varies = false;
    double s = active ? row_chain<false, !kMinMax>(sr + lane8, nsteps, sr[0], varies) : 0.0;
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    const unsigned vb = __ballot_sync(0xffffffffu, varies);
    const bool constant = !kMinMax && (vb & (0xffu << (tid & 24))) == 0u;  // uniform within the 8-lane group
    const double mean = constant ? 0.0 : __ddiv_rn(s, (double)l);
    double q = (active && !constant) ? row_chain<true>(sr + lane8, nsteps, mean, varies) : 0.0;
    q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 1));
    q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 2));
    q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 4));
    if (active && lane8 == 0) {
      s_mean[row] = mean;
      s_scale[row] = q;  // ssd for now (digit planes: the zero rule needs the min / max)
      s_zero[row] = constant || q == 0.0;
      if (!kMinMax) {
        const bool zero = constant || q == 0.0;
        s_scale[row] = zero ? 0.0 : __dsqrt_rn(q);
        if (MODE == kNormBcast) {
          for (int d = 0; d < dests.n; ++d) dests.flags[d][r0 + row] = zero ? 1 : 0;
        } else {
          zero_variance[r0 + row] = zero ? 1 : 0;
        }
      }
    }
  }
  __syncthreads();
  if (kMinMax) {
    if (nfw == 0) {  // every warp ran chains: min / max now, by all threads
      row_minmax(tid >> 5, kWarps);
      __syncthreads();
    }
    const int w0 = nfw == 0 ? 0 : chain_warps;
    if (tid < rows) {
      const int r = tid;
      double lo = s_min[w0][r], hi = s_max[w0][r];
      for (int w = w0 + 1; w < kWarps; ++w) {
        lo = fmin(lo, s_min[w][r]);
        hi = fmax(hi, s_max[w][r]);
      }
      s_min[0][r] = lo;  // the row's min / max (digit planes)
      s_max[0][r] = hi;
      const double q = s_scale[r];
      const bool zero = lo == hi || q == 0.0;  // constant (x == x[0] everywhere), or zero ssd
      s_zero[r] = zero;
      s_scale[r] = zero ? 0.0 : __dsqrt_rn(q);
      zero_variance[r0 + r] = zero ? 1 : 0;
    }
    __syncthreads();
  }
  K1_MARK(1);

  if (MODE == kNormDigits) {
    // 3'. digit planes instead of U: per row the exact max |u| = RN(max |x -
    //     mean| / scale) (division is monotone), its power-of-two scale, then
    //     each thread turns 4 consecutive u values -- the same IEEE
    //     operations as below, so the same bits as K1 + pcc_split_rows_f64 --
    //     into 7 radix-128 digits, one 32-bit store per digit plane
    constexpr int W = 64;  // SplitCfg::kRowBytes
    const int64_t kpad = (l + W - 1) / W * W;
    const int64_t plane = dests.rows_total * W;
    for (int r = 0; r < rows; ++r) {
      const double *ds = srow + s_base[r];
      const bool zero = s_zero[r] != 0;
      const double m0 = s_mean[r], sc = s_scale[r];
      const double lo = s_min[0][r], hi = s_max[0][r];
      const double dm = fmax(__dsub_rn(hi, m0), __dsub_rn(m0, lo));  // = max_k |RN(x_k - mean)|
      const double m = zero ? 0.0 : __ddiv_rn(dm, sc);
      int e = 0;
      if (m > 0.0) {
        frexp(m, &e);
        if (ldexp(m, 7 - e) >= 127.5) ++e;  // keep the leading digit within [-127, 127]
      }
      if (tid == 0) dests.scale[r0 + r] = m > 0.0 ? ldexp(1.0, e - 7) : 0.0;
      const double pw = m > 0.0 ? ldexp(1.0, 7 - e) : 0.0;  // 7 - e <= 14 for unit-norm rows
      const RowDiv dv = row_div(sc);
      auto emit = [&](bool exact) {
        bool bad = false;
        auto dq = [&](double a) { return exact ? __ddiv_rn(a, dv.b) : div_fast(a, dv, bad); };
        for (int64_t k = 4 * (int64_t)tid; k < kpad; k += 4 * kNormSmemThreads) {
          uint32_t packed[7] = {};
          if (m > 0.0) {
            double v4[4];
            if (k + 3 < l && (s_base[r] & 1) == 0) {  // 16-byte aligned: two LDS.128
              const double2 a = *reinterpret_cast<const double2 *>(ds + k);
              const double2 b = *reinterpret_cast<const double2 *>(ds + k + 2);
              v4[0] = a.x, v4[1] = a.y, v4[2] = b.x, v4[3] = b.y;
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) v4[j] = (k + j < l) ? ds[k + j] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) split_digits7((k + j < l) ? dq(__dsub_rn(v4[j], m0)) * pw : 0.0, j, packed);
          }
          int8_t *dst = dests.slices + (k / W) * 7 * plane + (r0 + r) * W + (k % W);
#pragma unroll
          for (int i = 0; i < 7; ++i) *reinterpret_cast<uint32_t *>(dst + i * plane) = packed[i];
        }
        return bad;
      };
      if (__syncthreads_or(emit(!dv.fast) ? 1 : 0)) emit(true);
    }
    return;
  }

  // 3. write U rows (coalesced): u = (x - mean) / scale, zero rows for zero
  //    variance, zero K padding
  for (int r = 0; r < rows; ++r) {
    const int64_t off = (r0 + r) * ldu;
    auto put = [&](int64_t k, double v) {  // one store, or one per destination
      if (MODE == kNormBcast) {
        for (int d = 0; d < dests.n; ++d) dests.u[d][off + k] = v;
      } else {
        u[off + k] = v;
      }
    };
    const double *ds = srow + s_base[r];
    if (s_zero[r]) {
      for (int64_t k = tid; k < ldu; k += kNormSmemThreads) put(k, 0.0);
    } else {
      const double m = s_mean[r];
      const RowDiv dv = row_div(s_scale[r]);
      // u = (x - mean) / scale; four independent divisions per iteration keep
      // more of their latency in flight; the IEEE fallback (div_fast) rewrites
      // the row in the rare case that any element needs it
      constexpr int64_t T = kNormSmemThreads;
      auto emit = [&](bool exact) {
        bool bad = false;
        auto dq = [&](double a) { return exact ? __ddiv_rn(a, dv.b) : div_fast(a, dv, bad); };
        int64_t k = tid;
        for (; k + 3 * T < l; k += 4 * T) {
          const double q0 = dq(__dsub_rn(ds[k], m)), q1 = dq(__dsub_rn(ds[k + T], m));
          const double q2 = dq(__dsub_rn(ds[k + 2 * T], m)), q3 = dq(__dsub_rn(ds[k + 3 * T], m));
          put(k, q0);
          put(k + T, q1);
          put(k + 2 * T, q2);
          put(k + 3 * T, q3);
        }
        for (; k < l; k += T) put(k, dq(__dsub_rn(ds[k], m)));
        return bad;
      };
      if (__syncthreads_or(emit(!dv.fast) ? 1 : 0)) emit(true);
      for (int64_t k = l + tid; k < ldu; k += kNormSmemThreads) put(k, 0.0);
    }
  }
  K1_MARK(2);
}

// Chunked K1 for long rows (host dispatch: rows 16-byte aligned, l even,
// l >= kChunkMinL).  One row per 64-thread CTA, never resident: the row
// streams through two shared-memory chunk buffers three times -- sum pass,
// ssd pass, output pass -- one bulk copy per chunk, the next chunk landing
// while the current one is consumed.  The staged kernel holds a whole row for
// its ~2 l/8 dependent adds, so at l = 8192 only 3 rows fit an SM; here a row
// occupies 2 chunks, and the rows in flight per SM are set by the host to
// what L2 can hold between the passes (the second and third reads of a row
// are L2 hits: DRAM traffic stays one read of X plus one write).  Lanes 0..7
// of warp 0 ARE the reference's lanes (same chains, same tree, same IEEE
// operations as normalize_rows_smem_kernel); warp 1 takes the row's min / max
// in the digit-plane mode; both warps write the output.
constexpr int kChunkThreads = 64;
#ifdef PCC_K1C_PROBE
// tools/k1c_probe.cu: clock64 totals (thread 0 of each CTA) -- [0..2] time in
// passes 0 / 1 / 2 (sum, ssd, output), [3] time waiting for chunks
__device__ unsigned long long g_k1c_probe[8];
#endif
template <int MODE>
__global__ void __launch_bounds__(kChunkThreads)
normalize_rows_chunked_kernel(const double *__restrict__ x, int64_t ldx, double *__restrict__ u, int64_t ldu,
                              uint8_t *__restrict__ zero_variance, int64_t l, int64_t row_lo, int ch,
                              NormDests dests) {
  extern __shared__ __align__(16) double cbuf[];  // [2][ch]
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ double s_mean, s_scale, s_pw, s_lo, s_hi;
  __shared__ int s_zero;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t row = row_lo + blockIdx.x;
  const double *xr = x + row * ldx;
  const int nc = (int)((l + ch - 1) / ch);
  const int items = 3 * nc;  // (pass, chunk): sum, ssd, output
  if (tid == 0) {
    mbar_init(smem_u32(&s_bar[0]), 1);
    mbar_init(smem_u32(&s_bar[1]), 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int it) {  // chunk it % nc into buffer it & 1
    const int64_t k0 = (int64_t)(it % nc) * ch;
    const uint32_t bytes = (uint32_t)((l - k0 < ch ? l - k0 : ch) * sizeof(double));
    const uint32_t bar = smem_u32(&s_bar[it & 1]);
    mbar_arrive_expect_tx(bar, bytes);
    bulk_copy_row(smem_u32(cbuf + (it & 1) * ch), xr + k0, bytes, bar);
  };
  // buffer b's chunks are issued by thread 32 b: a thread's bulk copies
  // complete one after another (tools/tma_issue_bw.cu), so the two buffers'
  // copies come from different threads
  if (tid == 0) issue(0);
  constexpr bool kMinMax = MODE == kNormDigits;  // constancy = (min == max) there
  double s = 0.0, q = 0.0, ref = 0.0, mean = 0.0, lo = 0.0, hi = 0.0;
  bool varies = false;
  constexpr int W = 64;  // digit-plane K block = SplitCfg::kRowBytes
  const int64_t kend = MODE == kNormDigits ? (l + W - 1) / W * W : ldu;  // outputs incl. padding
  for (int it = 0; it < items; ++it) {
#ifdef PCC_K1C_PROBE
    const long long t_item = clock64();
#endif
    if (tid == 32 * ((it + 1) & 1) && it + 1 < items) issue(it + 1);  // its buffer was released by item it - 1
    mbar_wait(smem_u32(&s_bar[it & 1]), (uint32_t)((it >> 1) & 1));
#ifdef PCC_K1C_PROBE
    if (tid == 0) atomicAdd(&g_k1c_probe[3], (unsigned long long)(clock64() - t_item));
#endif
    const int pass = it / nc, c = it % nc;
    const int64_t k0 = (int64_t)c * ch;
    const int cnt = (int)(l - k0 < ch ? l - k0 : ch);
    const double *p = cbuf + (it & 1) * ch;
    if (pass < 2 && tid < 8) {
      // the reference's lane tid over this chunk (chunks are multiples of 8)
      const int nsteps = (cnt - tid + 7) >> 3;
      if (pass == 0) {
        if (c == 0) ref = p[0];
#if defined(PCC_K1C_EXP) && (PCC_K1C_EXP & 2)  // probe experiment: no constancy compare on the chain
        row_chain_more<false, false>(s, p + tid, nsteps, ref, varies);
#else
        row_chain_more<false, !kMinMax>(s, p + tid, nsteps, ref, varies);
#endif
      } else {
        row_chain_more<true>(q, p + tid, nsteps, mean, varies);
      }
      if (c == nc - 1) {
        if (pass == 0) {  // tree ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), mean
          s = __dadd_rn(s, __shfl_xor_sync(0xffu, s, 1));
          s = __dadd_rn(s, __shfl_xor_sync(0xffu, s, 2));
          s = __dadd_rn(s, __shfl_xor_sync(0xffu, s, 4));
          const bool constant = !kMinMax && __ballot_sync(0xffu, varies) == 0u;
          mean = __ddiv_rn(s, (double)l);
          if (tid == 0) s_zero = constant ? 1 : 0;
        } else {
          q = __dadd_rn(q, __shfl_xor_sync(0xffu, q, 1));
          q = __dadd_rn(q, __shfl_xor_sync(0xffu, q, 2));
          q = __dadd_rn(q, __shfl_xor_sync(0xffu, q, 4));
          if (tid == 0) {
            const bool zero = (kMinMax ? s_lo == s_hi : s_zero != 0) || q == 0.0;
            const double sc = zero ? 0.0 : __dsqrt_rn(q);
            s_zero = zero ? 1 : 0;
            s_mean = mean;
            s_scale = sc;
            if (MODE == kNormBcast) {
              for (int d = 0; d < dests.n; ++d) dests.flags[d][row] = zero ? 1 : 0;
            } else {
              zero_variance[row] = zero ? 1 : 0;
            }
            if (MODE == kNormDigits) {
              // exact max |u| = RN(max |x - mean| / scale) (RN is monotone and odd)
              const double dm = fmax(__dsub_rn(s_hi, mean), __dsub_rn(mean, s_lo));
              const double m = zero ? 0.0 : __ddiv_rn(dm, sc);
              int e = 0;
              if (m > 0.0) {
                frexp(m, &e);
                if (ldexp(m, 7 - e) >= 127.5) ++e;  // keep the leading digit within [-127, 127]
              }
              dests.scale[row] = m > 0.0 ? ldexp(1.0, e - 7) : 0.0;
              s_pw = m > 0.0 ? ldexp(1.0, 7 - e) : 0.0;
            }
          }
        }
      }
    } else if (pass == 0 && kMinMax && tid >= 32) {
      // warp 1: the row's min / max (order-free), for the digits and the
      // constancy test min == max
      if (c == 0) lo = hi = p[0];
      for (int k = lane; k < cnt; k += 32) {
        lo = fmin(lo, p[k]);
        hi = fmax(hi, p[k]);
      }
      if (c == nc - 1) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
          s_lo = lo;
          s_hi = hi;
        }
      }
    } else if (pass == 2
#if defined(PCC_K1C_EXP) && (PCC_K1C_EXP & 1)  // probe experiment: no output pass work
               && false
#endif
    ) {
      // output of this chunk (+ the K padding after the last one)
      const bool zero = s_zero != 0;
      const double m0 = s_mean;
      const RowDiv dv = row_div(zero ? 1.0 : s_scale);
      const int64_t kb = k0 + (c == nc - 1 ? (kend - k0) : ch);  // this chunk's outputs: [k0, kb)
      if (MODE == kNormDigits) {
        const double pw = s_pw;
        const int64_t plane = dests.rows_total * W;
        auto emit = [&](bool exact) {
          bool bad = false;
          auto dq = [&](double a) { return exact ? __ddiv_rn(a, dv.b) : div_fast(a, dv, bad); };
          for (int64_t k = k0 + 4 * tid; k < kb; k += 4 * kChunkThreads) {
            uint32_t packed[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
            if (pw > 0.0) {
              double v4[4];
              if (k + 3 < l) {
                const double2 a = *reinterpret_cast<const double2 *>(p + (k - k0));
                const double2 b = *reinterpret_cast<const double2 *>(p + (k - k0) + 2);
                v4[0] = a.x, v4[1] = a.y, v4[2] = b.x, v4[3] = b.y;
              } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) v4[j] = (k + j < l) ? p[k - k0 + j] : 0.0;
              }
#pragma unroll
              for (int j = 0; j < 4; ++j)
                split_digits7((k + j < l) ? __dmul_rn(dq(__dsub_rn(v4[j], m0)), pw) : 0.0, j, packed);
            }
            int8_t *dst = dests.slices + (k / W) * 7 * plane + row * W + (k % W);
#pragma unroll
            for (int i = 0; i < 7; ++i) *reinterpret_cast<uint32_t *>(dst + i * plane) = packed[i];
          }
          return bad;
        };
        if (__syncthreads_or(emit(!dv.fast) ? 1 : 0)) emit(true);
      } else {
        const int64_t off = row * ldu;
        auto put = [&](int64_t k, double2 v) {
          if (MODE == kNormBcast) {
            for (int d = 0; d < dests.n; ++d) *reinterpret_cast<double2 *>(dests.u[d] + off + k) = v;
          } else {
            __stcs(reinterpret_cast<double2 *>(u + off + k), v);
          }
        };
        auto emit = [&](bool exact) {
          bool bad = false;
          auto dq = [&](double a) { return exact ? __ddiv_rn(a, dv.b) : div_fast(a, dv, bad); };
          int64_t k = k0 + 2 * tid;
          if (!zero) {
            // four independent pairs per thread in flight (the quotients are
            // latency chains of 4 FP64 operations)
            constexpr int S = 2 * kChunkThreads;
            const int64_t kl = kb < l ? kb : l;
            for (; k + 3 * S < kl; k += 4 * S) {
              double2 xv[4], v[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const double2 *>(p + (k + i * S - k0));
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                v[i].x = dq(__dsub_rn(xv[i].x, m0));
                v[i].y = dq(__dsub_rn(xv[i].y, m0));
              }
#pragma unroll
              for (int i = 0; i < 4; ++i) put(k + i * S, v[i]);
            }
          }
          for (; k < kb; k += 2 * kChunkThreads) {  // l, ldu even: pairs never straddle
            double2 v = make_double2(0.0, 0.0);
            if (!zero && k < l) {
              const double2 xv = *reinterpret_cast<const double2 *>(p + (k - k0));
              v.x = dq(__dsub_rn(xv.x, m0));
              v.y = dq(__dsub_rn(xv.y, m0));
            }
            put(k, v);
          }
          return bad;
        };
        if (__syncthreads_or(emit(!dv.fast) ? 1 : 0)) emit(true);
      }
    }
    __syncthreads();  // the buffer is free for item it + 2; s_* written above are visible
#ifdef PCC_K1C_PROBE
    if (tid == 0) atomicAdd(&g_k1c_probe[pass], (unsigned long long)(clock64() - t_item));
#endif
  }
}

}  // namespace pcc
