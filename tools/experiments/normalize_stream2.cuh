// EXPERIMENT (not built into the product library): the round-2 streamed K1,
// second design -- chain warps fed by dedicated TMA producer warps, output
// warps re-reading rows from L2 through their own TMA rings.  Bit-exact on
// c2/c4/c5 but slower than the staged kernel (c2 373 vs 237 us, c4 1333 vs
// 1255 us): at c4 the L2 re-reads miss (ncu: DRAM read 4.9 GB = 2.3x X, L2
// hit rate 28 %), and a thread's TMA copies complete one after another
// (tools/tma_issue_bw.cu), so the windows need many issuing lanes.  Record in
// profiles/r02_k1_experiments.md; probe: tools/k1s2_probe.cu.
//
// normalize_stream.cuh -- K1 for long rows: per-variable z-normalisation
// streamed through shared-memory windows, bit-exact to the reference's
// _kernels.normalize_rows (_kernels.py:226-252; same arithmetic contract as
// normalize.cuh: sum8 / ssd8 lane chains, exact constancy test, IEEE mean /
// sqrt / division).
//
// Why.  A row's statistics are 8 strictly sequential lane chains (sum8, then
// ssd8 with the mean: 2 * l/8 dependent FP64 adds), so a row is "in flight"
// for ~2 l/8 add latencies however many threads it gets.  The staged kernel
// (normalize.cuh) holds whole rows in shared memory for that time, which caps
// the rows in flight at 224 KB / row bytes (3 at l = 8192) and leaves HBM half
// idle.  Here a row is never resident: its windows stream through shared
// memory three times (sum pass, ssd pass, output pass), so only the windows
// in flight occupy shared memory.
//
// CTA = 8 warps, one per SM (persistent).  Warps sit on the four SM
// sub-partitions (SMSP = warp % 4) by role:
//   * chain warps (warps 0, 1: SMSPs 0 and 1) -- each owns 4 rows at a time
//     (8 lanes per row: lane j IS reference lane j).  Lanes 8q, 8q+1 issue
//     row q's windows (1-D bulk copies into the warp's ring: bulk copies
//     issued by one thread complete one after another, tools/bulk_bw.cu, so
//     eight issuing lanes).  Per full window the lane chain is straight-line
//     code with its shared-memory loads two batches ahead, so the dependent
//     adds run at FP64-add latency; the constancy test is not on the chain
//     (below).  Sum pass, then ssd pass; then row q's (mean, scale, digit
//     power, ssd == 0) go to a handoff slot.
//   * output warps (warps 2, 3, 6, 7 [, 4, 5]) -- one row job at a time: the
//     row's windows are re-read from L2 by bulk copies into the warp's own
//     ring, u = (x - mean) / scale (or the broadcast, or the split-mode digit
//     planes) is written with 16-byte stores, and the reference's exact
//     constancy test (every x == x[0], _kernels.py:209-223) runs on the same
//     values: a constant row whose rounded ssd is not 0 (rare) is rewritten
//     with zeros afterwards, and the zero-variance flag is written here.
// The first read of a row comes from HBM; the ssd and output passes follow
// within ~2 chain passes and hit L2: DRAM traffic stays one read of X plus one
// write of U (or of the digit planes).
//
// Requires 16-byte aligned rows (x and ldx) and even l: bulk copies move
// 16-byte multiples.  Other shapes use normalize_rows_smem_kernel (host
// dispatch in pcc_b200.cu).
#pragma once

#include "../../paper_1605_01584_b200/csrc/normalize.cuh"

namespace pcc {

#ifdef PCC_K1S_PROBE
// tools/k1s2_probe.cu: clock64 totals per role -- [0] chain total, [1] chain
// window waits, [2] chain handoff waits, [3] output total, [4] output handoff
// waits, [5] output window waits
__device__ unsigned long long g_k1s_probe[8];
#define K1S_T(v) const long long v = clock64()
#define K1S_ADD(i, t)                                                                               \
  do {                                                                                              \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_k1s_probe[i], (unsigned long long)(clock64() - (t))); \
  } while (0)
#ifndef PCC_K1S_EXP
#define PCC_K1S_EXP 0  // experiment bits: 1 output skips compute, 4 output copies nothing,
                       // 8 chains skip copies and waits, 16 chains skip the adds
#endif
#else
#define PCC_K1S_EXP 0
#define K1S_T(v) \
  do {           \
  } while (0)
#define K1S_ADD(i, t) \
  do {                \
  } while (0)
#endif

struct K1Stream {
  static constexpr int kWarps = 8;
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int kRows = 4;              // rows per chain group (8 lanes each)
  static constexpr int kWin = 512;             // doubles per row and chain window
  static constexpr int kCStages = 4;           // chain ring depth
  static constexpr int kBox = 256;             // doubles per TMA box (one row piece; box dims <= 256)
  static constexpr int kOWin = 512;            // doubles per output window
  static constexpr int kOStages = 3;           // output ring depth
  static constexpr int kHand = 2;              // handoff slots per chain warp
  static constexpr int kChainWarps = 2, kOutWarps = 4;
  // chain stage layout: [kWin / kBox pieces][kRows][kBox] -- one TMA box
  // {kBox, kRows} per piece (TMA destinations are 128-byte aligned)
  static constexpr int kCStageDoubles = kRows * kWin;
  __host__ __device__ static constexpr int chain_ring_doubles(int cw) { return cw * kCStages * kCStageDoubles; }
  __host__ __device__ static constexpr int out_ring_doubles(int ow) { return ow * kOStages * kOWin; }
  __host__ __device__ static constexpr int bar_count(int cw, int ow) {
    return 2 * cw * kCStages + ow * kOStages + 2 * cw * kHand;
  }
  // rings, then barriers, then the handoff values (4 doubles per row)
  __host__ __device__ static constexpr int smem_bytes(int cw, int ow) {
    return 128 + 8 * (chain_ring_doubles(cw) + out_ring_doubles(ow)) + 8 * bar_count(cw, ow) +
           8 * (cw * kHand * 4 * kRows);
  }
};

// Warp roles (CTA of 8 warps, SMSP = warp % 4): chain warps 0, 1 (SMSPs 0,
// 1), their TMA producers 4, 5 (same SMSPs: they only issue copies and wait),
// output warps 2, 3, 6, 7 (SMSPs 2, 3).
__host__ __device__ constexpr int k1s_chain_index(int w) { return w < 2 ? w : -1; }
__host__ __device__ constexpr int k1s_producer_index(int w) { return (w == 4 || w == 5) ? w - 4 : -1; }
__host__ __device__ constexpr int k1s_out_index(int w) { return (w & 3) >= 2 ? (w >> 2) * 2 + (w & 3) - 2 : -1; }

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// 2-D TMA tile load (box {kBox doubles, 1 row} of X) with an L2 eviction
// policy.  Tensor copies, unlike 1-D bulk copies, do not complete one after
// another per issuing thread (tools/k1s2_probe.cu: 1-D bulk copies made every
// window cost ~1,000 cycles of issue stall), so one lane issues a window.
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap *map, int32_t c0, int32_t c1,
                                                 uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}

// Offset of lane-chain step t (element 8 t of the row's window) from the
// lane's first element in a chain stage ([pieces][kRows][kBox] layout).
__host__ __device__ constexpr int k1s_step_off(int t) {
  return (8 * t / K1Stream::kBox) * (K1Stream::kRows * K1Stream::kBox) + (8 * t) % K1Stream::kBox;
}

// One lane chain over a FULL window (kWin / 8 steps, stride 8): straight-line
// code, loads two 8-step batches ahead of the adds.
//   SSD = false: s += x (sum8 lane);
//   SSD = true:  d = x - ref (the mean), s += RN(d * d) (ssd8 lane), and with
//                DMAX the max |d| of the window (a tree per batch, off the
//                chain; max is exact).
template <bool SSD, bool DMAX>
__device__ __forceinline__ void k1s_chain_full(double &s, const double *p, double ref, double &dmax) {
  constexpr int NB = K1Stream::kWin / 64;  // 8-step batches per window
  double v[3][8];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[b][i] = p[k1s_step_off(8 * b + i)];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b + 2 < NB) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[(b + 2) % 3][i] = p[k1s_step_off(8 * (b + 2) + i)];
    }
    double *cur = v[b % 3];
    if (SSD) {
      double d[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = __dsub_rn(cur[i], ref);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __dadd_rn(s, __dmul_rn(d[i], d[i]));
      if (DMAX) {
        const double m01 = fmax(fabs(d[0]), fabs(d[1])), m23 = fmax(fabs(d[2]), fabs(d[3]));
        const double m45 = fmax(fabs(d[4]), fabs(d[5])), m67 = fmax(fabs(d[6]), fabs(d[7]));
        dmax = fmax(dmax, fmax(fmax(m01, m23), fmax(m45, m67)));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __dadd_rn(s, cur[i]);
    }
  }
}

// The same chain over a partial window (the last window of a row whose l is
// not a multiple of kWin): nsteps elements at stride 8.
template <bool SSD, bool DMAX>
__device__ __forceinline__ void k1s_chain_part(double &s, const double *p, int nsteps, double ref, double &dmax) {
  for (int t = 0; t < nsteps; ++t) {
    const double v = p[k1s_step_off(t)];
    if (SSD) {
      const double d = __dsub_rn(v, ref);
      s = __dadd_rn(s, __dmul_rn(d, d));
      if (DMAX) dmax = fmax(dmax, fabs(d));
    } else {
      s = __dadd_rn(s, v);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(K1Stream::kThreads, 1)
normalize_rows_stream_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap4,
                             double *__restrict__ u, int64_t ldu, uint8_t *__restrict__ zero_variance, int64_t l,
                             int64_t row_lo, int64_t row_hi, NormDests dests) {
  using C = K1Stream;
  constexpr int CW = C::kChainWarps, OW = C::kOutWarps;
  extern __shared__ __align__(128) double k1s_smem_raw[];
  // TMA tensor destinations must be 128-byte aligned
  double *k1s_smem = k1s_smem_raw + ((128u - (smem_u32(k1s_smem_raw) & 127u)) & 127u) / 8;
  double *cring = k1s_smem;                              // [CW][kCStages][pieces][kRows][kBox]
  double *oring = k1s_smem + C::chain_ring_doubles(CW);  // [OW][kOStages][kOWin]
  const uint32_t bars = smem_u32(oring + C::out_ring_doubles(OW));
  auto cfull = [&](int c, int s) { return bars + 8u * (c * C::kCStages + s); };
  auto cempty = [&](int c, int s) { return bars + 8u * (CW * C::kCStages + c * C::kCStages + s); };
  auto ofull = [&](int o, int s) { return bars + 8u * (2 * CW * C::kCStages + o * C::kOStages + s); };
  auto hfull = [&](int c, int h) {
    return bars + 8u * (2 * CW * C::kCStages + OW * C::kOStages + c * C::kHand + h);
  };
  auto hempty = [&](int c, int h) {
    return bars + 8u * (2 * CW * C::kCStages + OW * C::kOStages + CW * C::kHand + c * C::kHand + h);
  };
  double *hand = oring + C::out_ring_doubles(OW) + C::bar_count(CW, OW);  // [CW][kHand][4][kRows]
  auto hslot = [&](int c, int h) { return hand + (c * C::kHand + h) * 4 * C::kRows; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwin = (l + C::kWin - 1) / C::kWin;
  const int nwi = (int)nwin;
  const int64_t groups = (row_hi - row_lo + C::kRows - 1) / C::kRows;
  const int64_t gstep = (int64_t)gridDim.x * CW;

  if (threadIdx.x == 0) {
    for (int c = 0; c < CW; ++c) {
      for (int s = 0; s < C::kCStages; ++s) {
        mbar_init(cfull(c, s), 1);
        mbar_init(cempty(c, s), 1);
      }
      for (int h = 0; h < C::kHand; ++h) {
        mbar_init(hfull(c, h), 1);
        mbar_init(hempty(c, h), C::kRows);  // one arrival per row job
      }
    }
    for (int o = 0; o < OW; ++o)
      for (int s = 0; s < C::kOStages; ++s) mbar_init(ofull(o, s), C::kOWin / C::kBox);
    mbar_fence_init();
    tma_prefetch_desc(&xmap);
    tma_prefetch_desc(&xmap4);
  }
  __syncthreads();

  const int pidx = k1s_producer_index(warp);
  if (pidx >= 0) {
    // -------------------------------------------------- chain-ring producer
    // The job stream of chain warp c -- (group, pass, window) in order -- one
    // TMA box {kBox, kRows} per window piece (rows past row_hi and samples
    // past l read as zeros: the map ends there), into ring slot job % kCStages
    // once the chain warp has released it.
    const int c = pidx;
    const int64_t g0 = (int64_t)blockIdx.x * CW + c;
    const int64_t my_groups = g0 < groups ? (groups - g0 + gstep - 1) / gstep : 0;
    const uint32_t ring_s = smem_u32(cring + c * C::kCStages * C::kCStageDoubles);
    // Lane p issues the jobs of slot p (a thread's TMA copies complete one
    // after another, tools/tma_issue_bw.cu: ~box bytes / 800 cycles per lane
    // from HBM, so one lane per slot keeps kCStages windows in flight).
    if (lane < C::kCStages && !(PCC_K1S_EXP & 8)) {
      const uint64_t pol = l2_evict_last_policy();  // X is read twice more (ssd, output)
      const int64_t total = my_groups * 2 * nwin;
      for (int64_t job = lane, use = 0; job < total; job += C::kCStages, ++use) {
        if (use > 0) mbar_wait(cempty(c, lane), (uint32_t)((use - 1) & 1));
        const int64_t gi = job / (2 * nwin), w = job % nwin;
        const int32_t r0 = (int32_t)(row_lo + (g0 + gi * gstep) * C::kRows);
        const int64_t k0 = w * C::kWin;
        const int pieces = (int)(((l - k0 < C::kWin ? l - k0 : C::kWin) + C::kBox - 1) / C::kBox);
        mbar_arrive_expect_tx(cfull(c, lane), (uint32_t)(pieces * C::kRows * C::kBox * 8));
        for (int h = 0; h < pieces; ++h)
          tma_load_2d_hint(ring_s + (uint32_t)((lane * C::kCStageDoubles + h * C::kRows * C::kBox) * 8), &xmap4,
                           (int32_t)(k0 + h * C::kBox), r0, cfull(c, lane), pol);
      }
    }
    return;
  }

  const int cidx = k1s_chain_index(warp);
  if (cidx >= 0) {
    // ------------------------------------------------------------ chain warp
    const int c = cidx, r = lane >> 3, j = lane & 7;
    const int64_t g0 = (int64_t)blockIdx.x * CW + c;
    const int64_t my_groups = g0 < groups ? (groups - g0 + gstep - 1) / gstep : 0;
    double *my_ring = cring + c * C::kCStages * C::kCStageDoubles;
    int slot = 0;
    uint32_t phase = 0;
    K1S_T(t_chain);
    for (int64_t gi = 0; gi < my_groups; ++gi) {
      const int64_t r0 = row_lo + (g0 + gi * gstep) * C::kRows;
      const bool active = r0 + r < row_hi;
      double s = 0.0, mean = 0.0, q = 0.0, dmax = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        for (int w = 0; w < nwi; ++w) {
          if (!(PCC_K1S_EXP & 8)) {
            K1S_T(tw);
            if (lane == 0) mbar_wait(cfull(c, slot), phase);
            __syncwarp();
            K1S_ADD(1, tw);
          }
          const int k0 = w * C::kWin;
          const int cnt = (int)(l - k0 < C::kWin ? l - k0 : C::kWin);
          const double *p = my_ring + slot * C::kCStageDoubles + r * C::kBox + j;
          if (active && !(PCC_K1S_EXP & 16)) {
            if (pass == 0) {
              if (cnt == C::kWin)
                k1s_chain_full<false, false>(s, p, 0.0, dmax);
              else
                k1s_chain_part<false, false>(s, p, (cnt - j + 7) >> 3, 0.0, dmax);
            } else {
              if (cnt == C::kWin)
                k1s_chain_full<true, MODE == kNormDigits>(q, p, mean, dmax);
              else
                k1s_chain_part<true, MODE == kNormDigits>(q, p, (cnt - j + 7) >> 3, mean, dmax);
            }
          }
          if (pass == 0 && w == nwi - 1) {  // sum pass done: tree ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), mean
            s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
            s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
            s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
            mean = __ddiv_rn(s, (double)l);
          }
          __syncwarp();  // every lane is done with the slot: release it to the producer
          if (lane == 0) mbar_arrive(cempty(c, slot));
          if (++slot == C::kCStages) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 1));
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 2));
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 4));
      const bool zero = q == 0.0;  // constancy is decided by the output warps
      const double sc = zero ? 0.0 : __dsqrt_rn(q);
      double pw = 0.0;
      if (MODE == kNormDigits) {
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        const double m = zero ? 0.0 : __ddiv_rn(dmax, sc);  // exact max |u| (division is monotone)
        int e = 0;
        if (m > 0.0) {
          frexp(m, &e);
          if (ldexp(m, 7 - e) >= 127.5) ++e;  // keep the leading digit within [-127, 127]
        }
        pw = m > 0.0 ? ldexp(1.0, 7 - e) : 0.0;
      }
      const int h = (int)(gi % C::kHand);
      if (gi >= C::kHand) {
        K1S_T(th);
        if (lane == 0) mbar_wait(hempty(c, h), (uint32_t)(((gi / C::kHand) - 1) & 1));
        __syncwarp();
        K1S_ADD(2, th);
      }
      if (active && j == 0) {
        double *hs = hslot(c, h);
        hs[r] = mean;
        hs[C::kRows + r] = sc;
        hs[2 * C::kRows + r] = pw;
        hs[3 * C::kRows + r] = zero ? 1.0 : 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(hfull(c, h));  // release: the slot's values are visible
    }
    K1S_ADD(0, t_chain);
    return;
  }

  const int oidx = k1s_out_index(warp);
  if (oidx < 0) return;
  // -------------------------------------------------------------- output warp
  // Row jobs in handoff order: job J = (round i, chain warp c, row r) with
  // J = (i * CW + c) * kRows + r; output warp o takes J = o, o + OW, ...
  const int o = oidx;
  const int64_t first = (int64_t)blockIdx.x * CW;
  const int64_t rounds = first < groups ? (groups - first + gstep - 1) / gstep : 0;
  const int64_t njobs = rounds * CW * C::kRows;
  double *my_ring = oring + o * C::kOStages * C::kOWin;
  const uint32_t my_ring_s = smem_u32(my_ring);
  const uint64_t pol = l2_evict_first_policy();  // last read of X
  constexpr int W = 64;  // digit-plane K block = SplitCfg::kRowBytes (split mode)
  const int64_t kend = MODE == kNormDigits ? (l + W - 1) / W * W : ldu;  // outputs per row incl. padding
  const int64_t otot = (kend + C::kOWin - 1) / C::kOWin;                  // windows of output
  const int64_t plane = dests.rows_total * W;
  int slot = 0;
  uint32_t phase = 0;
  K1S_T(t_out);
  for (int64_t J = o; J < njobs; J += OW) {
    const int64_t i = J / (CW * C::kRows);
    const int c = (int)((J / C::kRows) % CW), r = (int)(J % C::kRows);
    const int64_t g = first + c + i * gstep;
    const int h = (int)(i % C::kHand);
    if (g < groups) {
      K1S_T(th);
      if (lane == 0) mbar_wait(hfull(c, h), (uint32_t)((i / C::kHand) & 1));
      __syncwarp();
      K1S_ADD(4, th);
    }
    const int64_t row = row_lo + g * C::kRows + r;
    if (g < groups && row < row_hi) {
      const double *hs = hslot(c, h);
      const double m = hs[r], sc = hs[C::kRows + r], pw = hs[2 * C::kRows + r];
      const bool ssd_zero = hs[3 * C::kRows + r] != 0.0;
      const RowDiv dv = row_div(ssd_zero ? 1.0 : sc);
      const int64_t off = row * ldu;
      // window w of this row into slot s (lane 0): kBox pieces up to l, none
      // for ssd-zero rows or windows past l (their barriers complete by the
      // arrival alone)
      auto issue = [&](int64_t w, int s) {
        if (lane < C::kOWin / C::kBox) {  // lane h: piece h (one box {kBox, 1}), its own arrival
          const int64_t k0 = w * C::kOWin + lane * C::kBox;
          const bool live = !ssd_zero && k0 < l && !(PCC_K1S_EXP & 4);
          mbar_arrive_expect_tx(ofull(o, s), live ? (uint32_t)(C::kBox * 8) : 0u);
          if (live)
            tma_load_2d_hint(my_ring_s + (uint32_t)((s * C::kOWin + lane * C::kBox) * 8), &xmap, (int32_t)k0,
                             (int32_t)row, ofull(o, s), pol);
        }
      };
      int ps = slot;
      for (int64_t w = 0; w < C::kOStages - 1 && w < otot; ++w) {
        issue(w, ps);
        if (++ps == C::kOStages) ps = 0;
      }
      double x0 = 0.0;
      bool varies = false;
      for (int64_t w = 0; w < otot; ++w) {
        if (w + C::kOStages - 1 < otot) {
          issue(w + C::kOStages - 1, ps);
          if (++ps == C::kOStages) ps = 0;
        }
        {
          K1S_T(tw);
          if (lane == 0) mbar_wait(ofull(o, slot), phase);
          __syncwarp();
          K1S_ADD(5, tw);
        }
        const double *win = my_ring + slot * C::kOWin;
        if (w == 0) x0 = win[0];
        const int64_t k0 = w * C::kOWin;
        // u = (x - mean) / scale by the one-FMA-correction quotient (div_rn
        // of normalize.cuh, bit-identical to __ddiv_rn) wherever its guard
        // holds; the guard -- a == +0 or 2^-520 <= |a| (b is in range per
        // row: dv.fast) -- is tested on the bits, and a window in which any
        // element fails it (never seen in practice: -0, tiny or subnormal
        // x - mean) is emitted again with __ddiv_rn.  Loop bounds and the vote
        // are warp-uniform.
        bool bad = false;
        auto quot = [&](double a, bool exact) {
          if (exact) return __ddiv_rn(a, dv.b);
          const double q0 = __dmul_rn(a, dv.y);
          const int hi = __double2hiint(a), lo = __double2loint(a);
          bad |= ((hi & 0x7fffffff) < ((1023 - 520) << 20)) & ((hi | lo) != 0);
          return __fma_rn(__fma_rn(-q0, dv.b, a), dv.y, q0);
        };
        const bool full = k0 + C::kOWin <= l && k0 + C::kOWin <= kend;  // no bounds inside the window
        auto emit = [&](bool exact) {
          if (MODE == kNormDigits) {
            if (pw > 0.0 && full) {
#pragma unroll 2
              for (int it = 0; it < C::kOWin / 128; ++it) {
                const int kk = 128 * it + 4 * lane;
                const double2 a2 = *reinterpret_cast<const double2 *>(win + kk);
                const double2 b2 = *reinterpret_cast<const double2 *>(win + kk + 2);
                const double v4[4] = {a2.x, a2.y, b2.x, b2.y};
                if (!exact) varies |= (v4[0] != x0) | (v4[1] != x0) | (v4[2] != x0) | (v4[3] != x0);
                uint32_t packed[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
                for (int t = 0; t < 4; ++t) split_digits7(__dmul_rn(quot(__dsub_rn(v4[t], m), exact), pw), t, packed);
                const int64_t k = k0 + kk;
                int8_t *dst = dests.slices + (k / W) * 7 * plane + row * W + (k % W);
#pragma unroll
                for (int t = 0; t < 7; ++t) __stcs(reinterpret_cast<unsigned int *>(dst + t * plane), packed[t]);
              }
            } else {
              for (int it = 0; it < C::kOWin / 128; ++it) {
                if (k0 + 128 * it >= kend) break;
                const int kk = 128 * it + 4 * lane;
                const int64_t k = k0 + kk;
                uint32_t packed[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
                if (pw > 0.0) {
                  double v4[4];
#pragma unroll
                  for (int t = 0; t < 4; ++t) v4[t] = (k + t < l) ? win[kk + t] : x0;
                  if (!exact) varies |= (v4[0] != x0) | (v4[1] != x0) | (v4[2] != x0) | (v4[3] != x0);
#pragma unroll
                  for (int t = 0; t < 4; ++t)
                    split_digits7((k + t < l) ? __dmul_rn(quot(__dsub_rn(v4[t], m), exact), pw) : 0.0, t, packed);
                }
                if (k < kend) {
                  int8_t *dst = dests.slices + (k / W) * 7 * plane + row * W + (k % W);
#pragma unroll
                  for (int t = 0; t < 7; ++t) __stcs(reinterpret_cast<unsigned int *>(dst + t * plane), packed[t]);
                }
              }
            }
          } else {
            auto put = [&](int64_t k, double2 v) {
              if (MODE == kNormBcast) {
                for (int d = 0; d < dests.n; ++d) __stcs(reinterpret_cast<double2 *>(dests.u[d] + off + k), v);
              } else {
                __stcs(reinterpret_cast<double2 *>(u + off + k), v);
              }
            };
            if (!ssd_zero && full) {
              // 4 pairs per lane in flight: loads, then quotients, then stores
#pragma unroll
              for (int it = 0; it < C::kOWin / 64; it += 4) {
                double2 xv[4], v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) xv[q] = *reinterpret_cast<const double2 *>(win + 64 * (it + q) + 2 * lane);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  if (!exact) varies |= (xv[q].x != x0) | (xv[q].y != x0);
                  v[q].x = quot(__dsub_rn(xv[q].x, m), exact);
                  v[q].y = quot(__dsub_rn(xv[q].y, m), exact);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) put(k0 + 64 * (it + q) + 2 * lane, v[q]);
              }
            } else {
              for (int it = 0; it < C::kOWin / 64; ++it) {
                if (k0 + 64 * it >= kend) break;
                const int kk = 64 * it + 2 * lane;
                const int64_t k = k0 + kk;
                double2 v = make_double2(0.0, 0.0);
                if (!ssd_zero && k < l) {  // l even: a pair never straddles l
                  const double2 xv = *reinterpret_cast<const double2 *>(win + kk);
                  if (!exact) varies |= (xv.x != x0) | (xv.y != x0);
                  v.x = quot(__dsub_rn(xv.x, m), exact);
                  v.y = quot(__dsub_rn(xv.y, m), exact);
                }
                if (k < kend) put(k, v);
              }
            }
          }
        };
        if (!(PCC_K1S_EXP & 1)) {
          emit(!dv.fast);
          if (dv.fast && __any_sync(0xffffffffu, bad)) emit(true);
        }
        __syncwarp();  // the slot is consumed before it is refilled
        if (++slot == C::kOStages) {
          slot = 0;
          phase ^= 1u;
        }
      }
      // the reference's exact constancy test (x == x[0] everywhere); a
      // constant row with a nonzero rounded ssd is rewritten with zeros
      const bool constant = !ssd_zero && !__any_sync(0xffffffffu, varies) && !(PCC_K1S_EXP & 5);
      const bool zero = ssd_zero || constant;
      if (constant) {
        if (MODE == kNormDigits) {
          for (int64_t k = 4 * lane; k < kend; k += 128) {
            int8_t *dst = dests.slices + (k / W) * 7 * plane + row * W + (k % W);
            for (int t = 0; t < 7; ++t) *reinterpret_cast<unsigned int *>(dst + t * plane) = 0u;
          }
        } else {
          for (int64_t k = 2 * lane; k < kend; k += 64) {
            if (MODE == kNormBcast) {
              for (int d = 0; d < dests.n; ++d)
                *reinterpret_cast<double2 *>(dests.u[d] + off + k) = make_double2(0.0, 0.0);
            } else {
              *reinterpret_cast<double2 *>(u + off + k) = make_double2(0.0, 0.0);
            }
          }
        }
      }
      if (lane == 0) {
        if (MODE == kNormBcast) {
          for (int d = 0; d < dests.n; ++d) dests.flags[d][row] = zero ? 1 : 0;
        } else {
          zero_variance[row] = zero ? 1 : 0;
        }
        if (MODE == kNormDigits) dests.scale[row] = (zero || pw == 0.0) ? 0.0 : 1.0 / pw;  // 2^(e-7), exact
      }
    }
    if (g < groups) {
      __syncwarp();
      if (lane == 0) mbar_arrive(hempty(c, h));
    }
  }
  K1S_ADD(3, t_out);
}

}  // namespace pcc
