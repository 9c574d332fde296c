// EXPERIMENT (not built into the product library): the streamed K1 of round 2,
// measured slower than the staged kernel at every BASELINE config (DESIGN.md §3 K1,
// profiles/r02_k1_experiments.md).  Kept as the record of that design; the
// build line is in tools/k1s_probe.cu.
// normalize_stream.cuh -- K1, streamed: per-variable z-normalisation at HBM
// bandwidth, bit-exact to the reference's _kernels.normalize_rows
// (_kernels.py:226-252; same arithmetic contract as normalize.cuh).
//
// Why a second K1.  The reference's reductions are eight strictly
// sequential lane chains per row (sum8, then ssd8 with the mean, l/8
// dependent FP64 adds each, _kernels.py:71-165), so a row's statistics take
// 2 * l/8 DADD latencies (c4: ~16 K cycles) however many threads it gets.
// The staged kernel (normalize.cuh) keeps whole rows in shared memory for
// that time, which caps the rows in flight per SM at 228 KB / row bytes (3 at
// c4) and leaves HBM idle.  Here a row is never resident: it streams through
// shared memory three times -- sum pass, ssd pass, output pass -- in 512-
// element windows, and only the windows in flight occupy shared memory.
//
//   * one warp owns 4 rows (8 lanes each: lane j of row r IS reference lane j);
//     lane 0 is the warp's producer: per window one 1-D bulk copy per row
//     (cp.async.bulk, byte-counted mbarrier) into a kStages-deep per-warp
//     ring; the warp's three passes are one continuous job stream that runs
//     across row groups, so the next group's first windows land while the
//     current group's output pass runs;
//   * the first read of a row is from HBM (its whole rows are prefetched to L2
//     with cp.async.bulk.prefetch.L2 one group ahead); the second and third
//     reads hit L2 because the grid is sized so that the rows in flight fit a
//     fixed L2 budget (host side: pcc_b200.cu) -- DRAM traffic stays one read
//     of X + one write of U;
//   * output pass: all 32 lanes write u = (x - mean) / scale for the 4 rows
//     with coalesced stores (or the broadcast / digit-plane variants of the
//     staged kernel, same IEEE operations).
// Requires 16-byte aligned rows and even l (bulk copies move 16-byte
// multiples); other shapes use the staged kernel.
#pragma once

#include "../../paper_1605_01584_b200/csrc/normalize.cuh"

namespace pcc {

#ifdef PCC_K1S_PROBE
// tools/k1s_probe.cu: clock64 totals -- [0] chain data waits, [1] chain
// handoff waits, [2] chain total, [3] output waits, [4] output total
__device__ unsigned long long g_k1s_probe[8];
#define K1S_T0() const long long k1s_t0_ = clock64()
#define K1S_ADD(i, t) \
  do {                \
    if (lane == 0) atomicAdd(&g_k1s_probe[i], (unsigned long long)(clock64() - (t))); \
  } while (0)
#else
#define K1S_T0() \
  do {           \
  } while (0)
#define K1S_ADD(i, t) \
  do {                \
  } while (0)
#endif

struct K1Stream {
  static constexpr int kWin = 1024;      // doubles per row window
  static constexpr int kRows = 4;        // rows per chain warp (8 lanes each)
  // ring depth (windows in flight per chain warp): 6 with 1-2 chain warps, 3 with 3-4
  __host__ __device__ static constexpr int stages(int cw) { return cw <= 2 ? 3 : 1; }
  static constexpr int kHand = 2;        // handoff slots per chain warp (chain -> output warps)
  static constexpr int kApplyWarps = 8;  // output warps per CTA
  static constexpr int kStageDoubles = kRows * kWin;
  __host__ __device__ static constexpr int ring_bytes(int cw) { return stages(cw) * kStageDoubles * 8; }
  // rings + full barriers + handoff full/empty barriers + handoff values
  __host__ __device__ static constexpr int smem_bytes(int cw) {
    return cw * ring_bytes(cw) + 8 * (cw * stages(cw) + 2 * cw * kHand) + 8 * (cw * kHand * 4 * kRows);
  }
};

// 1-D bulk copy global -> shared with an L2 eviction-priority policy
// (createpolicy): the chain passes mark X evict_last so it survives until the
// output pass re-reads it.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_copy_row_hint(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                                   uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
// Digit planes of 4 consecutive normalised values (kNormDigits, as the
// staged kernel): 7 radix-128 digits each, packed 4 per uint32 per plane.
__device__ __forceinline__ void digits4(const double *v4, double m0, double sc, double pw, bool live,
                                        uint32_t packed[7]) {
#pragma unroll
  for (int i = 0; i < 7; ++i) packed[i] = 0u;
  if (!live) return;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double v = v4[j];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const double t = __dadd_rn(v, 0x1.8p52);  // rint by the 1.5 * 2^52 shift
      const double d = __dsub_rn(t, 0x1.8p52);
      v = __dmul_rn(__dsub_rn(v, d), 128.0);    // exact
      packed[i] |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * j);
    }
  }
}

// One reference lane chain continued over a window (stride 8), loads
// software-pipelined PF steps ahead of the dependent adds:
//   SSD = false: s += x (sum8 lane) and the constancy test x != ref (= x[0]);
//   SSD = true:  d = x - ref (= mean), s += RN(d * d) (ssd8 lane), and with
//                DMAX the running max |d| (split digits; max is exact).
template <bool SSD, bool DMAX, int PF>
__device__ __forceinline__ void stream_chain(double &s, const double *p, int nsteps, double ref, bool &varies,
                                             double &dmax) {
  auto step = [&](double v) {
    if (SSD) {
      const double d = __dsub_rn(v, ref);
      s = __dadd_rn(s, __dmul_rn(d, d));
      if (DMAX) dmax = fmax(dmax, fabs(d));
    } else {
      s = __dadd_rn(s, v);
      varies |= (v != ref);
    }
  };
  // two register batches in ping-pong: batch B loads while batch A adds and
  // vice versa -- no register copies between iterations
  const int full = (nsteps / (2 * PF)) * (2 * PF);
  double a[PF], b[PF];
  if (full > 0) {
#pragma unroll
    for (int i = 0; i < PF; ++i) a[i] = p[8 * i];
  }
  int t = 0;
  for (; t < full; t += 2 * PF) {
#pragma unroll
    for (int i = 0; i < PF; ++i) b[i] = p[8 * (t + PF + i)];
#pragma unroll
    for (int i = 0; i < PF; ++i) step(a[i]);
    if (t + 2 * PF < full) {
#pragma unroll
      for (int i = 0; i < PF; ++i) a[i] = p[8 * (t + 2 * PF + i)];
    }
#pragma unroll
    for (int i = 0; i < PF; ++i) step(b[i]);
  }
  for (; t < nsteps; ++t) step(p[8 * t]);
}

// ---------------------------------------------------------------------------
// The kernel.  CTA = CW chain warps + kApplyWarps output warps, one CTA per SM.
//
// Chain warp c owns 4 rows at a time (a "group"; groups are dealt round-robin
// over every chain warp of the grid).  Its lane 0 streams the group's rows
// through the warp's ring (one 1-D bulk copy per row and window, byte-counted
// mbarrier per slot): first the sum pass, then the ssd pass.  At the end of
// the ssd pass lane 8r publishes row r's (mean, scale, zero, digit scale) in
// one of kHand handoff slots and writes its flag; the chain warp moves on.
// The output warps take the handoff slots in group order, re-read the 4 rows
// from L2 with 16-byte loads and write U (or the broadcast / digit planes).
template <int MODE, int CW>
__global__ void __launch_bounds__((CW + K1Stream::kApplyWarps) * 32, 1)
normalize_rows_stream_kernel(const double *__restrict__ x, int64_t ldx, double *__restrict__ u, int64_t ldu,
                             uint8_t *__restrict__ zero_variance, int64_t l, int64_t row_lo, int64_t row_hi,
                             NormDests dests, int flags) {
  using C = K1Stream;
  constexpr int STAGES = C::stages(CW), RING = C::ring_bytes(CW);
  extern __shared__ __align__(128) double ring[];  // [CW][kStages][kRows][kWin], then barriers + handoff
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring_base = smem_u32(ring);
  const uint32_t bars = ring_base + CW * RING;
  auto full_bar = [&](int c, int s) { return bars + 8u * (c * STAGES + s); };
  auto hfull_bar = [&](int c, int h) { return bars + 8u * (CW * STAGES + c * C::kHand + h); };
  auto hempty_bar = [&](int c, int h) { return bars + 8u * (CW * STAGES + CW * C::kHand + c * C::kHand + h); };
  // handoff slot (c, h): per row mean, scale, digit power, zero flag
  double *hand = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(ring) + CW * RING +
                                            8 * (CW * STAGES + 2 * CW * C::kHand));
  auto hslot = [&](int c, int h) { return hand + (c * C::kHand + h) * 4 * C::kRows; };

  const int64_t nw = (l + C::kWin - 1) / C::kWin;  // windows per row
  const int64_t groups = (row_hi - row_lo + C::kRows - 1) / C::kRows;
  const int64_t gstep = (int64_t)gridDim.x * CW;    // chain warps in the grid

  if (threadIdx.x == 0) {
    for (int c = 0; c < CW; ++c) {
      for (int s = 0; s < STAGES; ++s) mbar_init(full_bar(c, s), C::kRows);
      for (int h = 0; h < C::kHand; ++h) {
        mbar_init(hfull_bar(c, h), 1);
        mbar_init(hempty_bar(c, h), C::kApplyWarps);
      }
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp < CW) {
    // ------------------------------------------------------------ chain warp
    const int c = warp;
    const int r = lane >> 3, j = lane & 7;
    const int64_t g0 = (int64_t)blockIdx.x * CW + c;
    if (g0 >= groups) return;
    const int64_t my_groups = (groups - g0 + gstep - 1) / gstep;
    const int64_t total_jobs = my_groups * 2 * nw;
    const uint32_t my_ring = ring_base + c * RING;
    const uint64_t pol = l2_policy_evict_last();
    const double *my_ring_p = ring + c * (RING / 8);

    // The warp's job stream: group gi (rows r0 .. r0 + 3), pass 0 / 1, window
    // w, into ring slot (job index) % kStages.  Producer cursor (lanes 8q):
    // lane 8q issues row q's window (bulk copies issued by one thread complete
    // one at a time -- tools/bulk_bw.cu -- so the four rows go out from four
    // lanes); each of the four lanes arrives on the slot's barrier (count 4),
    // with the expected bytes of its row if the row exists.  All indices are
    // advanced incrementally (no 64-bit division in the loop).
    const int nwi = (int)nw;
    int p_w = 0, p_pass = 0, p_slot = 0;
    int64_t p_r0 = row_lo + g0 * C::kRows, p_issued = 0;
    auto issue_next = [&]() {
      const int64_t k0 = (int64_t)p_w * C::kWin;
      const uint32_t bytes = (uint32_t)(min((int64_t)C::kWin, l - k0) * 8);
      if (p_r0 + r < row_hi) {
        mbar_arrive_expect_tx(full_bar(c, p_slot), bytes);
        bulk_copy_row_hint(my_ring + (uint32_t)((p_slot * C::kStageDoubles + r * C::kWin) * 8),
                           x + (p_r0 + r) * ldx + k0, bytes, full_bar(c, p_slot), pol);
      } else {
        mbar_arrive(full_bar(c, p_slot));
      }
      if (++p_w == nwi) {
        p_w = 0;
        if (++p_pass == 2) {
          p_pass = 0;
          p_r0 += gstep * C::kRows;
        }
      }
      if (++p_slot == STAGES) p_slot = 0;
      ++p_issued;
    };
    if (j == 0)
      for (int q = 0; q < STAGES - 1 && p_issued < total_jobs; ++q) issue_next();

#ifdef PCC_K1S_PROBE
    const long long tc = clock64();
#endif
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t gi = 0; gi < my_groups; ++gi) {
      const int64_t r0 = row_lo + (g0 + gi * gstep) * C::kRows;
      const int rows = (int)min((int64_t)C::kRows, row_hi - r0);
      const bool active = r < rows;
      double s = 0.0, ref = 0.0, mean = 0.0, q = 0.0, dmax = 0.0;
      bool varies = false, constant = false;
      for (int pass = 0; pass < 2; ++pass) {
        for (int w = 0; w < nwi; ++w) {
          if (j == 0 && p_issued < total_jobs) issue_next();
          {
#ifdef PCC_K1S_PROBE
            const long long tw = clock64();
#endif
            // one lane polls the barrier, the warp barrier publishes the window
            if (lane == 0) mbar_wait(full_bar(c, slot), phase);
            __syncwarp();
            K1S_ADD(0, tw);
          }
          const int k0 = w * C::kWin;
          const int cnt = (int)min((int64_t)C::kWin, l - (int64_t)k0);
          const double *p = my_ring_p + slot * C::kStageDoubles + r * C::kWin;
          const int nst = (cnt - j + 7) >> 3;
          if (pass == 0) {
            if (active) {
              if (w == 0) ref = p[0];  // x[0]: every element is compared with it
#ifndef PCC_K1S_NO_CHAIN
              stream_chain<false, false, 8>(s, p + j, nst, ref, varies, dmax);
#endif
            }
            if (w == nwi - 1) {  // sum pass done: tree, constancy, mean
              s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
              s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
              s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
              const unsigned vb = __ballot_sync(0xffffffffu, varies);
              constant = (vb & (0xffu << (lane & 24))) == 0u;
              mean = (active && !constant) ? __ddiv_rn(s, (double)l) : 0.0;
            }
          } else if (active && !constant) {
            stream_chain<true, MODE == kNormDigits, 8>(q, p + j, nst, mean, varies, dmax);
          }
          __syncwarp();  // every lane is done with the slot before it is refilled
          if (++slot == STAGES) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
      // ssd pass done: tree, zero-variance rule, scale
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 1));
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 2));
      q = __dadd_rn(q, __shfl_xor_sync(0xffffffffu, q, 4));
      const bool zero = constant || q == 0.0;
      const double sc = zero ? 0.0 : __dsqrt_rn(q);
      double pw = 0.0, row_scale = 0.0;
      if (MODE == kNormDigits) {
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        const double m = zero ? 0.0 : __ddiv_rn(dmax, sc);  // exact max |u| (division is monotone)
        int e = 0;
        if (m > 0.0) {
          frexp(m, &e);
          if (ldexp(m, 7 - e) >= 127.5) ++e;  // keep the leading digit within [-127, 127]
        }
        row_scale = m > 0.0 ? ldexp(1.0, e - 7) : 0.0;
        pw = m > 0.0 ? ldexp(1.0, 7 - e) : 0.0;
      }
      const int h = (int)(gi % C::kHand);
#ifdef PCC_K1S_PROBE
      const long long th = clock64();
#endif
      if (gi >= C::kHand) mbar_wait(hempty_bar(c, h), (uint32_t)(((gi / C::kHand) - 1) & 1));
      K1S_ADD(1, th);
      if (active && j == 0) {
        double *hs = hslot(c, h);
        hs[r] = mean;
        hs[C::kRows + r] = sc;
        hs[2 * C::kRows + r] = pw;
        hs[3 * C::kRows + r] = zero ? 1.0 : 0.0;
        if (MODE == kNormBcast) {
          for (int d = 0; d < dests.n; ++d) dests.flags[d][r0 + r] = zero ? 1 : 0;
        } else {
          zero_variance[r0 + r] = zero ? 1 : 0;
        }
        if (MODE == kNormDigits) dests.scale[r0 + r] = row_scale;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(hfull_bar(c, h));  // release: the slot's values are visible
    }
    K1S_ADD(2, tc);
    return;
  }

  // ------------------------------------------------------------ output warps
  constexpr int AT = C::kApplyWarps * 32;
  const int ta = threadIdx.x - CW * 32;
  const int64_t first = (int64_t)blockIdx.x * CW;
  const int64_t rounds = first < groups ? (groups - first + gstep - 1) / gstep : 0;
#ifdef PCC_K1S_PROBE
  const long long ta0 = clock64();
#endif
  for (int64_t gi = 0; gi < rounds; ++gi) {
    for (int c = 0; c < CW; ++c) {
      const int64_t g = first + c + gi * gstep;
      if (g >= groups) break;
      const int h = (int)(gi % C::kHand);
#ifdef PCC_K1S_PROBE
      const long long tw = clock64();
#endif
      if (lane == 0) mbar_wait(hfull_bar(c, h), (uint32_t)((gi / C::kHand) & 1));
      __syncwarp();
      K1S_ADD(3, tw);
      const double *hs = hslot(c, h);
      const int64_t r0 = row_lo + g * C::kRows;
      const int rows = (int)min((int64_t)C::kRows, row_hi - r0);
#ifdef PCC_K1S_NO_APPLY
      if (rows >= 0) {
      } else
#endif
      if (MODE == kNormDigits) {
        // 4 consecutive elements per thread and step, the next step's two
        // 16-byte loads in flight while this step's digits are computed
        constexpr int W = 64;  // SplitCfg::kRowBytes
        const int64_t plane = dests.rows_total * W;
        const int64_t kpad = (l + W - 1) / W * W;
        const int64_t steps_row = (kpad + 4 * AT - 1) / (4 * AT);
        const int64_t nsteps = rows * steps_row;
        auto load4 = [&](int64_t q, double2 &a0, double2 &a1) {
          const int rr = (int)(q / steps_row);
          const int64_t k = (q - rr * steps_row) * (4 * AT) + 4 * ta;
          const double *xr = x + (r0 + rr) * ldx;
          a0 = (k + 1 < l) ? __ldcs(reinterpret_cast<const double2 *>(xr + k)) : make_double2(k < l ? xr[k] : 0.0, 0.0);
          a1 = (k + 3 < l) ? __ldcs(reinterpret_cast<const double2 *>(xr + k + 2))
                           : make_double2(k + 2 < l ? xr[k + 2] : 0.0, 0.0);
        };
        auto emit4 = [&](int64_t q, double2 a0, double2 a1) {
          const int rr = (int)(q / steps_row);
          const int64_t k = (q - rr * steps_row) * (4 * AT) + 4 * ta;
          if (k >= kpad) return;
          const double m = hs[rr], sc = hs[C::kRows + rr], pw = hs[2 * C::kRows + rr];
          const bool zero = hs[3 * C::kRows + rr] != 0.0;
          double v4[4] = {a0.x, a0.y, a1.x, a1.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v4[i] = (k + i < l && !zero) ? __dmul_rn(div_rn(__dsub_rn(v4[i], m), row_div(sc)), pw) : 0.0;
          uint32_t packed[7];
          digits4(v4, m, sc, pw, pw > 0.0, packed);
          int8_t *dst = dests.slices + (k / W) * 7 * plane + (r0 + rr) * W + (k % W);
#pragma unroll
          for (int i = 0; i < 7; ++i) __stcs(reinterpret_cast<unsigned int *>(dst + i * plane), packed[i]);
        };
        double2 p0, p1, q0, q1;
        if (nsteps > 0) load4(0, p0, p1);
        for (int64_t q = 0; q < nsteps; q += 2) {
          if (q + 1 < nsteps) load4(q + 1, q0, q1);
          emit4(q, p0, p1);
          if (q + 2 < nsteps) load4(q + 2, p0, p1);
          if (q + 1 < nsteps) emit4(q + 1, q0, q1);
        }
      } else {
        // U rows (or the broadcast): chunks of 2 * AT * U doubles, the next
        // chunk's U 16-byte loads in flight while this chunk is divided and
        // stored; the chunk sequence runs over the group's rows and the zero
        // K padding (l and ldu are even, so a 16-byte pair never straddles l)
        constexpr int U = 16, CH = 2 * AT * U;
        for (int rr = 0; rr < rows; ++rr) {
          const double m = hs[rr];
          const bool zero = hs[3 * C::kRows + rr] != 0.0;
          const RowDiv dv = row_div(hs[C::kRows + rr]);
          const double *xr = x + (r0 + rr) * ldx;
          const int64_t off = (r0 + rr) * ldu;
          for (int64_t k0 = 2 * (int64_t)ta; k0 < ldu; k0 += CH) {
            double2 v[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
              const int64_t kk = k0 + 2 * AT * i;
              v[i] = (kk < l) ? __ldcs(reinterpret_cast<const double2 *>(xr + kk)) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int i = 0; i < U; ++i) {
              const int64_t kk = k0 + 2 * AT * i;
              if (kk >= ldu) continue;
              double2 o = make_double2(0.0, 0.0);
              if (!zero && kk < l) {
                o.x = div_rn(__dsub_rn(v[i].x, m), dv);
                o.y = div_rn(__dsub_rn(v[i].y, m), dv);
              }
              if (MODE == kNormBcast) {
                for (int d = 0; d < dests.n; ++d) __stcs(reinterpret_cast<double2 *>(dests.u[d] + off + kk), o);
              } else {
                __stcs(reinterpret_cast<double2 *>(u + off + kk), o);
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(hempty_bar(c, h));
    }
  }
  K1S_ADD(4, ta0);
}

}  // namespace pcc
