// split.cuh -- the split-integer contraction ("split mode"): U·Uᵀ to FP64
// accuracy on the 5th-generation tensor cores (tcgen05.mma kind::i8, s32
// accumulators in TMEM), the Ozaki splitting scheme.
//
// Each normalised row u_r (‖u_r‖ = 1 or u_r = 0) is written exactly as
//     u_r = 2^(e_r) · Σ_{i=1..7} s_{r,i} · 2^(-7i) + ρ_r,
// s_{r,1} ∈ [-127, 127], s_{r,i≥2} ∈ [-64, 64] (round-to-nearest digits of
// a radix-128 expansion; every step is an exact FP64 operation), with
// 2^(e_r) ≤ 2·max|u_r| and |ρ_r,k| ≤ max|u_r|·2^-49.  Then
//     u_y·u_x ≈ 2^(e_y+e_x) Σ_{d=2..9} 2^(-7d) · A_d,
//     A_d = Σ_{i+j=d} S_i(y)·S_j(x)            (int8 dot products, exact in s32)
// i.e. 34 int8 GEMM products (all i, j ≤ 7 with i + j ≤ 9), summed per
// diagonal d in one s32 TMEM accumulator each (|A_d| ≤ 7·127·64·l < 2³¹ for
// l ≤ 8192), combined in FP64 by Horner's rule in the epilogue.  Error
// bound per coefficient at full depth, l ≤ 8192 (K2s):
// representation ≤ 2·√l·2^-49 ≈ 3.2e-13, dropped products (i + j ≥ 10)
// ≤ 5.7e-13, FP64 combination ~1e-16 — inside the north star's 1e-12.
//
// (1-based digit indices above; the code uses 0-based i, j = 0..6 and
// diagonals sd = i + j = d - 2.)  Adaptive depth drops sd = 7 per tile pair
// when its rows allow (split_drop_top); DESIGN.md §3 "K2s" has the bounds.
//
// Layouts.  Slices: int8 [KB][7][R][64] (KB = ⌈l/64⌉ K blocks of 64, R =
// padded rows): one TMA box {64 B, 128 rows, 1 slice} is an 8 KB operand
// tile of two MMA K steps, K-major with the 64-byte swizzle the UMMA
// descriptor names.  Scales: double[R] = 2^(e_r - 7), 0 for all-zero rows.
//
// Kernel (one 128 x 128 GPU tile of the bijection per CTA at a time,
// persistent, grouped L2-locality order like K2): warp 0 = TMA producer,
// warp 1 = TMEM owner + MMA issuer (one thread), warps 2..9 = epilogue.
// TMEM (512 columns) holds four 128 x 128 s32 accumulators, so each tile
// takes two passes over K: pass 0 accumulates sd = 4..7 (slices 0..6),
// pass 1 sd = 0..3 (slices 0..3) -- at adaptive depth sd = 3..6 (slices
// 0..6), then sd = 0..2 (slices 0..2) -- each with the "domino" schedules below
// (N = 256 MMAs for neighbouring-diagonal digit pairs); the epilogue warps
// fold pass 0 into FP64 registers (Horner) while pass 1 runs, then finish
// and store through the same store_cell() as K2 (packed / dense / tiles).
#pragma once

#include "common.cuh"
#include "syrk.cuh"
#include "tcgen05.cuh"

namespace pcc {

struct SplitCfg {
  static constexpr int kSlices = 7;
  static constexpr int kKStep = 32;                      // int8 K of one MMA
  static constexpr int kRowBytes = 64;                   // int8 K per staged row = per stage (2 MMA K steps)
  static constexpr int kKSub = kRowBytes / kKStep;
  static constexpr int kSliceBytes = kTile * kRowBytes;  // 8 KB: one 128-row operand tile of a stage
  static constexpr int kOpBytes = kSlices * kSliceBytes; // 56 KB
  static constexpr int kStageBytes = 2 * kOpBytes;       // A + B
  static constexpr int kStages = 2;
  static constexpr int kEpiWarps = 8;
  static constexpr int kThreads = 32 * (2 + kEpiWarps);
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kBarBytes = 8 * (kStages * kSlices + kStages + 2) + 16;  // full per (stage, slice)
  static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kBarBytes;
  static constexpr int64_t kMaxL = 8192;  // the error bound above holds up to here
  // Adaptive depth: a tile pair skips diagonal d = 9 (0-based sd = 7: 6 of
  // the 34 products) when its own rows bound the resulting error by
  // kDropBudget (split_drop_top below).
  static constexpr double kDropBudget = 5e-13;
};

// Whole warp, same result in every lane: may tile pair (Y, X) drop the sd = 7
// products?  With s = the tile's largest row scale (scale_r = 2^(e_r-7),
// |digits| <= 64 past the first), the dropped products sd >= 7 add at most
//     s_Y s_X l 64^2 (6 + 5/128 + ...) 128^-7  <=  s_Y s_X l 6.04 2^-37
// per coefficient, and the 7-digit representation (|rho| <= s 2^-43,
// ||u||_1 <= sqrt(l)) at most (s_Y + s_X) 2^-43 sqrt(l); drop when their sum
// is <= kDropBudget.  Rows that are all zero (and pad rows) have scale 0.
__device__ __forceinline__ bool split_drop_top(const double *__restrict__ scale, uint64_t Y, uint64_t X, int lane,
                                               double l_f, double sqrt_l) {
  double sy = 0.0, sx = 0.0;
#pragma unroll
  for (int r = lane; r < kTile; r += 32) {
    sy = fmax(sy, __ldg(scale + Y * kTile + r));
    sx = fmax(sx, __ldg(scale + X * kTile + r));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sy = fmax(sy, __shfl_xor_sync(0xffffffffu, sy, o));
    sx = fmax(sx, __shfl_xor_sync(0xffffffffu, sx, o));
  }
  const double bound = sy * sx * l_f * (6.04 * 0x1p-37) + (sy + sx) * 0x1p-43 * sqrt_l;
  return bound <= SplitCfg::kDropBudget;
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int32_t c0, int32_t c1,
                                            int32_t c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// ---- MMA schedules -------------------------------------------------------
// An int8 MMA costs ~92 clk for N <= 128 but only 128 clk for N = 256 (the
// MAC floor, profiles/r01_i8_mma_peak.log), so digit pairs (i, j), (i, j+1)
// of neighbouring diagonals go out as one N = 256 MMA whose B operand is the
// two consecutive slice tiles j, j+1 of the X band and whose two 128-column
// halves land in neighbouring accumulators.  Entry = i | j << 3 | wide << 6 |
// zero << 7; `zero` marks each accumulator's first write of a tile (no
// accumulate at the first K step) and precedes every other entry touching
// it.  Entries are ordered by the highest slice they read (the stage's
// slices land one by one) and so that consecutive MMAs mostly target
// different accumulators.  The integer sums are exact, so any schedule gives
// the same bits.
// Schedule S entry e, as i | j << 3 | wide << 6 | zero << 7 -- a constexpr
// switch so the unrolled issue loop folds every entry into immediates:
//   full depth (34 products):      pass 0 = S 1, diagonals 4..7 (24 products,
//                                  slices 0..6); pass 1 = S 0, diagonals 0..3
//                                  (10 products, slices 0..3);
//   adaptive depth (28 products):  pass 0 = S 3, diagonals 3..6 (22 products,
//                                  slices 0..6); pass 1 = S 2, diagonals 0..2
//                                  (6 products, slices 0..2, accumulator 3 unused).
// Either way the epilogue's Horner chain runs from the top diagonal down to 0
// in the same order (pass 0's accumulators, then pass 1's), so the split of
// the diagonals between the passes does not change a bit of the result; the
// adaptive split loads 10 digit slices per K block instead of 11 and issues
// 22 N = 256 + 4 N = 128 MMAs per K step pair instead of 20 + 16.
__host__ __device__ constexpr int sched_len(int S) { return S == 0 ? 6 : (S == 1 ? 13 : (S == 2 ? 4 : 12)); }
// First diagonal of schedule S (its accumulator 0).
__host__ __device__ constexpr int sched_lo(int S) { return S == 1 ? 4 : (S == 3 ? 3 : 0); }
__host__ __device__ constexpr uint32_t sched_entry(int S, int e) {
  if (S == 0) {
    switch (e) {
      case 0: return 2u | (0u << 3) | (1u << 6) | (1u << 7);  // (2, 0) wide zero
      case 1: return 0u | (0u << 3) | (1u << 6) | (1u << 7);  // (0, 0) wide zero
      case 2: return 1u | (2u << 3) | (0u << 6) | (0u << 7);  // (1, 2)
      case 3: return 1u | (0u << 3) | (1u << 6) | (0u << 7);  // (1, 0) wide
      case 4: return 3u | (0u << 3) | (0u << 6) | (0u << 7);  // (3, 0)
      case 5: return 0u | (2u << 3) | (1u << 6) | (0u << 7);  // (0, 2) wide
    }
  }
  if (S == 1) {
    switch (e) {
      case 0: return 3u | (1u << 3) | (1u << 6) | (1u << 7);  // (3, 1) wide zero
      case 1: return 3u | (3u << 3) | (1u << 6) | (1u << 7);  // (3, 3) wide zero
      case 2: return 2u | (2u << 3) | (1u << 6) | (0u << 7);  // (2, 2) wide
      case 3: return 4u | (2u << 3) | (1u << 6) | (0u << 7);  // (4, 2) wide
      case 4: return 4u | (0u << 3) | (1u << 6) | (0u << 7);  // (4, 0) wide
      case 5: return 2u | (4u << 3) | (1u << 6) | (0u << 7);  // (2, 4) wide
      case 6: return 1u | (3u << 3) | (1u << 6) | (0u << 7);  // (1, 3) wide
      case 7: return 6u | (0u << 3) | (1u << 6) | (0u << 7);  // (6, 0) wide
      case 8: return 0u | (4u << 3) | (1u << 6) | (0u << 7);  // (0, 4) wide
      case 9: return 1u | (5u << 3) | (1u << 6) | (0u << 7);  // (1, 5) wide
      case 10: return 5u | (0u << 3) | (1u << 6) | (0u << 7);  // (5, 0) wide
      case 11: return 5u | (2u << 3) | (0u << 6) | (0u << 7);  // (5, 2)
      case 12: return 0u | (6u << 3) | (0u << 6) | (0u << 7);  // (0, 6)
    }
  }
  if (S == 2) {  // adaptive depth, second pass: diagonals 0..2 (6 products, accumulator 3 unused)
    switch (e) {
      case 0: return 0u | (0u << 3) | (1u << 6) | (1u << 7);  // (0, 0) wide zero
      case 1: return 2u | (0u << 3) | (0u << 6) | (1u << 7);  // (2, 0) zero
      case 2: return 1u | (0u << 3) | (1u << 6) | (0u << 7);  // (1, 0) wide
      case 3: return 0u | (2u << 3) | (0u << 6) | (0u << 7);  // (0, 2)
    }
  }
  if (S == 3) {  // adaptive depth, first pass: diagonals 3..6 (22 products)
    switch (e) {
      case 0: return 2u | (1u << 3) | (1u << 6) | (1u << 7);  // (2, 1) wide zero
      case 1: return 3u | (2u << 3) | (1u << 6) | (1u << 7);  // (3, 2) wide zero
      case 2: return 3u | (0u << 3) | (1u << 6) | (0u << 7);  // (3, 0) wide
      case 3: return 1u | (2u << 3) | (1u << 6) | (0u << 7);  // (1, 2) wide
      case 4: return 2u | (3u << 3) | (1u << 6) | (0u << 7);  // (2, 3) wide
      case 5: return 0u | (3u << 3) | (1u << 6) | (0u << 7);  // (0, 3) wide
      case 6: return 4u | (2u << 3) | (0u << 6) | (0u << 7);  // (4, 2)
      case 7: return 4u | (0u << 3) | (1u << 6) | (0u << 7);  // (4, 0) wide
      case 8: return 1u | (4u << 3) | (1u << 6) | (0u << 7);  // (1, 4) wide
      case 9: return 5u | (0u << 3) | (1u << 6) | (0u << 7);  // (5, 0) wide
      case 10: return 0u | (5u << 3) | (1u << 6) | (0u << 7);  // (0, 5) wide
      case 11: return 6u | (0u << 3) | (0u << 6) | (0u << 7);  // (6, 0)
    }
  }
  return 0;
}


// Issue one stage's MMAs for schedule S (0: diagonals 0..3; 1: 4..7; 2:
// 4..6) in straight-line code: both K steps of the 64-byte rows (K step
// outer, so consecutive MMAs alternate accumulators), each entry after
// waiting for the stage's slices it reads (the slices land in order; the
// barriers of (stage, slice) are 8 bytes apart from full0).
template <int S>
__device__ __forceinline__ void issue_stage(uint32_t tmem, uint32_t a, uint32_t b, bool first_k, uint32_t full0,
                                            uint32_t phase) {
  using C = SplitCfg;
  constexpr uint32_t idesc = idesc_i8_s32<128, 128>(), idesc256 = idesc_i8_s32<128, 256>();
  constexpr int s_lo = sched_lo(S);
  const uint64_t desc0 = umma_desc_k_sw64(0);
  int ready = -1;
#pragma unroll
  for (int ks = 0; ks < C::kKSub; ++ks) {
#pragma unroll
    for (int e = 0; e < sched_len(S); ++e) {
      const uint32_t ent = sched_entry(S, e);
      const uint32_t i = ent & 7u, j = (ent >> 3) & 7u, wide = (ent >> 6) & 1u, zero = ent >> 7;
      const int need = (int)(i > j + wide ? i : j + wide);
      if (ready < need) {
        while (ready < need) mbar_wait(full0 + 8u * (uint32_t)(++ready), phase);
        tc_fence_after();
      }
      const uint64_t da = desc0 + ((a + i * C::kSliceBytes + ks * C::kKStep) >> 4);
      const uint64_t db = desc0 + ((b + j * C::kSliceBytes + ks * C::kKStep) >> 4);
      umma_i8(tmem + 128u * (i + j - (uint32_t)s_lo), da, db, wide ? idesc256 : idesc,
              (zero && first_k && ks == 0) ? 0u : 1u);
    }
  }
}

// ---- slicing: U rows -> int8 digit planes + per-row scale ------------------
// One warp per row; lane handles 4 consecutive K of every 128-K chunk, so 8
// lanes fill one 32-byte (K block, slice, row) segment per store.
__global__ void __launch_bounds__(256) split_rows_kernel(const double *__restrict__ u, int64_t ldu, int64_t l,
                                                         int64_t row_lo, int64_t row_hi, int64_t rows_total,
                                                         int8_t *__restrict__ slices, double *__restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t r = row_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= row_hi) return;
  const double *row = u + r * ldu;  // rows start 256-byte aligned (ldu % 32 == 0)
  double m = 0.0;
  {
    const int64_t l2 = l & ~(int64_t)1;
    for (int64_t k = 2 * lane; k < l2; k += 64) {
      const double2 p = __ldg(reinterpret_cast<const double2 *>(row + k));
      m = fmax(m, fmax(fabs(p.x), fabs(p.y)));
    }
    if ((l & 1) && lane == 0) m = fmax(m, fabs(row[l - 1]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0) {
    frexp(m, &e);                                // m = f·2^e, f in [0.5, 1)
    if (ldexp(m, 7 - e) >= 127.5) ++e;           // keep the leading digit within [-127, 127]
  }
  if (lane == 0) scale[r] = m > 0.0 ? ldexp(1.0, e - 7) : 0.0;  // all-zero rows: 0 (digits are 0 too)
  // v = u * 2^(7-e): one exact multiply by a power of two (ldexp only when
  // that power itself would not be a finite double -- not for normalised rows)
  const bool pw_ok = 7 - e <= 1000;
  const double pw = pw_ok ? ldexp(1.0, 7 - e) : 0.0;
  constexpr int W = SplitCfg::kRowBytes;
  const int64_t kb_count = (l + W - 1) / W;
  const int64_t plane = rows_total * W;          // bytes between slice planes
  for (int64_t k0 = 0; k0 < kb_count * W; k0 += 128) {
    const int64_t k = k0 + 4 * lane;
    if (k >= kb_count * W) break;
    double x4[4];
    if (k + 3 < l) {
      const double2 p0 = __ldg(reinterpret_cast<const double2 *>(row + k));
      const double2 p1 = __ldg(reinterpret_cast<const double2 *>(row + k + 2));
      x4[0] = p0.x, x4[1] = p0.y, x4[2] = p1.x, x4[3] = p1.y;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) x4[j] = (k + j < l) ? row[k + j] : 0.0;
    }
    uint32_t packed[SplitCfg::kSlices] = {};
#pragma unroll
    for (int j = 0; j < 4; ++j) split_digits7(pw_ok ? x4[j] * pw : ldexp(x4[j], 7 - e), j, packed);
    const int64_t kb = k / W;
    int8_t *dst = slices + (kb * SplitCfg::kSlices) * plane + r * W + (k % W);
#pragma unroll
    for (int i = 0; i < SplitCfg::kSlices; ++i) *reinterpret_cast<uint32_t *>(dst + i * plane) = packed[i];
  }
}

// ---- the contraction ----------------------------------------------------
template <int LAYOUT>
__global__ void __launch_bounds__(SplitCfg::kThreads, 1)
    syrk_split_kernel(const __grid_constant__ CUtensorMap map1, const double *__restrict__ scale, int64_t n, int64_t l, int k_blocks, uint64_t m_g,
                      TileOrder order, Epilogue ep, int dbg) {
  using C = SplitCfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t ring = (raw + 1023u) & ~1023u;  // 32-byte swizzle atoms: keep 1 KB alignment
  const uint32_t bars = ring + C::kStages * C::kStageBytes;
  // one "full" barrier per (stage, slice): the MMAs of a stage start on the
  // first slices while the later ones are still landing; one "empty" per stage
  auto full_bar = [&](int s, int sl) { return bars + 8u * (s * C::kSlices + sl); };
  auto empty_bar = [&](int s) { return bars + 8u * (C::kStages * C::kSlices + s); };
  const uint32_t tfull = bars + 8u * (C::kStages * C::kSlices + C::kStages);
  const uint32_t tempty = tfull + 8u;
  const uint32_t tmem_slot = tempty + 8u;
  uint32_t *tmem_slot_ptr =
      reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      for (int sl = 0; sl < C::kSlices; ++sl) mbar_init(full_bar(s, sl), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, C::kEpiWarps);
    mbar_fence_init();
    tma_prefetch_desc(&map1);
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  const uint64_t count = order.total;
  const double l_f = (double)l, sqrt_l = sqrt((double)l);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (uint64_t s = blockIdx.x; s < count; s += gridDim.x) {
      uint64_t Y, X;
      tile_at(order, m_g, s, Y, X);
      const bool drop = split_drop_top(scale, Y, X, lane, l_f, sqrt_l);  // whole warp
      if (lane == 0) {
        for (int pass = 0; pass < 2; ++pass) {
          // pass 0 reads all digit slices; pass 1 slices 0..3 (full depth) or 0..2 (adaptive)
          const int n_sl = pass == 0 ? C::kSlices : (drop ? 3 : 4);
          for (int kb = 0; kb < k_blocks; ++kb) {
            mbar_wait(empty_bar(stage), phase ^ 1);
            const uint32_t a = ring + stage * C::kStageBytes;
            for (int sl = 0; sl < n_sl; ++sl) {  // slice by slice, in the order the MMAs need them
              if (dbg == 1 || dbg == 3) {
                mbar_arrive(full_bar(stage, sl));
                continue;
              }
              // dbg 5 (timing experiment, wrong results): every other A slice is
              // not loaded -- the L2 traffic a 2-CTA multicast of A would save
              const bool skip_a = dbg == 5 && (sl & 1);
              mbar_arrive_expect_tx(full_bar(stage, sl), (skip_a ? 1u : 2u) * C::kSliceBytes);
              if (!skip_a)
                tma_load_3d(a + sl * C::kSliceBytes, &map1, 0, (int32_t)(Y * kTile), kb * C::kSlices + sl,
                            full_bar(stage, sl));
              tma_load_3d(a + C::kOpBytes + sl * C::kSliceBytes, &map1, 0, (int32_t)(X * kTile),
                          kb * C::kSlices + sl, full_bar(stage, sl));
            }
            // slices this pass does not load: their barriers still complete a
            // phase, so every slice barrier of a stage stays in step with the
            // stage's phase (a stage is reused by passes of 7 and of 3 / 4
            // slices; a barrier left a phase behind would let a later wait on
            // it return before its data lands)
            for (int sl = n_sl; sl < C::kSlices; ++sl) mbar_arrive(full_bar(stage, sl));
            if (++stage == C::kStages) stage = 0, phase ^= 1;
          }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int stage = 0;
    uint32_t phase = 0, use = 0;
    for (uint64_t s = blockIdx.x; s < count; s += gridDim.x) {
      uint64_t Y, X;
      tile_at(order, m_g, s, Y, X);
      const bool drop = split_drop_top(scale, Y, X, lane, l_f, sqrt_l);
      if (lane == 0) {
        for (int pass = 0; pass < 2; ++pass, ++use) {
          mbar_wait(tempty, (use & 1) ^ 1);  // the epilogue has drained the accumulators
          tc_fence_after();
          for (int kb = 0; kb < k_blocks; ++kb) {
            const uint32_t a = ring + stage * C::kStageBytes, b = a + C::kOpBytes;
            // the pass's MMA schedule (sched_entry), fully unrolled
            const bool first_k = kb == 0;
            if (dbg != 2 && dbg != 4) {
              if (pass == 0 && !drop)
                issue_stage<1>(tmem, a, b, first_k, full_bar(stage, 0), phase);
              else if (pass == 0)
                issue_stage<3>(tmem, a, b, first_k, full_bar(stage, 0), phase);
              else if (!drop)
                issue_stage<0>(tmem, a, b, first_k, full_bar(stage, 0), phase);
              else
                issue_stage<2>(tmem, a, b, first_k, full_bar(stage, 0), phase);
            } else {
              for (int sl = 0; sl < (pass == 1 ? (drop ? 3 : 4) : C::kSlices); ++sl)
                mbar_wait(full_bar(stage, sl), phase);
            }
            umma_commit(empty_bar(stage));  // the slot is free once these MMAs have read it
            if (++stage == C::kStages) stage = 0, phase ^= 1;
          }
          umma_commit(tfull);
        }
      } else {
        use += 2;
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    const int quad = warp & 3;             // TMEM lanes this warp may access
    const int half = (warp - 2) >> 2;      // column half of the tile
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    const uint64_t un = (uint64_t)n;
    uint32_t use = 0;
    for (uint64_t s = blockIdx.x; s < count; s += gridDim.x) {
      uint64_t Y, X;
      tile_at(order, m_g, s, Y, X);
      // pass 1's top accumulator: diagonal 3 (full depth) or 2 (adaptive);
      // pass 0 always fills all four (diagonals 4..7 or 3..6)
      const int top1 = split_drop_top(scale, Y, X, lane, l_f, sqrt_l) ? 2 : 3;
      double t[64];
#pragma unroll
      for (int pass = 0; pass < 2; ++pass, ++use) {
        mbar_wait(tfull, use & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4 && dbg < 3; ++c) {
#pragma unroll
          for (int q = 3; q >= 0; --q) {
            if (pass == 1 && q > top1) continue;
            int32_t v[16];
            tmem_ld16(tmem + lane_base + 128u * q + (uint32_t)(64 * half + 16 * c), v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              t[16 * c + j] = (pass == 0 && q == 3) ? (double)v[j] : fma(t[16 * c + j], 0.0078125, (double)v[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      const uint64_t y = Y * kTile + 32 * quad + lane;
      if (y < un && dbg < 3) {
        const double sy = scale[y];
        const uint64_t prb = (LAYOUT == kLayoutPacked) ? row_prefix(un, y) - y - ep.out_base : 0;
        const uint64_t x0 = X * kTile + 64 * half;
        if (LAYOUT == kLayoutPacked) {
          // the row's cells [max(x0, y), min(x0 + 64, n)) are contiguous in the
          // packed triangle: 16-byte stores (two cells per request) on the
          // aligned pairs, single cells at the ends
          const uint64_t xa = x0 > y ? x0 : y, xb = x0 + 64 < un ? x0 + 64 : un;
          if (xa < xb) {
            const int ja = (int)(xa - x0), jb = (int)(xb - x0);
            double *row = ep.out + prb + x0;
            auto cell = [&](int j) { return t[j] * sy * __ldg(scale + x0 + j); };
            auto one = [&](int j) {
              if (j >= ja && j < jb) __stcs(row + j, cell(j));
            };
            auto pair = [&](int j) {
              if (j >= ja && j + 1 < jb) {
                __stcs(reinterpret_cast<double2 *>(row + j), make_double2(cell(j), cell(j + 1)));
              } else {
                one(j);
                one(j + 1);
              }
            };
            if (((prb + x0) & 1) == 0) {
#pragma unroll
              for (int j = 0; j < 64; j += 2) pair(j);
            } else {
              one(0);
#pragma unroll
              for (int j = 1; j < 63; j += 2) pair(j);
              one(63);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const uint64_t x = x0 + j;
            if (x >= y && x < un) store_cell<LAYOUT>(ep, y, x, prb, t[j] * sy * __ldg(scale + x));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

}  // namespace pcc
