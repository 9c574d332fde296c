// exact.cuh -- K2x: the contraction in the reference's own arithmetic, bit for
// bit.  Every coefficient is _kernels.dot8(u[y], u[x]) (_kernels.py:30-68):
// eight lane sums, lane j adding RN(u[y][k] * u[x][k]) for k = j (mod 8) in
// increasing k (separate multiply and add -- no FMA), then the fixed tree
// ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)).  It runs on the FP64 CUDA cores
// (DMUL + DADD: two FP64 operations per term, vs one DMMA FMA lane-op on the
// tensor path), so it is the bit-exact mode, not the fast one.
//
// Work unit = one 32 x 64 sub-block of a 128 x 128 GPU tile (8 per tile,
// persistent grid-stride over the range's tiles in the grouped order x 8).  512 threads (16
// warps: the multiply -> add dependency needs them to fill the FP64 pipe):
// thread t is reference lane j = t & 7 for a 4 x 8 cell block, so each
// thread carries 32 independent lane accumulators and the 8 lanes of a cell
// sit in 8 consecutive threads.  U's rows stream through a 2-stage cp.async ring of 128-column
// K chunks (pitch 136 doubles; rows of odd 8-row blocks shifted by 8 doubles,
// so the four 8-lane groups of a warp reading four different row blocks
// pair up on opposite bank halves: the minimum two wavefronts per 64-bit
// load).  Zero K padding only adds +0.0 to lane sums
// that can never be -0.0, so the padded length changes no bit.  The tree is
// three xor-shuffles (1, 2, 4), which pair the lanes exactly as the tree.
#pragma once

#include "syrk.cuh"

namespace pcc {

struct ExactCfg {
  static constexpr int RT = 4;        // cell rows per thread (x 8 columns)
  static constexpr int kThreads = 256 * 8 / RT;
  static constexpr int BM = 32;      // sub-block rows (y)
  static constexpr int BN = 64;      // sub-block columns (x)
  static constexpr int BK = 128;          // K chunk (16 steps of each lane)
  static constexpr int kPitch = BK + 8;   // doubles per staged row
  static constexpr int STAGES = 2;
  static constexpr int kStageDoubles = (BM + BN) * kPitch;
  static constexpr int kRingBytes = STAGES * kStageDoubles * (int)sizeof(double);
  static constexpr int kSmemBytes = kRingBytes + 8 * STAGES;  // + one mbarrier per stage (bulk copies)
  static constexpr int kSubPerTile = (kTile / BM) * (kTile / BN);  // 8
};

// Staged row r of a chunk (0..BM-1: A rows, BM..: B rows) starts here.
__device__ __forceinline__ int row_off(int r) { return r * ExactCfg::kPitch + ((r >> 3) & 1) * 8; }

__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// BULK (production): each staged row arrives by one 1-D bulk copy
// (cp.async.bulk, issued by one thread per row, completion counted in bytes
// on the stage's mbarrier, thread 0 waits and one CTA barrier per chunk
// publishes it) instead of 16-byte cp.async pieces issued by every thread:
// c2 82.4 -> 74.3 ms (80 % of the FP64 ALU peak).
template <int LAYOUT, bool BULK = true>
__global__ void __launch_bounds__(ExactCfg::kThreads, 1)
syrk_exact_kernel(const double *__restrict__ u, int64_t n, int64_t ldu, int k_chunks, uint64_t m_g,
                  TileOrder order, Epilogue ep) {
  using C = ExactCfg;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x;
  const int lane8 = tid & 7;
  const int grp = tid >> 3;         // which RT x 8 cell block
  const int bi = grp >> 3;          // rows bi*RT .. +RT of the sub-block
  const int bj = grp & 7;           // cols bj*8 .. +8
  const uint64_t un = (uint64_t)n;
  const uint64_t units = order.total * C::kSubPerTile;
  const uint32_t full0 = smem_u32(smem) + C::kRingBytes;  // BULK: one mbarrier per stage after the ring
  uint32_t chunk_seq = 0;                                  // chunks consumed by this CTA (barrier phases)
  if (BULK) {
    if (tid == 0) {
      for (int st = 0; st < C::STAGES; ++st) mbar_init(full0 + 8 * st, 1);
      mbar_fence_init();
    }
    __syncthreads();
  }

  for (uint64_t w = blockIdx.x; w < units; w += gridDim.x) {
    // tiles in the grouped L2-locality order (as the tensor path), the 8
    // sub-blocks of a tile on consecutive units
    const int sub = (int)(w % C::kSubPerTile);
    uint64_t Y, X;
    tile_at(order, m_g, w / C::kSubPerTile, Y, X);
    const uint64_t row0 = Y * kTile + (uint64_t)(sub >> 1) * C::BM;
    const uint64_t col0 = X * kTile + (uint64_t)(sub & 1) * C::BN;
    // nothing of the triangle / of [0, n) in this sub-block: skip it
    if (row0 >= un || col0 >= un || col0 + C::BN - 1 < row0) continue;

    auto load_chunk = [&](int stage, int kc) {
      double *sa = smem + stage * C::kStageDoubles;
      const int64_t k0 = (int64_t)kc * C::BK;
      if (BULK) {
        const int cols = (int)((ldu - k0) < C::BK ? (ldu - k0) : C::BK);  // multiple of 32
        if (tid == 0) mbar_arrive_expect_tx(full0 + 8 * stage, (uint32_t)((C::BM + C::BN) * cols * 8));
        if (tid < C::BM + C::BN) {
          const uint64_t grow = tid < C::BM ? row0 + tid : col0 + (tid - C::BM);
          bulk_copy_g2s(smem_u32(sa + row_off(tid)), u + grow * (uint64_t)ldu + k0, (uint32_t)(cols * 8),
                        full0 + 8 * stage);
        }
        return;
      }
      // (BM + BN) rows x 32 doubles = 8 x 16-byte pieces per row
      for (int i = tid; i < (C::BM + C::BN) * (C::BK / 2); i += C::kThreads) {
        const int r = i / (C::BK / 2), piece = i % (C::BK / 2);
        const uint64_t grow = r < C::BM ? row0 + r : col0 + (r - C::BM);
        double *dst = sa + row_off(r) + piece * 2;
        if (k0 + piece * 2 < ldu) {
#ifndef PCC_EXACT_NOLOAD  // tools/exact_bench.cu: math-only timing (stale operands)
          cp_async_16(smem_u32(dst), u + grow * (uint64_t)ldu + k0 + piece * 2);
#endif
        } else {  // past the row's padded width (ldu is a multiple of 32, BK of 64): zeros
          *reinterpret_cast<double2 *>(dst) = make_double2(0.0, 0.0);
        }
      }
    };

    double acc[C::RT][8];
#pragma unroll
    for (int i = 0; i < C::RT; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;

    const uint32_t seq0 = chunk_seq;  // BULK: stage of chunk kc = (seq0 + kc) % STAGES
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; ++s) {
      if (s < k_chunks) load_chunk(BULK ? (seq0 + s) % C::STAGES : s, s);
      if (!BULK) cp_async_commit();
    }
    for (int kc = 0; kc < k_chunks; ++kc) {
      const int cur = BULK ? (int)((seq0 + kc) % C::STAGES) : kc % C::STAGES;
      if (BULK) {
        if (tid == 0) mbar_wait(full0 + 8 * cur, ((seq0 + kc) / C::STAGES) & 1);
      } else {
        cp_async_wait<C::STAGES - 2>();
      }
      __syncthreads();
      {
        const int nxt = kc + C::STAGES - 1;
        if (nxt < k_chunks) load_chunk(BULK ? (int)((seq0 + nxt) % C::STAGES) : nxt % C::STAGES, nxt);
        if (!BULK) cp_async_commit();
      }
      const int msteps = BULK ? (int)((ldu - (int64_t)kc * C::BK) < C::BK ? (ldu - (int64_t)kc * C::BK) : C::BK) / 8
                              : C::BK / 8;
      const double *sa = smem + cur * C::kStageDoubles + row_off(bi * C::RT) + lane8;
      const double *sb = smem + cur * C::kStageDoubles + row_off(C::BM + bj * 8) + lane8;
#pragma unroll
      for (int m = 0; m < C::BK / 8; ++m) {  // this lane's k = kc*BK + m*8 + lane8, increasing
        if (BULK && m >= msteps) break;       // (a short chunk only at the padded end of the row)
        double a[C::RT], b[8];
#pragma unroll
        for (int i = 0; i < C::RT; ++i) a[i] = sa[i * C::kPitch + m * 8];
#pragma unroll
        for (int c = 0; c < 8; ++c) b[c] = sb[c * C::kPitch + m * 8];
#pragma unroll
        for (int i = 0; i < C::RT; ++i) {
          // all eight products of the row first: each add waits on a
          // multiply issued eight FP64 instructions earlier
          double p[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) p[c] = __dmul_rn(a[i], b[c]);
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[i][c] = __dadd_rn(acc[i][c], p[c]);
        }
      }
    }
    if (!BULK) cp_async_wait<0>();
    chunk_seq += (uint32_t)k_chunks;
    __syncthreads();  // the ring is reloaded by the next unit

    // the fixed tree across the 8 lanes of each cell, then lane j stores
    // column j of the thread group's 8 x 8 block (8 consecutive cells per row)
#pragma unroll
    for (int i = 0; i < C::RT; ++i) {
      double mine = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double v = acc[i][c];
        v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1));
        v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 2));
        v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 4));
        if (c == lane8) mine = v;
      }
      const uint64_t y = row0 + bi * C::RT + i;
      const uint64_t x = col0 + bj * 8 + lane8;
      if (y < un && x >= y && x < un) {
        const uint64_t prb = (LAYOUT == kLayoutPacked) ? row_prefix(un, y) - y - ep.out_base : 0;
        store_cell<LAYOUT>(ep, y, x, prb, mine);
      }
    }
  }
}

}  // namespace pcc
