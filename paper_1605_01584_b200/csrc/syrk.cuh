// syrk.cuh -- K2: symmetric upper-triangular tiled U.U^T contraction in FP64
// on the B200 tensor pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), with the
// reference's output layouts written by a fused epilogue.
//
// Replaces _kernels.compute_tile_range + dot8 + scatter_range
// (_kernels.py:30-68, 322-373) and the tile walk of the paper's Alg. 1
// (PAPER.md:193-233): a persistent grid walks GPU tile ids
// J = tile_begin + blockIdx.x, J += gridDim.x (Alg. 1's J_t += numGroups),
// each J decoded to its (Y, X) tile coordinate by the job-id <-> coordinate
// bijection (tile_row, common.cuh).
//
// Tile: 128 x 128 cells per CTA, 8 warps in a 2 x 4 grid, each warp owns a
// 64 x 32 sub-tile = 8 x 4 DMMA 8x8 accumulators (64 doubles per thread).
// K is staged 16 doubles at a time through a 6-deep TMA ring (32 KB per
// stage), stored as 8-double "slabs": smem[slab][row][8].
// Fragment loads are one 16-byte LDS per thread per 8x8 operand tile; a
// quarter-warp (the LDS.128 phase) touches rows r, r+1 x 4 chunks = 128
// distinct bytes, so the layout is bank-conflict free without padding.
//
// K permutation: within each slab thread `tig` feeds k = 2*tig to the first
// DMMA and k = 2*tig+1 to the second.  A and B use the same map, so the
// contraction is the same sum in a fixed order that depends only on the
// kernel -- every cell is bitwise identical whatever the tile range, grid
// size or device count (the reference's schedule-invariance guarantee,
// engine.py:32-37).
//
// Bound: FP64 compute (arithmetic intensity 83-1365 flop/B at every config,
// SURVEY.md §8d).  Per tile: 2 * 128 * 128 * K flop on 2 * 128 * K * 8 B of
// operand traffic (L2-resident A band shared by concurrent CTAs).
#pragma once

#include "common.cuh"

namespace pcc {

constexpr int kTile = 128;  // GPU tile edge (PCC_GPU_TILE)
constexpr int kSlab = 8;    // doubles per smem row-slab (one DMMA k8 pair)

enum : int { kLayoutPacked = 0, kLayoutDense = 1, kLayoutTiles = 2 };

// Kernel shape: WARPS_M x WARPS_N warps, each owning MI x NI DMMA 8x8
// accumulators (CTA tile kEdge x kEdge: the 128 x 128 GPU tile, or one 64 x 64
// quadrant of it for the tail kernel), K staged BK doubles per stage
// through a STAGES-deep ring.
template <int WARPS_M_, int WARPS_N_, int MI_, int NI_, int BK_, int STAGES_, int AHEAD_ = STAGES_ / 2>
struct SyrkCfg {
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, MI = MI_, NI = NI_, BK = BK_, STAGES = STAGES_;
  static constexpr int AHEAD = AHEAD_;  // TMA producer lead (K steps) over warp 0
  static constexpr int kThreads = 32 * WARPS_M * WARPS_N;
  static constexpr int kEdge = WARPS_M * MI * 8;  // CTA tile edge (rows == cols)
  static constexpr int kSlabs = BK / kSlab;
  static constexpr int kOpDoubles = kSlabs * kEdge * kSlab;
  static constexpr int kStageDoubles = 2 * kOpDoubles;
  static constexpr int kSmemBytes = STAGES * kStageDoubles * (int)sizeof(double);
  static constexpr int kChunksPerRow = BK / 2;                 // 16-byte chunks
  static constexpr int kRowsPerPass = kThreads / kChunksPerRow;
  static constexpr int kPasses = kEdge / kRowsPerPass;
  static_assert(kEdge == WARPS_N * NI * 8 && (kEdge == kTile || 2 * kEdge == kTile), "CTA tile: 128^2 or a 64^2 quadrant");
  static_assert(BK % kSlab == 0 && kThreads % kChunksPerRow == 0 && kEdge % kRowsPerPass == 0, "bad shape");
};

struct Epilogue {
  double *out;
  int64_t ld_out;      // dense row stride
  uint64_t out_base;   // packed: index of out[0] in the full triangle
  int64_t ref_t;       // tiles: reference tile edge t
  uint64_t ref_m;      // tiles: ceil(n / t)
  uint64_t ref_begin;  // tiles: [ref_begin, ref_end) reference tile ids
  uint64_t ref_end;
};

template <int LAYOUT>
__device__ __forceinline__ void store_cell(const Epilogue &ep, uint64_t y, uint64_t x, uint64_t packed_row_base,
                                           double v) {
  if (LAYOUT == kLayoutPacked) {
    __stcs(ep.out + packed_row_base + x, v);  // streaming: the result is never re-read here, keep L2 for U
  } else if (LAYOUT == kLayoutDense) {
    ep.out[y * (uint64_t)ep.ld_out + x] = v;
    if (x != y) ep.out[x * (uint64_t)ep.ld_out + y] = v;
  } else {
    const uint64_t t = (uint64_t)ep.ref_t;
    const uint64_t yt = y / t, xt = x / t;
    const uint64_t jr = row_prefix(ep.ref_m, yt) + xt - yt;
    if (jr >= ep.ref_begin && jr < ep.ref_end)
      ep.out[(jr - ep.ref_begin) * t * t + (y - yt * t) * t + (x - xt * t)] = v;
  }
}

// ---------------------------------------------------------------------------
// TMA + mbarrier variant (production).  GROUPED = true (production) visits
// the range in the L2-locality TileOrder (common.cuh): same time as the
// plain id order, 3.5x less DRAM traffic.  U's row bands stream into a STAGES-deep shared
// ring with TMA (cp.async.bulk.tensor.2d: one 8-double x 128-row box per
// operand slab, completion counted in bytes on the slot's "full" mbarrier).
// Thread 0 doubles as the producer: before each K step it tops the ring up
// to kAhead steps in front of its own warp (blocking only when the ring is
// empty), following the CTA's tile sequence across tile boundaries, so the
// next tile's first stages land while the epilogue runs.  Every warp waits
// on "full", runs its DMMA slab(s) and releases the slot with one arrive on
// the slot's "empty" mbarrier.  There is no block-wide barrier in the K
// loop; warps drift within the ring's slack.
template <class C>
struct TmaLayout {
  static constexpr int kBarOffset = C::kSmemBytes;  // 2 * STAGES mbarriers after the ring
  static constexpr int kSmemBytes = C::kSmemBytes + 2 * C::STAGES * 8;
  static constexpr int kThreads = C::kThreads;
  static constexpr int kAhead = C::AHEAD;
  static constexpr uint32_t kStageBytes = (uint32_t)(C::kStageDoubles * sizeof(double));
  static constexpr uint32_t kSlabBytes = (uint32_t)(C::kEdge * kSlab * sizeof(double));
};

// Schedule slot s -> tile (Y, X): the grouped L2-locality order
// (production: a wave of ~148 tiles spans ~12 row bands x ~12 column bands,
// so each K slice of a band is fetched from DRAM about once per wave; c2:
// 20.3 -> 5.8 GB DRAM reads per launch) or plain bijection id order.
template <bool GROUPED>
__device__ __forceinline__ void slot_tile(const TileOrder &o, uint64_t m, uint64_t s, uint64_t &Y, uint64_t &X) {
  if (GROUPED) {
    tile_at(o, m, s, Y, X);
  } else {
    const uint64_t J = o.tb + s;
    Y = tile_row(m, J);
    X = J + Y - row_prefix(m, Y);
  }
}

// Schedule slot -> origin (row0, col0) of the CTA tile.  Quadrant mode (the
// tail kernel, 64 x 64 CTA tiles): slot s is quadrant s % 4 of GPU tile
// order.tb + s / 4 -- the same cells, the same per-cell K order, four CTAs.
template <class C, bool GROUPED>
__device__ __forceinline__ void slot_origin(const TileOrder &o, uint64_t m, uint64_t s, uint64_t &row0,
                                            uint64_t &col0) {
  uint64_t Y, X;
  if (C::kEdge == kTile) {
    slot_tile<GROUPED>(o, m, s, Y, X);
    row0 = Y * kTile;
    col0 = X * kTile;
  } else {
    slot_tile<false>(o, m, s >> 2, Y, X);
    row0 = Y * kTile + ((s >> 1) & 1) * C::kEdge;
    col0 = X * kTile + (s & 1) * C::kEdge;
  }
}

template <class C, int LAYOUT, bool GROUPED = false, bool SKEW = false, bool STAGE_FRAGS = (C::kSlabs <= 2)>
__global__ void __launch_bounds__(C::kThreads, 1)
syrk_tma_kernel(const __grid_constant__ CUtensorMap umap, int64_t n, int k_tiles, uint64_t m_g, TileOrder order,
                Epilogue ep) {
  using TL = TmaLayout<C>;
  extern __shared__ __align__(1024) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t full0 = smem_base + TL::kBarOffset;
  const uint32_t empty0 = full0 + C::STAGES * 8;
  constexpr int kWarps = C::WARPS_M * C::WARPS_N;

  if (tid == 0) {
    tma_prefetch_desc(&umap);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, kWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // Producer cursor (meaningful in thread 0 only): next K step to load.
  const uint64_t first = blockIdx.x;
  const uint64_t my_tiles = first < order.total ? (order.total - first + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t total_steps = my_tiles * (uint64_t)k_tiles;
  uint64_t p_step = 0;
  int p_kt = 0, p_stage = 0;
  uint32_t p_phase = 0;
  uint64_t p_s = first;
  int32_t p_ya = 0, p_xb = 0;
  if (tid == 0 && my_tiles) {
    uint64_t r0, c0;
    slot_origin<C, GROUPED>(order, m_g, p_s, r0, c0);
    p_ya = (int32_t)r0;
    p_xb = (int32_t)c0;
  }
  // Issue loads while the cursor is less than `want` steps ahead; block on a
  // busy slot only if the consumer would otherwise find the ring empty.
  auto produce = [&](uint64_t c_step) {
    while (p_step < total_steps && p_step < c_step + TL::kAhead) {
      const uint32_t empty = empty0 + 8 * p_stage;
      if (p_step > c_step) {
        if (!mbar_try_wait(empty, p_phase ^ 1)) break;
      } else {
        mbar_wait(empty, p_phase ^ 1);
      }
      const uint32_t full = full0 + 8 * p_stage;
      mbar_arrive_expect_tx(full, TL::kStageBytes);
      const uint32_t dst = smem_base + (uint32_t)p_stage * TL::kStageBytes;
#pragma unroll
      for (int slab = 0; slab < C::kSlabs; ++slab) {
        const int32_t k0 = p_kt * C::BK + slab * kSlab;
        tma_load_2d(dst + slab * TL::kSlabBytes, &umap, k0, p_ya, full);
        tma_load_2d(dst + (uint32_t)(C::kOpDoubles * sizeof(double)) + slab * TL::kSlabBytes, &umap, k0, p_xb, full);
      }
      ++p_step;
      if (++p_stage == C::STAGES) {
        p_stage = 0;
        p_phase ^= 1;
      }
      if (++p_kt == k_tiles && p_step < total_steps) {
        p_kt = 0;
        p_s += gridDim.x;
        uint64_t r0, c0;
        slot_origin<C, GROUPED>(order, m_g, p_s, r0, c0);
        p_ya = (int32_t)r0;
        p_xb = (int32_t)c0;
      }
    }
  };

  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, tig = lane & 3;
  uint64_t c_step = 0;
  int stage = 0;
  uint32_t phase = 0;
  for (uint64_t si = first; si < order.total; si += gridDim.x) {
    uint64_t row0, col0;
    slot_origin<C, GROUPED>(order, m_g, si, row0, col0);

    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < C::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    // One 8-deep K slab of stage `st`: 12 fragment loads, 64 DMMAs.
    auto slab_mma = [&](int st, int slab) {
      const double *sA =
          smem + st * C::kStageDoubles + (wm * C::MI * 8 + g) * kSlab + tig * 2 + slab * C::kEdge * kSlab;
      const double *sB = smem + st * C::kStageDoubles + C::kOpDoubles + (wn * C::NI * 8 + g) * kSlab + tig * 2 +
                         slab * C::kEdge * kSlab;
      double2 a[C::MI], b[C::NI];
#pragma unroll
      for (int mi = 0; mi < C::MI; ++mi) a[mi] = *reinterpret_cast<const double2 *>(sA + mi * 8 * kSlab);
#pragma unroll
      for (int ni = 0; ni < C::NI; ++ni) b[ni] = *reinterpret_cast<const double2 *>(sB + ni * 8 * kSlab);
#pragma unroll
      for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, b[ni].x);
#pragma unroll
      for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, b[ni].y);
    };
    auto advance = [](int &st, uint32_t &ph) {
      if (++st == C::STAGES) {
        st = 0;
        ph ^= 1;
      }
    };

    if (SKEW && wm == 1) {
      // Half-stage skew: these warps share SMSPs with warps wm == 0 (warp w and
      // w + 4) and run their stage waits and fragment loads between the other
      // warps' slab boundaries, so the two warps never stall together.  Each
      // accumulator still sees slab 0 then slab 1 of every stage, in order.
      static_assert(!SKEW || C::kSlabs == 2, "skew needs two slabs per stage");
      mbar_wait(full0 + 8 * stage, phase);
      slab_mma(stage, 0);
      for (int kt = 0; kt < k_tiles; ++kt) {
        const int cur = stage;
        advance(stage, phase);
        if (kt + 1 < k_tiles) mbar_wait(full0 + 8 * stage, phase);
        slab_mma(cur, 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * cur);
        if (kt + 1 < k_tiles) slab_mma(stage, 0);
      }
      c_step += k_tiles;
    } else if (STAGE_FRAGS) {
      // Production: all fragments of a stage are loaded before its DMMAs
      // (253 registers, no spills), so the second slab's loads overlap the
      // first slab's math and every accumulator's next DMMA is 32 DMMAs
      // away (measured 94.3 -> 97.1 % of the FP64 peak on c2).
      for (int kt = 0; kt < k_tiles; ++kt, ++c_step) {
        if (tid == 0) produce(c_step);
        mbar_wait(full0 + 8 * stage, phase);
        const double *sA = smem + stage * C::kStageDoubles + (wm * C::MI * 8 + g) * kSlab + tig * 2;
        const double *sB = smem + stage * C::kStageDoubles + C::kOpDoubles + (wn * C::NI * 8 + g) * kSlab + tig * 2;
        double2 a[C::kSlabs][C::MI], b[C::kSlabs][C::NI];
#pragma unroll
        for (int slab = 0; slab < C::kSlabs; ++slab) {
#pragma unroll
          for (int mi = 0; mi < C::MI; ++mi)
            a[slab][mi] = *reinterpret_cast<const double2 *>(sA + slab * C::kEdge * kSlab + mi * 8 * kSlab);
#pragma unroll
          for (int ni = 0; ni < C::NI; ++ni)
            b[slab][ni] = *reinterpret_cast<const double2 *>(sB + slab * C::kEdge * kSlab + ni * 8 * kSlab);
        }
#pragma unroll
        for (int slab = 0; slab < C::kSlabs; ++slab) {
#pragma unroll
          for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < C::NI; ++ni)
              dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[slab][mi].x, b[slab][ni].x);
#pragma unroll
          for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < C::NI; ++ni)
              dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[slab][mi].y, b[slab][ni].y);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * stage);
        advance(stage, phase);
      }
    } else {
      for (int kt = 0; kt < k_tiles; ++kt, ++c_step) {
        if (tid == 0) produce(c_step);
        mbar_wait(full0 + 8 * stage, phase);
#pragma unroll
        for (int slab = 0; slab < C::kSlabs; ++slab) slab_mma(stage, slab);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * stage);
        advance(stage, phase);
      }
    }

    const uint64_t un = (uint64_t)n;
    const uint64_t y0 = row0 + wm * C::MI * 8 + g;
    const uint64_t x0 = col0 + wn * C::NI * 8 + 2 * tig;
#pragma unroll
    for (int mi = 0; mi < C::MI; ++mi) {
      const uint64_t y = y0 + mi * 8;
      if (y >= un) continue;
      const uint64_t prb = (LAYOUT == kLayoutPacked) ? row_prefix(un, y) - y - ep.out_base : 0;
#pragma unroll
      for (int ni = 0; ni < C::NI; ++ni) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint64_t x = x0 + ni * 8 + e;
          if (x >= y && x < un) store_cell<LAYOUT>(ep, y, x, prb, acc[mi][ni][e]);
        }
      }
    }
  }
}

// Device-side scatter_range (_kernels.py:322-348): cells y <= x < n of
// `count` consecutive reference t x t tiles from a flat pass buffer into the
// packed triangle.  One thread per cell, grid-stride.
__global__ void scatter_range_kernel(double *__restrict__ packed, const double *__restrict__ values,
                                     uint64_t first_tile, uint64_t count, int64_t t, int64_t n,
                                     uint64_t m) {
  const uint64_t t2 = (uint64_t)t * (uint64_t)t;
  const uint64_t cells = count * t2;
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cells;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = c / t2, w = c - k * t2;
    const uint64_t ry = w / (uint64_t)t, cx = w - ry * (uint64_t)t;
    const uint64_t jt = first_tile + k;
    const uint64_t yt = tile_row(m, jt);
    const uint64_t xt = jt + yt - row_prefix(m, yt);
    const uint64_t y = yt * t + ry, x = xt * t + cx;
    if (y <= x && x < (uint64_t)n) packed[row_prefix((uint64_t)n, y) - y + x] = values[c];
  }
}

// FP64 tensor-pipe probe: register-resident DMMA chains (no memory traffic),
// for the live roofline denominator.
__global__ void dmma_probe_kernel(double *out, int iters) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace pcc
