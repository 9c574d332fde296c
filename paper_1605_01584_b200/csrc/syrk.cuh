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
// K is staged 16 doubles at a time through a 4-deep cp.async ring (32 KB
// per stage, 128 KB total), stored as 8-double "slabs": smem[slab][row][8].
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

constexpr int kTile = 128;
constexpr int kBK = 16;
constexpr int kStages = 4;
constexpr int kSyrkThreads = 256;
constexpr int kSlab = 8;
constexpr int kSlabsPerStage = kBK / kSlab;
constexpr int kOperandDoubles = kSlabsPerStage * kTile * kSlab;  // 2048
constexpr int kStageDoubles = 2 * kOperandDoubles;                // A + B
constexpr int kSyrkSmemBytes = kStages * kStageDoubles * (int)sizeof(double);

enum : int { kLayoutPacked = 0, kLayoutDense = 1, kLayoutTiles = 2 };

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
__device__ __forceinline__ void store_cell(const Epilogue &ep, uint64_t n, uint64_t y, uint64_t x,
                                           uint64_t packed_row_base, double v) {
  if (LAYOUT == kLayoutPacked) {
    ep.out[packed_row_base + x] = v;
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

template <int LAYOUT>
__global__ void __launch_bounds__(kSyrkThreads, 1)
syrk_kernel(const double *__restrict__ u, int64_t n, int64_t ldu, int k_tiles, uint64_t m_g,
            uint64_t tile_begin, uint64_t tile_end, Epilogue ep) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t smem_base = smem_u32(smem);

  // Copy assignment: 2 x 1024 16-byte chunks per stage; thread tid owns
  // chunk q = tid % 8 of rows tid/8 + 32 i (i < 4) for both operands.
  const int cq = tid & 7;
  const int crow = tid >> 3;
  const uint32_t copy_soff =
      (uint32_t)(((cq >> 2) * kTile * kSlab + crow * kSlab + (cq & 3) * 2) * sizeof(double));

  for (uint64_t J = tile_begin + blockIdx.x; J < tile_end; J += gridDim.x) {
    const uint64_t Y = tile_row(m_g, J);
    const uint64_t X = J + Y - row_prefix(m_g, Y);
    const double *ga = u + (int64_t)(Y * kTile + crow) * ldu + cq * 2;
    const double *gb = u + (int64_t)(X * kTile + crow) * ldu + cq * 2;

    auto load_stage = [&](int slot, int kt) {
      const uint32_t s = smem_base + (uint32_t)(slot * kStageDoubles * sizeof(double)) + copy_soff;
      const int64_t k0 = (int64_t)kt * kBK;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t roff = (int64_t)(32 * i) * ldu + k0;
        cp_async_16(s + (uint32_t)(32 * i * kSlab * sizeof(double)), ga + roff);
        cp_async_16(s + (uint32_t)((kOperandDoubles + 32 * i * kSlab) * sizeof(double)), gb + roff);
      }
    };

    double acc[8][4][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < k_tiles) load_stage(s, s);
      cp_async_commit();
    }

    for (int kt = 0; kt < k_tiles; ++kt) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      const int nk = kt + kStages - 1;
      if (nk < k_tiles) load_stage(nk % kStages, nk);
      cp_async_commit();

      const double *sA = smem + (kt % kStages) * kStageDoubles;
      const double *sB = sA + kOperandDoubles;
#pragma unroll
      for (int slab = 0; slab < kSlabsPerStage; ++slab) {
        double2 a[8], b[4];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
          a[mi] = *reinterpret_cast<const double2 *>(sA + slab * kTile * kSlab +
                                                     (wm * 64 + mi * 8 + g) * kSlab + tig * 2);
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
          b[ni] = *reinterpret_cast<const double2 *>(sB + slab * kTile * kSlab +
                                                     (wn * 32 + ni * 8 + g) * kSlab + tig * 2);
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, b[ni].x);
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, b[ni].y);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // ring slots are rewritten by the next tile's prologue

    // Fused epilogue: cells y <= x < n straight from the accumulators.
    const uint64_t un = (uint64_t)n;
    const uint64_t y0 = Y * kTile + wm * 64 + g;
    const uint64_t x0 = X * kTile + wn * 32 + 2 * tig;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const uint64_t y = y0 + mi * 8;
      if (y >= un) continue;
      const uint64_t prb = (LAYOUT == kLayoutPacked) ? row_prefix(un, y) - y - ep.out_base : 0;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint64_t x = x0 + ni * 8 + e;
          if (x >= y && x < un) store_cell<LAYOUT>(ep, un, y, x, prb, acc[mi][ni][e]);
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
