// TMA tensor-copy throughput per issuing thread: L issuing lanes of one warp
// per CTA (one CTA per SM), each streaming its own part of a large FP64
// matrix through a private ring of S slots of one box {BW doubles, BR rows}
// (2-D tiled tensor map, mbarrier complete_tx), consumer = the same lane
// (wait, then re-issue).  Prints B/clk/SM and GB/s for box shapes and lane
// counts -- the supply model of the streamed K1 (csrc/normalize_stream.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/tma_issue_bw tools/tma_issue_bw.cu
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1605_01584_b200/csrc/common.cuh"

using namespace pcc;

__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap *map, int32_t c0, int32_t c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__global__ void bw(const __grid_constant__ CUtensorMap map, int lanes, int slots, int bw_, int br, int64_t rows,
                   int64_t cols, int iters, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  __shared__ __align__(8) uint64_t bars[32 * 8];
  const int lane = threadIdx.x;
  const int box_bytes = bw_ * br * 8;
  if (lane < lanes)
    for (int s = 0; s < slots; ++s) mbar_init(smem_u32(&bars[lane * 8 + s]), 1);
  mbar_fence_init();
  __syncwarp();
  const long long t0 = clock64();
  if (lane < lanes) {
    // lane's tiles: column blocks of bw_, row blocks of br, strided over CTAs and lanes
    const int64_t tiles_c = cols / bw_, tiles = (rows / br) * tiles_c;
    int64_t t = (int64_t)blockIdx.x * lanes + lane;
    const int64_t tstep = (int64_t)gridDim.x * lanes;
    for (int i = 0; i < iters; ++i) {
      const int s = i % slots;
      const uint32_t bar = smem_u32(&bars[lane * 8 + s]);
      if (i >= slots) mbar_wait(bar, ((i / slots) - 1) & 1);
      const int64_t tt = t % tiles;
      mbar_arrive_expect_tx(bar, (uint32_t)box_bytes);
      tma2d(base + (uint32_t)((lane * slots + s) * box_bytes), &map, (int32_t)((tt % tiles_c) * bw_),
            (int32_t)((tt / tiles_c) * br), bar);
      t += tstep;
    }
    for (int i = iters; i < iters + slots; ++i) {
      const int s = i % slots;
      if (i >= slots) mbar_wait(smem_u32(&bars[lane * 8 + s]), ((i / slots) - 1) & 1);
    }
  }
  __syncwarp();
  if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t rows = 32768, cols = 8192;  // 2 GB of FP64 (larger than L2)
  double *x;
  cudaMalloc(&x, rows * cols * 8);
  cudaMemset(x, 0, rows * cols * 8);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  long long *cyc;
  cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Shape { int bw, br; } shapes[] = {{256, 1}, {256, 4}, {256, 8}, {128, 8}, {64, 32}};
  for (auto sh : shapes) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
    const cuuint32_t box[2] = {(cuuint32_t)sh.bw, (cuuint32_t)sh.br}, estr[2] = {1, 1};
    reinterpret_cast<EncodeTiledFn>(p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int box_bytes = sh.bw * sh.br * 8;
    for (int lanes : {1, 2, 4, 8, 16}) {
      int slots = (160 * 1024) / (lanes * box_bytes);
      if (slots > 8) slots = 8;
      if (slots < 2) continue;
      const int iters = (int)((int64_t)256 * 1024 * 1024 / 148 / lanes / box_bytes);  // ~256 MB per launch
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      bw<<<148, 32, 200 * 1024>>>(m, lanes, slots, sh.bw, sh.br, rows, cols, iters, cyc);
      cudaEventRecord(a);
      bw<<<148, 32, 200 * 1024>>>(m, lanes, slots, sh.bw, sh.br, rows, cols, iters, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      long long c0;
      cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)iters * lanes * box_bytes;
      printf("box {%3d doubles, %2d rows} = %5d B, %2d lanes x %d slots: %7.1f B/clk/SM  %6.0f GB/s  (%s)\n", sh.bw,
             sh.br, box_bytes, lanes, slots, bytes / c0, bytes * 148 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
