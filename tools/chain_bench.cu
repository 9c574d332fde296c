// Cycles per step of the K1 lane chains (stream_chain) out of shared memory,
// one warp per SM: ROWS rows x 8 lanes, windows of 512 doubles per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/chain_bench tools/chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "experiments/normalize_stream.cuh"

template <bool SSD, int ROWS, int STRIDE>
__global__ void bench(double *out, int windows, long long *cyc, int nst_rt) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x, r = lane >> 3, j = lane & 7;
  for (int i = lane; i < 4 * STRIDE; i += 32) sm[i] = 1.0 + 1e-3 * (i % 97);
  __syncwarp();
  double s = 0.0, dmax = 0.0;
  bool varies = false;
  const long long t0 = clock64();
  if (r < ROWS)
    for (int w = 0; w < windows; ++w) {
      const double *p = sm + r * STRIDE + (w & 1) * 8 * 64;
      pcc::stream_chain<SSD, false, 8>(s, p + j, nst_rt > 0 ? nst_rt : 64, 1.0005, varies, dmax);
    }
  __syncwarp();
  const long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 123.0 || varies == (s < -1)) out[lane] = s;
}

template <bool SSD, int ROWS, int STRIDE>
void run(const char *name, int nst_rt = 0) {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 256);
  cudaMalloc(&cyc, 8 * 148);
  const int smem = 4 * STRIDE * 8 + 8 * 64 * 8;
  cudaFuncSetAttribute(bench<SSD, ROWS, STRIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int windows = 1000;
  bench<SSD, ROWS, STRIDE><<<148, 32, smem>>>(out, windows, cyc, nst_rt);
  bench<SSD, ROWS, STRIDE><<<148, 32, smem>>>(out, windows, cyc, nst_rt);
  long long c[148];
  cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  printf("%-40s rows=%d stride=%5d nst=%s: %.2f cycles/step (%s)\n", name, ROWS, STRIDE, nst_rt ? "runtime" : "const", (double)c[0] / (windows * 64.0),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<false, 1, 512>("sum8 chain + constancy");
  run<false, 4, 512>("sum8 chain + constancy");
  run<false, 4, 520>("sum8 chain + constancy (padded rows)");
  run<true, 1, 512>("ssd8 chain");
  run<true, 4, 512>("ssd8 chain");
  run<true, 4, 520>("ssd8 chain (padded rows)");
  run<false, 4, 512>("sum8 chain + constancy", 64);
  run<true, 4, 512>("ssd8 chain", 64);
  return 0;
}
