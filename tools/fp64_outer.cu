// FP64 CUDA-core throughput of the exact contraction's inner block: a 4 x 8
// outer product of register operands accumulated with separately rounded
// DMUL + DADD (operands refreshed from shared memory every step), 16 warps/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_outer tools/fp64_outer.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int RT, bool SMEM>
__global__ void __launch_bounds__(512, 1) outer(double *out, int iters) {
  __shared__ double buf[512 * 2];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc[RT][8];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;
  double a[RT], b[8];
#pragma unroll
  for (int i = 0; i < RT; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int c = 0; c < 8; ++c) b[c] = 0.5 + c * 1e-3;
  const int lane = threadIdx.x & 7;
  for (int it = 0; it < iters; ++it) {
    if (SMEM) {
#pragma unroll
      for (int i = 0; i < RT; ++i) a[i] = buf[(i * 40 + lane + (it & 3) * 8) & 1023];
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] = buf[(512 + c * 40 + lane + (it & 3) * 8) & 1023];
    }
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = __dadd_rn(acc[i][c], __dmul_rn(a[i], b[c]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[i][c];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](auto kern, int rt, const char *name) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      kern<<<sms, 512>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double ops = (double)sms * 512 * iters * rt * 8 * 2;
    printf("%-28s %.3f ms  %.1f ops/clk/SM @1.965GHz\n", name, best, ops / (best * 1e-3) / 1.965e9 / sms);
  };
  run(outer<4, false>, 4, "4x8 outer, register operands");
  run(outer<4, true>, 4, "4x8 outer, smem operands");
  run(outer<2, true>, 2, "2x8 outer, smem operands");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
