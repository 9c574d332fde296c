// FP64 CUDA-core throughput of separately rounded multiply + add (the exact
// contraction's inner operation) vs DFMA, 8/16/32 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_alu tools/fp64_alu.cu
#include <cstdio>
#include <cuda_runtime.h>
template <bool FMA>
__global__ void alu(double *out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double x = a + threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FMA) acc[i] = __fma_rn(x, b, acc[i]);
      else acc[i] = __dadd_rn(acc[i], __dmul_rn(x, acc[(i + 8) & 15]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int fma = 0; fma < 2; ++fma) {
      float best = 1e9;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        if (fma) alu<true><<<sms, warps * 32>>>(o, iters, 1.0000001, 0.999999);
        else alu<false><<<sms, warps * 32>>>(o, iters, 1.0000001, 0.999999);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      const double ops = (double)sms * warps * 32 * iters * 16 * (fma ? 1 : 2);
      printf("%2d warps/SM %s: %.3f ms  %.2f Tops/s  %.1f ops/clk/SM @1.965GHz\n", warps, fma ? "DFMA     " : "DMUL+DADD",
             best, ops / (best * 1e-3) / 1e12, ops / (best * 1e-3) / 1.965e9 / sms);
    }
  }
  return 0;
}
