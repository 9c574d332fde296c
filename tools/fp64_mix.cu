// Do DMMA (FP64 tensor pipe) and DFMA (FP64 ALU pipe) execute concurrently on
// B200?  Half the warps of each CTA run DMMA chains, half DFMA chains; compare
// the combined FLOP rate with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void mix(double* out, int iters, int dmma_warps, int dfma_warps) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w < dmma_warps) {
    double c[8][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else if (w < dmma_warps + dfma_warps) {
    double acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    double a = 1.0000001, b = 1e-9;
    // 8 DMMA (2048 FMA/warp) vs 16 DFMA (512 FMA/warp) per iteration: run 4x the iterations
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    for (int i = 0; i < 16; ++i) s += acc[i];
  }
  if (s == 1234.5) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int cfg[][2] = {{8, 0}, {0, 8}, {4, 4}, {8, 8}, {16, 0}, {0, 16}, {8, 4}, {12, 4}};
  for (auto& c : cfg) {
    int threads = 32 * (c[0] + c[1]);
    int iters = 4000;
    mix<<<sms, threads>>>(d, 100, c[0], c[1]);
    cudaEventRecord(e0);
    mix<<<sms, threads>>>(d, iters, c[0], c[1]);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * sms * ((double)c[0] * 8 * 256 * iters + (double)c[1] * 32 * 16 * iters * 4);
    printf("dmma_warps=%2d dfma_warps=%2d: %.3f ms  %.2f TFLOP/s\n", c[0], c[1], ms, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
