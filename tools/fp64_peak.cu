// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64).
// Used once to decide the contraction kernel's inner loop and to measure the
// FP64 roofline denominator on the box.  Not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int iters = 20000;
      dfma_loop<<<sms * bps, tpb>>>(out, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_loop<<<sms * bps, tpb>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * iters * (double)tpb * sms * bps;
      printf("DFMA tpb=%d ctas/sm=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, bps, flops / ms / 1e9, ms);
    }
  }
  for (int tpb : {128, 256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int iters = 20000;
      dmma_loop<<<sms * bps, tpb>>>(out, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dmma_loop<<<sms * bps, tpb>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * iters * (double)(tpb / 32) * sms * bps;
      printf("DMMA tpb=%d ctas/sm=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, bps, flops / ms / 1e9, ms);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
