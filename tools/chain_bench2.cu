// What limits one reference lane chain step (s = RN(s + x_k)) out of shared
// memory on B200?  One warp per SM; variants:
//   A  DADD chain, operands from registers (pure latency)
//   B  DADD chain, operands from smem (8-deep register ping-pong prefetch)
//   C  B + the constancy test (DSETP into an OR chain)
//   D  B with two independent chains per lane (rows r and r + 4)
//   E  ssd chain: d = x - m; s = RN(s + RN(d*d))
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/chain_bench2 tools/chain_bench2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int STEPS = 64;  // per window, per lane (512-element window, 8 lanes)

template <int V>
__global__ void bench(double *out, int windows, long long *cyc, int stride) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x, j = lane & 7, r = lane >> 3;
  for (int i = lane; i < 8 * 520 + 1024; i += 32) sm[i] = 1.0 + 1e-3 * (i % 97);
  __syncwarp();
  double s = 0.0, s2 = 0.0, x0 = sm[0], m = 1.0003;
  bool varies = false;
  const double *p = sm + r * stride + j, *p2 = sm + (r + 4) * stride + j;
  long long t0 = clock64();
  for (int w = 0; w < windows; ++w) {
    const int off = (w & 1) * 8;  // keep the compiler from hoisting the loads out
    if (V == 0) {
#pragma unroll 16
      for (int t = 0; t < STEPS; ++t) s = __dadd_rn(s, x0 + (double)off);
    } else {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = p[off + 8 * i];
      double a2[8], b2[8];
      if (V == 3) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a2[i] = p2[off + 8 * i];
      }
      for (int t = 0; t < STEPS; t += 16) {
#pragma unroll
        for (int i = 0; i < 8; ++i) b[i] = p[off + 8 * (t + 8 + i)];
        if (V == 3) {
#pragma unroll
          for (int i = 0; i < 8; ++i) b2[i] = p2[off + 8 * (t + 8 + i)];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (V == 4) { const double d = __dsub_rn(a[i], m); s = __dadd_rn(s, __dmul_rn(d, d)); }
          else s = __dadd_rn(s, a[i]);
          if (V == 2) varies |= a[i] != x0;
          if (V == 3) s2 = __dadd_rn(s2, a2[i]);
        }
        if (t + 16 < STEPS) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = p[off + 8 * (t + 16 + i)];
          if (V == 3) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a2[i] = p2[off + 8 * (t + 16 + i)];
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (V == 4) { const double d = __dsub_rn(b[i], m); s = __dadd_rn(s, __dmul_rn(d, d)); }
          else s = __dadd_rn(s, b[i]);
          if (V == 2) varies |= b[i] != x0;
          if (V == 3) s2 = __dadd_rn(s2, b2[i]);
        }
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
  if (s == 123.0 || s2 == 7.0 || varies == (s < -1)) out[lane] = s + s2;
}

template <int V>
void run(const char *name, int warps_rows, int stride) {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 256);
  cudaMalloc(&cyc, 8 * 148);
  const int smem = (8 * 520 + 1024) * 8;
  cudaFuncSetAttribute(bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int windows = 2000;
  bench<V><<<148, 32, smem>>>(out, windows, cyc, stride);
  bench<V><<<148, 32, smem>>>(out, windows, cyc, stride);
  long long c[148];
  cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  printf("%-58s stride %4d: %6.2f cycles/step  (%s)\n", name, stride, (double)c[0] / (windows * (double)STEPS),
         cudaGetErrorString(cudaGetLastError()));
  (void)warps_rows;
}

int main() {
  run<0>("A  DADD chain, register operands", 4, 512);
  run<1>("B  DADD chain, smem operands (4 rows x 8 lanes)", 4, 512);
  run<1>("B' same, rows 520 doubles apart", 4, 520);
  run<2>("C  B + constancy DSETP/OR", 4, 512);
  run<3>("D  two chains per lane (rows r, r+4)", 4, 520);
  run<4>("E  ssd chain (DSUB, DMUL, DADD)", 4, 512);
  return 0;
}
