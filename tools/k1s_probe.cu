// Where the streamed K1 spends its time (clock64 totals per warp):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCC_K1S_PROBE -o tools/k1s_probe tools/k1s_probe.cu
//   ./tools/k1s_probe n l cw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "experiments/normalize_stream.cuh"

template <int CW>
void run(const double *x, double *u, uint8_t *f, long n, long l, long ldu) {
  auto k = pcc::normalize_rows_stream_kernel<pcc::kNormLocal, CW>;
  const int smem = pcc::K1Stream::smem_bytes(CW);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long groups = (n + 3) / 4;
  long grid = (groups + CW - 1) / CW;
  if (grid > sms) grid = sms;
  pcc::NormDests d{};
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(pcc::g_k1s_probe, z, sizeof z);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<(unsigned)grid, (CW + pcc::K1Stream::kApplyWarps) * 32, smem>>>(x, l, u, ldu, f, l, 0, n, d, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long ph[8];
    cudaMemcpyFromSymbol(ph, pcc::g_k1s_probe, sizeof ph);
    if (rep == 2) {
      const double nc = (double)grid * CW, na = (double)grid * pcc::K1Stream::kApplyWarps;
      printf("n=%ld l=%ld CW=%d grid=%ld: %.3f ms (%.0f GB/s)  chain warp: total %.0f clk, data wait %.0f, handoff wait "
             "%.0f | output warp: total %.0f, wait %.0f  (%s)\n",
             n, l, CW, grid, ms, 16.0 * n * l / ms / 1e6, ph[2] / nc, ph[0] / nc, ph[1] / nc, ph[4] / na, ph[3] / na,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 65536, l = argc > 2 ? atol(argv[2]) : 2048;
  const long ldu = (l + 31) / 32 * 32;
  std::vector<double> h(n * l);
  for (long i = 0; i < n * l; ++i) h[i] = (double)((i * 2654435761u) % 1000003) * 1e-3;
  double *x, *u;
  uint8_t *f;
  cudaMalloc(&x, n * l * 8);
  cudaMalloc(&u, n * ldu * 8);
  cudaMalloc(&f, n);
  cudaMemcpy(x, h.data(), n * l * 8, cudaMemcpyHostToDevice);
  run<1>(x, u, f, n, l, ldu);
  run<2>(x, u, f, n, l, ldu);

  return 0;
}
