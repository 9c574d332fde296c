// Where the chunked K1 (normalize_rows_chunked_kernel, csrc/normalize.cuh)
// spends its time: clock64 per pass and chunk waits, for chunk sizes and
// rows in flight per SM; U checked bit for bit against normalize_rows_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCC_K1C_PROBE -I include \
//        -o tools/k1c_probe tools/k1c_probe.cu && ./tools/k1c_probe n l
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1605_01584_b200/csrc/normalize.cuh"

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 32768, l = argc > 2 ? atol(argv[2]) : 8192;
  const long ldu = (l + 31) / 32 * 32;
  std::vector<double> h(n * l);
  unsigned long long st = 0x9E3779B97F4A7C15ull;
  for (long i = 0; i < n * l; ++i) {
    st ^= st << 13, st ^= st >> 7, st ^= st << 17;
    h[i] = (double)(st >> 11) * 0x1p-53 - 0.5;
  }
  double *x, *u;
  uint8_t *f;
  cudaMalloc(&x, n * l * 8);
  cudaMalloc(&u, n * ldu * 8);
  cudaMalloc(&f, n);
  cudaMemcpy(x, h.data(), n * l * 8, cudaMemcpyHostToDevice);
  pcc::normalize_rows_kernel<<<(unsigned)((n + pcc::kNormRowsPerCta - 1) / pcc::kNormRowsPerCta), pcc::kNormThreads>>>(
      x, l, u, ldu, f, l, 0, n);
  std::vector<double> ref(n * ldu), got(n * ldu);
  cudaMemcpy(ref.data(), u, n * ldu * 8, cudaMemcpyDeviceToHost);
  auto k = pcc::normalize_rows_chunked_kernel<pcc::kNormLocal>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  pcc::NormDests d{};
  for (int ch : {1024, 2048, 4096}) {
    for (int ctas : {4, 6, 8, 12}) {
      const int budget = 224 * 1024 / ctas - 1024;
      if (2 * ch * 8 > budget) continue;
      unsigned long long z[8] = {0};
      cudaMemcpyToSymbol(pcc::g_k1c_probe, z, sizeof z);
      cudaMemset(u, 0xff, n * ldu * 8);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<(unsigned)n, pcc::kChunkThreads, budget>>>(x, l, u, ldu, f, l, 0, ch, d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      unsigned long long ph[8];
      cudaMemcpyFromSymbol(ph, pcc::g_k1c_probe, sizeof ph);
      cudaMemcpy(got.data(), u, n * ldu * 8, cudaMemcpyDeviceToHost);
      const bool same = memcmp(got.data(), ref.data(), n * ldu * 8) == 0;
      printf("n=%ld l=%ld ch=%d ctas/SM=%d: %.3f ms (%.0f GB/s) %s | per row: sum %.0f clk, ssd %.0f, output %.0f, "
             "chunk waits %.0f  (%s)\n",
             n, l, ch, ctas, ms, 16.0 * n * l / ms / 1e6, same ? "bit-exact" : "MISMATCH", (double)ph[0] / n,
             (double)ph[1] / n, (double)ph[2] / n, (double)ph[3] / n, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
