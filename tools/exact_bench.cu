// Standalone timing of the exact-mode contraction (csrc/exact.cuh) on a
// random padded U, packed output; -DPCC_EXACT_NOLOAD skips the global->shared
// copies (stale operands) to separate the math from the data movement.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exact_bench tools/exact_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1605_01584_b200/csrc/exact.cuh"

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 16384, l = argc > 2 ? atol(argv[2]) : 4096;
  const long ldu = (l + 31) / 32 * 32, rows = (n + 127) / 128 * 128;
  std::vector<double> h(rows * ldu, 0.0);
  for (long r = 0; r < n; ++r)
    for (long k = 0; k < l; ++k) h[r * ldu + k] = ((r * 7919 + k * 104729) % 1000) * 1e-3 - 0.5;
  double *u, *out;
  cudaMalloc(&u, rows * ldu * 8);
  cudaMalloc(&out, (size_t)n * (n + 1) / 2 * 8);
  cudaMemcpy(u, h.data(), rows * ldu * 8, cudaMemcpyHostToDevice);
  using C = pcc::ExactCfg;
  cudaFuncSetAttribute(pcc::syrk_exact_kernel<pcc::kLayoutPacked, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::kSmemBytes);
  cudaFuncSetAttribute(pcc::syrk_exact_kernel<pcc::kLayoutPacked, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       C::kSmemBytes);
  const bool bulk = !(argc > 3 && argv[3][0] == 'c');  // 'c': the cp.async variant

  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t m = (n + 127) / 128, T = m * (m + 1) / 2;
  uint32_t group = 1;
  while ((uint64_t)(group + 1) * (group + 1) * C::kSubPerTile <= (uint64_t)sms) ++group;
  const pcc::TileOrder order = pcc::make_tile_order(m, 0, T, group);
  pcc::Epilogue ep{out, 0, 0, 0, 0, 0, 0};
  const int k_chunks = (int)((l + C::BK - 1) / C::BK);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    if (bulk)
      pcc::syrk_exact_kernel<pcc::kLayoutPacked, true><<<sms, C::kThreads, C::kSmemBytes>>>(u, n, ldu, k_chunks, m,
                                                                                            order, ep);
    else
      pcc::syrk_exact_kernel<pcc::kLayoutPacked, false><<<sms, C::kThreads, C::kSmemBytes>>>(u, n, ldu, k_chunks, m,
                                                                                             order, ep);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  const double ops = 2.0 * l * (double)n * (n + 1) / 2;
  std::vector<double> res((size_t)n * (n + 1) / 2);
  cudaMemcpy(res.data(), out, res.size() * 8, cudaMemcpyDeviceToHost);
  double cs = 0;
  for (size_t i = 0; i < res.size(); i += 997) cs += res[i];
  printf("%s checksum %.17g\n", bulk ? "bulk" : "cp.async", cs);
  printf("n=%ld l=%ld: %.3f ms  %.2f Tops/s  %.1f%% of 18.52 (%s)\n", n, l, best, ops / (best * 1e-3) / 1e12,
         ops / (best * 1e-3) / 1e12 / 18.52 * 100, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
