// Phase breakdown of K1's staged kernel (clock64 per CTA, thread 0):
// staging, lane chains (sum + constancy, ssd), output.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCC_K1_PHASES -o tools/k1_phases tools/k1_phases.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1605_01584_b200/csrc/normalize.cuh"

template <int T>
void run(const double *x, double *u, uint8_t *f, long n, long l, long ldu, int rows_per_cta) {
  const long lds = (l % 2) ? ((l + 3) & ~1L) : l;  // the host's slot stride for odd / misaligned rows
  const size_t smem = (size_t)rows_per_cta * lds * sizeof(double);
  cudaFuncSetAttribute(pcc::normalize_rows_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcc::normalize_rows_smem_kernel<T>, T, smem);
  const unsigned grid = (unsigned)((n + rows_per_cta - 1) / rows_per_cta);
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(pcc::g_k1_phase, z, sizeof z);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    pcc::normalize_rows_smem_kernel<T><<<grid, T, smem>>>(x, l, u, ldu, f, l, 0, n, rows_per_cta, lds, pcc::NormDests{});
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long ph[8];
    cudaMemcpyFromSymbol(ph, pcc::g_k1_phase, sizeof ph);
    if (rep == 2) {
      printf("threads %d rows/cta %d occupancy %d CTAs/SM: %.3f ms  per-CTA clk:", T, rows_per_cta, occ, ms);
      const char *nm[3] = {"stage", "chains", "out"};
      double tot = 0;
      for (int i = 0; i < 3; ++i) tot += (double)ph[i] / grid;
      for (int i = 0; i < 3; ++i) printf(" %s %.0f", nm[i], (double)ph[i] / grid);
      printf("  total %.0f\n", tot);
    }
  }
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 16384, l = argc > 2 ? atol(argv[2]) : 4096;
  const long ldu = (l + 31) / 32 * 32;
  std::vector<double> h(n * l);
  for (long i = 0; i < n * l; ++i) h[i] = (double)((i * 2654435761u) % 1000003) * 1e-3;
  double *x, *u; uint8_t *f;
  cudaMalloc(&x, n * l * 8); cudaMalloc(&u, n * ldu * 8); cudaMalloc(&f, n);
  cudaMemcpy(x, h.data(), n * l * 8, cudaMemcpyHostToDevice);
  const int rows_list[] = {1, 2, 3, 4, 8};
  for (int r : rows_list) {
    if ((long)r * l * 8 > 200 * 1024) continue;
    run<64>(x, u, f, n, l, ldu, r);
    run<128>(x, u, f, n, l, ldu, r);
    run<256>(x, u, f, n, l, ldu, r);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
