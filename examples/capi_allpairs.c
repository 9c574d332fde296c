/* The C ABI from plain C -- no Python, no torch: what a non-Python caller of
 * the engine (or a cgo / JNI binding) does.  Normalises a small random
 * dataset with pcc_normalize_rows_f64, contracts it with pcc_syrk_f64 (packed
 * layout, FP64 tensor cores), pcc_syrk_exact_f64 (the reference's dot8) and
 * split mode (pcc_split_rows_f64 + pcc_syrk_split_f64: int8 tensor cores on
 * exact digit planes), and checks all three against a direct O(n^2 l)
 * Pearson computation on the host.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/capi_allpairs.c -o examples/capi_allpairs \
 *       -L paper_1605_01584_b200/lib -lpcc_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,'$ORIGIN/../paper_1605_01584_b200/lib' -Wl,-rpath,/usr/local/cuda/lib64 -lm
 *   ./examples/capi_allpairs 300 77
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pcc_b200.h"

#define CHECK_PCC(call)                                                    \
  do {                                                                     \
    int rc_ = (call);                                                      \
    if (rc_ != PCC_OK) {                                                   \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, pcc_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)
#define CHECK_CUDA(call)                                                          \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));          \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

/* Pearson's r from the definition (two-pass, for the check only). */
static double pearson(const double *a, const double *b, int64_t l) {
  double ma = 0, mb = 0, sab = 0, saa = 0, sbb = 0;
  for (int64_t k = 0; k < l; ++k) ma += a[k], mb += b[k];
  ma /= (double)l, mb /= (double)l;
  for (int64_t k = 0; k < l; ++k) {
    sab += (a[k] - ma) * (b[k] - mb);
    saa += (a[k] - ma) * (a[k] - ma);
    sbb += (b[k] - mb) * (b[k] - mb);
  }
  return (saa == 0 || sbb == 0) ? 0.0 : sab / sqrt(saa * sbb);
}

int main(int argc, char **argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 300, l = argc > 2 ? atoll(argv[2]) : 77;
  const int64_t ldu = pcc_ldu(l), rows = pcc_rows_padded(n), pairs = n * (n + 1) / 2;
  double *x = malloc(sizeof(double) * n * l), *packed = malloc(sizeof(double) * pairs);
  uint8_t *zv = malloc(n);
  uint64_t s = 12345;
  for (int64_t i = 0; i < n * l; ++i) {  /* splitmix64 -> uniform [0, 1) */
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = (double)((z ^ (z >> 31)) >> 11) * 0x1.0p-53;
  }
  for (int64_t k = 0; k < l; ++k) x[1 * l + k] = 2.5; /* a constant row: zero variance */

  pcc_device_info_t info;
  CHECK_PCC(pcc_device_info(0, &info));
  printf("libpcc_b200 v%d: %d SMs, sm_%d%d, %d contraction CTAs/SM\n", pcc_version(), info.sm_count, info.cc_major,
         info.cc_minor, info.syrk_ctas_per_sm);

  double *dx, *du, *dout;
  uint8_t *dzv;
  CHECK_CUDA(cudaMalloc((void **)&dx, sizeof(double) * n * l));
  CHECK_CUDA(cudaMalloc((void **)&du, sizeof(double) * rows * ldu));
  CHECK_CUDA(cudaMalloc((void **)&dout, sizeof(double) * pairs));
  CHECK_CUDA(cudaMalloc((void **)&dzv, n));
  CHECK_CUDA(cudaMemcpy(dx, x, sizeof(double) * n * l, cudaMemcpyHostToDevice));
  CHECK_PCC(pcc_normalize_rows_f64(dx, l, du, ldu, dzv, l, 0, n, NULL));  /* K1 */
  CHECK_PCC(pcc_zero_rows_f64(du, ldu, n, rows, NULL));                 /* pad rows */
  const uint64_t tiles = pcc_gpu_tile_count(n);
  int8_t *dslices;
  double *dscale;
  CHECK_CUDA(cudaMalloc((void **)&dslices, pcc_split_slice_bytes(n, l)));
  CHECK_CUDA(cudaMalloc((void **)&dscale, sizeof(double) * rows));
  CHECK_PCC(pcc_split_rows_f64(du, n, l, ldu, 0, rows, dslices, dscale, NULL)); /* digit planes, pad rows too */
  double worst[3] = {0, 0, 0};
  for (int exact = 0; exact < 3; ++exact) {
    if (exact == 1)
      CHECK_PCC(pcc_syrk_exact_f64(du, n, l, ldu, 0, tiles, PCC_LAYOUT_PACKED, dout, 0, 0, 0, 0, 0, NULL));
    else if (exact == 2)
      CHECK_PCC(pcc_syrk_split_f64(dslices, dscale, n, l, 0, tiles, PCC_LAYOUT_PACKED, dout, 0, 0, 0, 0, 0, NULL));
    else
      CHECK_PCC(pcc_syrk_f64(du, n, l, ldu, 0, tiles, PCC_LAYOUT_PACKED, dout, 0, 0, 0, 0, 0, NULL));
    CHECK_CUDA(cudaMemcpy(packed, dout, sizeof(double) * pairs, cudaMemcpyDeviceToHost));
    for (int64_t y = 0, idx = 0; y < n; ++y)
      for (int64_t xx = y; xx < n; ++xx, ++idx) {
        const double d = fabs(packed[idx] - pearson(x + y * l, x + xx * l, l));
        if (d > worst[exact]) worst[exact] = d;
      }
  }
  CHECK_CUDA(cudaMemcpy(zv, dzv, n, cudaMemcpyDeviceToHost));
  printf("n=%lld l=%lld: max |r - definition| tensor path %.2e, exact mode %.2e, split mode %.2e; "
         "zero-variance row 1 flagged %d\n",
         (long long)n, (long long)l, worst[0], worst[1], worst[2], zv[1]);
  const int ok = worst[0] < 1e-12 && worst[1] < 1e-12 && worst[2] < 1e-12 && zv[1] == 1;
  cudaFree(dx), cudaFree(du), cudaFree(dout), cudaFree(dzv), cudaFree(dslices), cudaFree(dscale);
  free(x), free(packed), free(zv);
  printf(ok ? "ok\n" : "FAILED\n");
  return ok ? 0 : 1;
}
