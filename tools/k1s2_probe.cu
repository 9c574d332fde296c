// Where the streamed K1 (csrc/normalize_stream.cuh) spends its time: clock64
// totals per role, per launch shape; checks U bit for bit against the plain
// 8-lane kernel (normalize_rows_kernel, same arithmetic contract).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPCC_K1S_PROBE -I include \
//        -o tools/k1s2_probe tools/k1s2_probe.cu
//   ./tools/k1s2_probe n l
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "experiments/normalize_stream2.cuh"

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
CUtensorMap xmap_of(const double *x, long ldx, long l, long rows, int box_rows) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)l, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
  const cuuint32_t box[2] = {(cuuint32_t)pcc::K1Stream::kBox, (cuuint32_t)box_rows}, estr[2] = {1, 1};
  reinterpret_cast<EncodeTiledFn>(p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(x), dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

void run(const double *x, double *u, uint8_t *f, long n, long l, long ldu, const std::vector<double> &ref) {
  using S = pcc::K1Stream;
  auto k = pcc::normalize_rows_stream_kernel<pcc::kNormLocal>;
  constexpr int CW = S::kChainWarps, OW = S::kOutWarps;
  const int smem = S::smem_bytes(CW, OW);
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
    cudaMemset(u, 0xff, n * ldu * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<(unsigned)grid, S::kThreads, smem>>>(xmap_of(x, l, l, n, 1), xmap_of(x, l, l, n, 4), u, ldu, f, l, 0, n, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long ph[8];
    cudaMemcpyFromSymbol(ph, pcc::g_k1s_probe, sizeof ph);
    if (rep == 2) {
      std::vector<double> h(n * ldu);
      cudaMemcpy(h.data(), u, n * ldu * 8, cudaMemcpyDeviceToHost);
      const bool same = memcmp(h.data(), ref.data(), n * ldu * 8) == 0;
      const double nc = (double)grid * CW, no = (double)grid * OW;
      printf("n=%ld l=%ld CW=%d OW=%d: %.3f ms (%.0f GB/s) %s | chain: total %.0f clk, window waits %.0f, handoff "
             "waits %.0f | output: total %.0f, handoff waits %.0f, window waits %.0f  (%s)\n",
             n, l, CW, OW, ms, 16.0 * n * l / ms / 1e6, same ? "bit-exact" : "MISMATCH", ph[0] / nc, ph[1] / nc,
             ph[2] / nc, ph[3] / no, ph[4] / no, ph[5] / no, cudaGetErrorString(cudaGetLastError()));
    }
  }
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 32768, l = argc > 2 ? atol(argv[2]) : 8192;
  const long ldu = (l + 31) / 32 * 32;
  std::vector<double> h(n * l);
  unsigned long long st = 0x9E3779B97F4A7C15ull;
  for (long i = 0; i < n * l; ++i) {
    st ^= st << 13, st ^= st >> 7, st ^= st << 17;
    h[i] = (double)(st >> 11) * 0x1p-53 - 0.5;
  }
  for (long r = 0; r < n; r += 97)  // planted constant rows
    for (long k = 0; k < l; ++k) h[r * l + k] = 0.25;
  double *x, *u;
  uint8_t *f;
  cudaMalloc(&x, n * l * 8);
  cudaMalloc(&u, n * ldu * 8);
  cudaMalloc(&f, n);
  cudaMemcpy(x, h.data(), n * l * 8, cudaMemcpyHostToDevice);
  cudaMemset(u, 0, n * ldu * 8);
  pcc::normalize_rows_kernel<<<(unsigned)((n + pcc::kNormRowsPerCta - 1) / pcc::kNormRowsPerCta), pcc::kNormThreads>>>(
      x, l, u, ldu, f, l, 0, n);
  std::vector<double> ref(n * ldu);
  cudaMemcpy(ref.data(), u, n * ldu * 8, cudaMemcpyDeviceToHost);
  run(x, u, f, n, l, ldu, ref);
  return 0;
}
