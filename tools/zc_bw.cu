// Microbenchmark: GPU -> host bandwidth of (a) cudaMemcpyAsync D2H into pinned
// memory and (b) SM stores straight into mapped pinned memory ("zero-copy"),
// for the store patterns a packed-output epilogue can produce:
//   line  : each warp store covers 256 contiguous bytes
//   seg64 : each warp store covers 4 rows x 64 B (rows far apart)
//   seg32 : each warp store covers 8 rows x 32 B (the DMMA accumulator layout)
// plus H2D copy alone and concurrently with zero-copy writes (PCIe duplex).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_bw tools/zc_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); return 1; } } while (0)

// seg = contiguous doubles per row within one warp store; rows spaced by `pitch` doubles
template <int SEG>
__global__ void zc_write(double *__restrict__ dst, long long rows, long long pitch, long long row_len, double v) {
  constexpr int kRowsPerStore = 32 / SEG;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long segs_per_row = row_len / SEG;
  const long long groups = (rows / kRowsPerStore) * segs_per_row;
  for (long long g = warp; g < groups; g += nwarps) {
    const long long rg = g / segs_per_row, sg = g % segs_per_row;
    const long long row = rg * kRowsPerStore + lane / SEG;
    const long long col = sg * SEG + lane % SEG;
    __stcs(dst + row * pitch + col, v + col);
  }
}

int main() {
  const size_t bytes = 1ull << 30;  // 1 GiB
  const long long nd = bytes / 8;
  double *h, *hd, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  double *h2;
  CK(cudaHostAlloc(&h2, bytes / 2, cudaHostAllocDefault));
  double *d2;
  CK(cudaMalloc(&d2, bytes / 2));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t a, b, c, e;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c)); CK(cudaEventCreate(&e));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float ms;
  auto report = [&](const char *what, double gb, float t) { printf("%-44s %8.3f ms  %7.2f GB/s\n", what, t, gb / (t * 1e-3)); };

  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(a, s0)); CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s0)); CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    if (rep) report("memcpy D2H 1 GiB", bytes / 1e9, ms);
    CK(cudaEventRecord(a, s0)); CK(cudaMemcpyAsync(d2, h2, bytes / 2, cudaMemcpyHostToDevice, s0)); CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
    if (rep) report("memcpy H2D 0.5 GiB", bytes / 2e9, ms);
    // row_len 16384 doubles, pitch = row_len: contiguous overall but split per row
    const long long row_len = 16384, rows = nd / row_len;
    for (int blocks_per_sm : {1, 2, 4}) {
      const int grid = sms * blocks_per_sm;
      char name[96];
      CK(cudaEventRecord(a, s0)); zc_write<32><<<grid, 256, 0, s0>>>(hd, rows, row_len, row_len, 1.0); CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      snprintf(name, sizeof name, "zero-copy line (256 B/store), %d CTA/SM", blocks_per_sm);
      if (rep) report(name, bytes / 1e9, ms);
      CK(cudaEventRecord(a, s0)); zc_write<8><<<grid, 256, 0, s0>>>(hd, rows, row_len, row_len, 1.0); CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      snprintf(name, sizeof name, "zero-copy seg64 (4 rows x 64 B), %d CTA/SM", blocks_per_sm);
      if (rep) report(name, bytes / 1e9, ms);
      CK(cudaEventRecord(a, s0)); zc_write<4><<<grid, 256, 0, s0>>>(hd, rows, row_len, row_len, 1.0); CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      snprintf(name, sizeof name, "zero-copy seg32 (8 rows x 32 B), %d CTA/SM", blocks_per_sm);
      if (rep) report(name, bytes / 1e9, ms);
    }
    // duplex: zero-copy writes on s0 while H2D runs on s1
    CK(cudaEventRecord(a, s0)); CK(cudaStreamWaitEvent(s1, a, 0));
    zc_write<32><<<sms * 2, 256, 0, s0>>>(hd, rows, row_len, row_len, 1.0); CK(cudaEventRecord(b, s0));
    CK(cudaMemcpyAsync(d2, h2, bytes / 2, cudaMemcpyHostToDevice, s1)); CK(cudaEventRecord(c, s1));
    CK(cudaEventSynchronize(b)); CK(cudaEventSynchronize(c));
    float m1, m2; CK(cudaEventElapsedTime(&m1, a, b)); CK(cudaEventElapsedTime(&m2, a, c));
    if (rep) { report("duplex: zero-copy line 1 GiB", bytes / 1e9, m1); report("duplex: H2D 0.5 GiB", bytes / 2e9, m2); }
    // duplex: memcpy D2H on s0 while H2D on s1
    CK(cudaEventRecord(a, s0)); CK(cudaStreamWaitEvent(s1, a, 0));
    CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s0)); CK(cudaEventRecord(b, s0));
    CK(cudaMemcpyAsync(d2, h2, bytes / 2, cudaMemcpyHostToDevice, s1)); CK(cudaEventRecord(c, s1));
    CK(cudaEventSynchronize(b)); CK(cudaEventSynchronize(c));
    CK(cudaEventElapsedTime(&m1, a, b)); CK(cudaEventElapsedTime(&m2, a, c));
    if (rep) { report("duplex: memcpy D2H 1 GiB", bytes / 1e9, m1); report("duplex: H2D 0.5 GiB", bytes / 2e9, m2); }
  }
  CK(cudaDeviceSynchronize());
  printf("check %.1f %.1f\n", h[0], h[nd - 1]);
  return 0;
}
