// Microbenchmark: dependent FP64 add chain latency on B200 (one warp), and
// the same chain fed from shared memory (LDS + DADD) as in K1's lane chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dadd_chain(double* out, int iters, double x) {
  double s = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { s = __dadd_rn(s, x); s = __dadd_rn(s, x); s = __dadd_rn(s, x); s = __dadd_rn(s, x); }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = s; out[1] = (double)(t1 - t0) / (4.0 * iters); }
}
__global__ void lds_dadd_chain(double* out, int iters) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 1e-3;
  __syncthreads();
  double s = 0; int lane = threadIdx.x & 7;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    #pragma unroll 8
    for (int k = lane; k < 4096; k += 8) s = __dadd_rn(s, buf[k]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = s; out[1] = (double)(t1 - t0) / (512.0 * iters); }
}
int main() {
  double* d; cudaMalloc(&d, 16); double h[2];
  dadd_chain<<<1, 32>>>(d, 100000, 1e-9); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DADD dependent chain: %.2f cycles/add\n", h[1]);
  lds_dadd_chain<<<1, 32>>>(d, 200); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("LDS+DADD lane chain (unroll 8): %.2f cycles/step\n", h[1]);
  lds_dadd_chain<<<1, 8>>>(d, 200); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("LDS+DADD lane chain, 8 threads: %.2f cycles/step\n", h[1]);
  return 0;
}
