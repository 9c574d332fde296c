// Bulk-copy (cp.async.bulk, 1-D) throughput from global memory into shared
// memory: W warps per CTA, one CTA per SM, each warp's lane 0 keeps D copies
// of S bytes in flight on per-slot mbarriers.  Prints GB/s for each (S, D, W).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bulk_bw tools/bulk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// LANES issuing threads per warp, each with its own D slots of S bytes.
__global__ void k(const char *src, size_t total, uint32_t S, int D, int iters, unsigned long long *sink, int LANES) {
  extern __shared__ __align__(128) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int ch = warp * LANES + lane;  // issuing channel
  const uint32_t base = smem_u32(sm) + ch * D * S;
  const uint32_t bars = smem_u32(sm) + W * LANES * D * S + ch * D * 8;
  if (lane < LANES) {
    for (int d = 0; d < D; ++d) mbar_init(bars + 8 * d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const size_t gw = (size_t)blockIdx.x * W * LANES + ch, nw = (size_t)gridDim.x * W * LANES;
  unsigned long long acc = 0;
  if (lane < LANES) {
    for (int i = 0; i < D && i < iters; ++i) {
      mbar_expect(bars + 8 * i, S);
      bulk(base + i * S, src + ((gw + (size_t)i * nw) * S) % total, S, bars + 8 * i);
    }
    for (int i = 0; i < iters; ++i) {
      const int s = i % D;
      while (!mbar_try(bars + 8 * s, (i / D) & 1)) {
      }
      acc += sm[base - smem_u32(sm) + s * S];
      const int nx = i + D;
      if (nx < iters) {
        mbar_expect(bars + 8 * s, S);
        bulk(base + s * S, src + ((gw + (size_t)nx * nw) * S) % total, S, bars + 8 * s);
      }
    }
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)4 << 30;
  char *src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t sizes[] = {2048, 4096, 8192};
  const int depths[] = {2, 4};
  const int warps[] = {1, 2};
  const int lanes_[] = {1, 2, 4, 8};
  for (uint32_t S : sizes)
    for (int D : depths)
      for (int W : warps)
      for (int LN : lanes_) {
        const size_t smem = (size_t)W * LN * D * S + W * LN * D * 8;
        if (smem > 220 * 1024) continue;
        const int iters = (int)(((size_t)1 << 31) / ((size_t)sms * W * LN * S));  // 2 GB per run
        k<<<sms, 32 * W, smem>>>(src, total, S, D, iters, sink, LN);
        cudaEventRecord(e0);
        k<<<sms, 32 * W, smem>>>(src, total, S, D, iters, sink, LN);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)sms * W * LN * S * iters;
        printf("S=%6u D=%d W=%d lanes=%d : %7.1f GB/s  (%.1f B/clk/SM @1.9GHz)  %s\n", S, D, W, LN, bytes / ms / 1e6,
               bytes / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
        (void)LN;
      }
  return 0;
}
