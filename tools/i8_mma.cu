// i8_mma.cu -- tcgen05.mma kind::i8 on one B200: (1) correctness of the
// descriptor encodings in csrc/tcgen05.cuh (K-major, 32-byte swizzle, s32
// accumulators in TMEM) against a host integer GEMM, (2) the tensor pipe's
// int8 throughput for M = 128 and N = 64 / 128 / 256 with random operands
// (power draw depends on the data), one CTA per SM.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1605_01584_b200/csrc \
//        tools/i8_mma.cu -o tools/i8_mma && ./tools/i8_mma
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tcgen05.cuh"

using namespace pcc;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

// byte offset of (row r, k byte c) in a K-major 32-byte-swizzled operand
__host__ __device__ inline uint32_t sw32(uint32_t r, uint32_t c) {
  uint32_t off = r * 32 + c;
  return off ^ (((off >> 7) & 1) << 4);
}

__device__ inline void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// D[128 x 64] = sum_s A_s[128 x 32] B_s[64 x 32]^T over `steps` K steps.
__global__ void check_kernel(const int8_t *a, const int8_t *b, int steps, int32_t *d) {
  __shared__ __align__(1024) int8_t sa[4][128 * 32];
  __shared__ __align__(1024) int8_t sb[4][64 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int s = 0; s < steps; ++s) {
    for (int i = tid; i < 128 * 32; i += blockDim.x) sa[s][sw32(i / 32, i % 32)] = a[s * 128 * 32 + i];
    for (int i = tid; i < 64 * 32; i += blockDim.x) sb[s][sw32(i / 32, i % 32)] = b[s * 64 * 32 + i];
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), 64);
  if (tid == 0) mbar_init(smem_u32(&bar), 1), mbar_fence_init();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    for (int s = 0; s < steps; ++s)
      umma_i8(tm, umma_desc_k_sw32(smem_u32(sa[s])), umma_desc_k_sw32(smem_u32(sb[s])), idesc_i8_s32<128, 64>(),
              s > 0);
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  for (int c = 0; c < 64; c += 16) {
    int32_t v[16];
    tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) d[(warp * 32 + (tid & 31)) * 64 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 64);
}

template <int N>
__global__ void peak_kernel(const int8_t *src, int iters, int32_t *sink, long long *cycles, int zero) {
  constexpr int kAcc = 512 / N;  // accumulators that fit in TMEM
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  int8_t *sa = (int8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);  // 7 x 128 x 32
  int8_t *sb = sa + 7 * 128 * 32;                                      // 7 x N x 32
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 7 * (128 + N) * 32; i += blockDim.x)
    sa[i] = zero ? (int8_t)0 : src[(blockIdx.x * 977 + i) & ((1 << 20) - 1)];
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), 512);
  if (tid == 0) mbar_init(smem_u32(&bar), 1), mbar_fence_init();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  long long c0 = clock64();
  if (tid == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    for (int it = 0; it < iters; ++it) {
      int q = 0;
#pragma unroll 1
      for (int i = 0; i < 7; ++i)
#pragma unroll 1
        for (int j = 0; j < 7 && i + j <= 7; ++j, ++q)
          umma_i8(tm + (uint32_t)(((i + j) % kAcc) * N), umma_desc_k_sw32(a0 + i * 128 * 32),
                  umma_desc_k_sw32(b0 + j * N * 32), idesc_i8_s32<128, N>(), it > 0 || q >= kAcc);
    }
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  if (tid == 0 && cycles) cycles[blockIdx.x] = clock64() - c0;
  tc_fence_after();
  int32_t v[16];
  tmem_ld16(tm + ((uint32_t)(warp * 32) << 16), v);
  tmem_ld_wait();
  if (v[0] == 0x7fffffff) sink[tid] = v[1];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

// A operand from tensor memory (".kind::i8 [d], [a_tmem], b_desc"): 3
// accumulators of N columns + 7 A slices of 8 columns (128 rows x 32 int8).
template <int N>
__global__ void peak_ts_kernel(const int8_t *src, int iters, int32_t *sink, long long *cycles) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  int8_t *sb = (int8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);  // 7 x N x 32
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 7 * N * 32; i += blockDim.x) sb[i] = src[(blockIdx.x * 977 + i) & ((1 << 20) - 1)];
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), 512);
  if (tid == 0) mbar_init(smem_u32(&bar), 1), mbar_fence_init();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  long long c0 = clock64();
  if (tid == 0) {
    const uint32_t b0 = smem_u32(sb);
    for (int it = 0; it < iters; ++it) {
      int q = 0;
#pragma unroll 1
      for (int i = 0; i < 7; ++i)
#pragma unroll 1
        for (int j = 0; j < 7 && i + j <= 7; ++j, ++q) {
          const uint32_t d = tm + (uint32_t)(((i + j) % 3) * N), a = tm + 384u + 8u * i;
          const uint64_t bd = umma_desc_k_sw32(b0 + j * N * 32);
          const uint32_t acc = (it > 0 || q >= 3) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
              "r"(a), "l"(bd), "r"(idesc_i8_s32<128, N>()), "r"(acc));
        }
    }
    umma_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  if (tid == 0 && cycles) cycles[blockIdx.x] = clock64() - c0;
  tc_fence_after();
  int32_t v[16];
  tmem_ld16(tm + ((uint32_t)(warp * 32) << 16), v);
  tmem_ld_wait();
  if (v[0] == 0x7fffffff) sink[tid] = v[1];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

template <int N>
void run_peak_ts(const int8_t *src, int32_t *sink, int sms) {
  const size_t smem = 1024 + 7 * N * 32;
  CK(cudaFuncSetAttribute(peak_ts_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int iters = 20000;
  long long *cyc;
  CK(cudaMalloc(&cyc, sms * sizeof(long long)));
  peak_ts_kernel<N><<<sms, 128, smem>>>(src, 100, sink, nullptr);
  CK(cudaDeviceSynchronize());
  for (int rep = 0; rep < 3; ++rep) {
    peak_ts_kernel<N><<<sms, 128, smem>>>(src, iters, sink, cyc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(sms);
    CK(cudaMemcpy(c.data(), cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost));
    long long cmax = 0;
    for (auto v : c) cmax = v > cmax ? v : cmax;
    printf("TS (A in TMEM) M=128 N=%3d K=32: %.1f SM clk per MMA (clock64)\n", N, (double)cmax / (34.0 * iters));
  }
  CK(cudaFree(cyc));
}

// CTA pair (cta_group::2): M = 256 (128 rows per CTA), N columns; the leader
// CTA issues, completion multicast to both CTAs' barriers.  Throughput only.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) peak_pair_kernel(const int8_t *src, int iters, long long *cycles) {
  constexpr int kAcc = 512 / N;
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  int8_t *sa = (int8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);  // 7 x 128 x 32
  int8_t *sb = sa + 7 * 128 * 32;                                      // 7 x N x 32
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 7 * (128 + N) * 32; i += blockDim.x) sa[i] = src[(blockIdx.x * 977 + i) & ((1 << 20) - 1)];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (tid == 0) mbar_init(smem_u32(&bar), 1), mbar_fence_init();
  fence_async_smem();
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  tc_fence_after();
  const uint32_t tm = tmem_base;
  long long c0 = clock64();
  if (tid == 0 && rank == 0) {
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    for (int it = 0; it < iters; ++it) {
      int q = 0;
#pragma unroll 1
      for (int i = 0; i < 7; ++i)
#pragma unroll 1
        for (int j = 0; j < 7 && i + j <= 7; ++j, ++q) {
          const uint32_t acc = (it > 0 || q >= kAcc) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + (uint32_t)(((i + j) % kAcc) * N)),
              "l"(umma_desc_k_sw32(a0 + i * 128 * 32)), "l"(umma_desc_k_sw32(b0 + j * N * 32)), "r"(idesc), "r"(acc));
        }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  mbar_wait(smem_u32(&bar), 0);
  if (tid == 0 && cycles) cycles[blockIdx.x] = clock64() - c0;
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

template <int N>
void run_peak_pair(const int8_t *src, int sms) {
  const size_t smem = 1024 + 7 * (128 + N) * 32;
  CK(cudaFuncSetAttribute(peak_pair_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int iters = 20000;
  long long *cyc;
  CK(cudaMalloc(&cyc, sms * sizeof(long long)));
  const int grid = sms & ~1;
  peak_pair_kernel<N><<<grid, 128, smem>>>(src, 100, nullptr);
  CK(cudaDeviceSynchronize());
  for (int rep = 0; rep < 3; ++rep) {
    peak_pair_kernel<N><<<grid, 128, smem>>>(src, iters, cyc);
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(grid);
    CK(cudaMemcpy(c.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));
    long long cmax = 0;
    for (auto v : c) cmax = v > cmax ? v : cmax;
    printf("PAIR cta_group::2 M=256 N=%3d K=32: %.1f SM clk per MMA (clock64) = %.1f clk per 128x%d per SM\n", N,
           (double)cmax / (34.0 * iters), (double)cmax / (34.0 * iters), N);
  }
  CK(cudaFree(cyc));
}

template <int N>
void run_peak(const int8_t *src, int32_t *sink, int sms, int zero) {
  const size_t smem = 1024 + 7 * (128 + N) * 32;
  CK(cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int iters = 20000;
  long long *cyc;
  CK(cudaMalloc(&cyc, sms * sizeof(long long)));
  peak_kernel<N><<<sms, 128, smem>>>(src, 100, sink, nullptr, zero);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    peak_kernel<N><<<sms, 128, smem>>>(src, iters, sink, cyc, zero);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(sms);
    CK(cudaMemcpy(c.data(), cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost));
    long long cmax = 0;
    for (auto v : c) cmax = v > cmax ? v : cmax;
    const double ops = 2.0 * 128 * N * 32 * 34.0 * iters * sms;  // 34 MMAs per iteration (i + j <= 7, i, j < 7)
    printf("M=128 N=%3d K=32 s8*s8->s32 %s: %.3f ms  %.1f TOPS  %.1f SM clk per MMA (clock64), avg clock %.0f MHz\n",
           N, zero ? "zeros " : "random", ms, ops / ms / 1e9, (double)cmax / (34.0 * iters), cmax / (ms * 1e3));
  }
  CK(cudaFree(cyc));
}

// Sustained rate: back-to-back launches of the M128 N256 random-operand
// kernel for `seconds`; the median over the launches after the first second
// (the power-capped steady state the split contraction runs in, bench.py).
void run_sustained(const int8_t *src, int32_t *sink, int sms, double seconds) {
  constexpr int N = 256;
  const size_t smem = 1024 + 7 * (128 + N) * 32;
  CK(cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int iters = 20000;
  long long *cyc;
  CK(cudaMalloc(&cyc, sms * sizeof(long long)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  std::vector<double> tops, mhz;
  double elapsed = 0.0;
  while (elapsed < seconds * 1e3) {
    cudaEventRecord(e0);
    peak_kernel<N><<<sms, 128, smem>>>(src, iters, sink, cyc, 0);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(sms);
    CK(cudaMemcpy(c.data(), cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost));
    long long cmax = 0;
    for (auto v : c) cmax = v > cmax ? v : cmax;
    const double ops = 2.0 * 128 * N * 32 * 34.0 * iters * sms;
    if (elapsed >= 1000.0) {
      tops.push_back(ops / ms / 1e9);
      mhz.push_back(cmax / (ms * 1e3));
    }
    elapsed += ms;
  }
  std::sort(tops.begin(), tops.end());
  std::sort(mhz.begin(), mhz.end());
  printf("SUSTAINED M=128 N=256 K=32 random, %.1f s back to back: median %.1f TOPS (min %.1f, max %.1f) over %zu "
         "launches, median clock %.0f MHz\n",
         seconds, tops[tops.size() / 2], tops.front(), tops.back(), tops.size(), mhz[mhz.size() / 2]);
  CK(cudaFree(cyc));
}

int main(int argc, char **argv) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
  const bool sustain_only = argc > 1 && strcmp(argv[1], "sustain") == 0;
  // (1) correctness, 1..4 accumulated K steps
  srand(7);
  std::vector<int8_t> a(4 * 128 * 32), b(4 * 64 * 32);
  for (auto &x : a) x = (int8_t)(rand() % 255 - 127);
  for (auto &x : b) x = (int8_t)(rand() % 255 - 127);
  int8_t *da, *db;
  int32_t *dd;
  CK(cudaMalloc(&da, a.size()));
  CK(cudaMalloc(&db, b.size()));
  CK(cudaMalloc(&dd, 128 * 64 * 4));
  CK(cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice));
  int bad_total = 0;
  for (int steps = 1; steps <= 4; ++steps) {
    check_kernel<<<1, 128>>>(da, db, steps, dd);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> d(128 * 64);
    CK(cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 64; ++c) {
        int32_t ref = 0;
        for (int s = 0; s < steps; ++s)
          for (int k = 0; k < 32; ++k) ref += (int32_t)a[s * 4096 + r * 32 + k] * (int32_t)b[s * 2048 + c * 32 + k];
        if (ref != d[r * 64 + c] && bad++ < 3) printf("  mismatch r=%d c=%d got %d want %d\n", r, c, d[r * 64 + c], ref);
      }
    printf("check steps=%d: %s (%d mismatches)\n", steps, bad ? "FAIL" : "ok", bad);
    bad_total += bad;
  }
  // (2) throughput
  std::vector<int8_t> r(1 << 20);
  for (auto &x : r) x = (int8_t)(rand() % 255 - 127);
  int8_t *src;
  int32_t *sink;
  CK(cudaMalloc(&src, r.size()));
  CK(cudaMalloc(&sink, 4096));
  CK(cudaMemcpy(src, r.data(), r.size(), cudaMemcpyHostToDevice));
  if (sustain_only) {
    run_sustained(src, sink, p.multiProcessorCount, argc > 2 ? atof(argv[2]) : 5.0);
    return bad_total ? 1 : 0;
  }
  run_peak_pair<128>(src, p.multiProcessorCount);
  run_peak_pair<256>(src, p.multiProcessorCount);
  run_peak_ts<64>(src, sink, p.multiProcessorCount);
  run_peak_ts<128>(src, sink, p.multiProcessorCount);
  for (int zero = 0; zero < 2; ++zero) {
    run_peak<64>(src, sink, p.multiProcessorCount, zero);
    run_peak<128>(src, sink, p.multiProcessorCount, zero);
    run_peak<256>(src, sink, p.multiProcessorCount, zero);
  }
  return bad_total ? 1 : 0;
}
