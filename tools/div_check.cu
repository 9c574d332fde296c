// Is q = fma(fma(-RN(a*y), b, a), y, RN(a*y)) with y = RN(1/b) bit-identical to
// IEEE a / b (__ddiv_rn)?  (Markstein's correction step; guarded to exponent
// ranges where no intermediate underflows.)  Random a, b over several ranges.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/div_check tools/div_check.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; return x ^ (x >> 31);
}
__device__ __forceinline__ double fast_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double e = __fma_rn(-q0, b, a);
  return __fma_rn(e, y, q0);
}

__global__ void k(uint64_t seed, long iters, int mode, unsigned long long *bad, unsigned long long *cnt, double *ex) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long nb = 0, nc = 0;
  for (long i = 0; i < iters; ++i) {
    const uint64_t r1 = mix(seed ^ (tid * 0x9E3779B97F4A7C15ull + i)), r2 = mix(r1 + 0x1234567ull);
    double a, b;
    if (mode == 0) {  // a, b uniform mantissas, exponents around 1
      a = __longlong_as_double((long long)((r1 & 0x000FFFFFFFFFFFFFull) | (0x3FEull + (r1 >> 60)) << 52));
      b = __longlong_as_double((long long)((r2 & 0x000FFFFFFFFFFFFFull) | (0x3FEull + (r2 >> 61)) << 52));
      if (r1 & (1ull << 59)) a = -a;
    } else if (mode == 1) {  // wide exponents, |a| <= b as in (x - mean) / sqrt(ssd)
      const int ea = 1023 - 600 + (int)((r1 >> 52) % 1100), eb = 1023 - 450 + (int)((r2 >> 52) % 900);
      a = __longlong_as_double((long long)((r1 & 0x000FFFFFFFFFFFFFull) | ((uint64_t)ea << 52)));
      b = __longlong_as_double((long long)((r2 & 0x000FFFFFFFFFFFFFull) | ((uint64_t)eb << 52)));
      if (r2 & 1) a = -a;
    } else {  // b = sqrt(s), a = small integers / mantissa-poor values (data-like)
      b = __dsqrt_rn((double)(r2 % 100000000ull + 1) * 0.001);
      a = ((double)(long long)(r1 % 20001) - 10000.0) * 0.0625;
    }
    const double y = __drcp_rn(b);
    const double q = fast_div(a, b, y), ref = __ddiv_rn(a, b);
    ++nc;
    if (__double_as_longlong(q) != __double_as_longlong(ref)) {
      if (nb == 0) { ex[0] = a; ex[1] = b; }
      ++nb;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(cnt, nc);
}

int main() {
  unsigned long long *bad, *cnt;
  double *ex;
  cudaMalloc(&bad, 8); cudaMalloc(&cnt, 8); cudaMalloc(&ex, 16);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(bad, 0, 8); cudaMemset(cnt, 0, 8);
    for (int rep = 0; rep < 8; ++rep) k<<<148 * 8, 256, 0>>>(1000 + rep * 7919 + mode, 4096, mode, bad, cnt, ex);
    unsigned long long b = 0, c = 0; double e[2] = {0, 0};
    cudaMemcpy(&b, bad, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&c, cnt, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(e, ex, 16, cudaMemcpyDeviceToHost);
    printf("mode %d: %llu mismatches of %llu  (first: a=%.17g b=%.17g)  %s\n", mode, b, c, e[0], e[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
