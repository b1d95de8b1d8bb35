// Checks the add / sub weight divisions (csrc/combine.cuh, ASB_DIV): with
// y = RN(1/b) (IEEE 1.0 / b), q = RN(a y), e = fma(-b, q, a), RN(q + e y) must
// equal the IEEE quotient a / b.  Cases: every b = p in 1..255 against random a
// (random significands, all-ones / all-zeros significands, both signs) over
// the guarded range |a| in [2^-800, 2^800]; and random b, a both in
// [2^-400, 2^400] (the divisions by s = s1 + s2).  Prints the mismatch counts.
//   make -C tools/microbench markstein_check && tools/microbench/markstein_check
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x *= 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 32;
  return x;
}

__device__ __forceinline__ double make(uint64_t x, int emin, int emax, uint64_t i) {
  uint64_t mant = x & 0xFFFFFFFFFFFFFull;
  if ((i & 255) == 0) mant = 0xFFFFFFFFFFFFFull;
  if ((i & 255) == 1) mant = 0;
  if ((i & 255) == 2) mant = 0xFFFFFFFFFFFFEull;
  const int64_t e = 1023 + emin + (int64_t)((x >> 52) % (uint64_t)(emax - emin + 1));
  const uint64_t sign = (x >> 11) & 1;
  return __longlong_as_double((int64_t)((sign << 63) | ((uint64_t)e << 52) | mant));
}

__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double e = fma(-b, q, a);
  return fma(e, y, q);
}

__global__ void k_small(uint64_t seed, uint64_t n, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double a = make(mix(i + seed), -800, 800, i >> 8);
    const double b = (double)(1 + (i % 255));
    const double y = 1.0 / b;
    const double q = div_rcp(a, b, y);
    if (__double_as_longlong(q) != __double_as_longlong(a / b)) atomicAdd(bad, 1ull);
  }
}

__global__ void k_wide(uint64_t seed, uint64_t n, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = mix(i + seed);
    const double a = make(x, -400, 400, i);
    const double b = fabs(make(mix(x ^ 0x5555), -400, 400, i >> 3));
    const double y = 1.0 / b;
    const double q = div_rcp(a, b, y);
    if (__double_as_longlong(q) != __double_as_longlong(a / b)) atomicAdd(bad, 1ull);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const uint64_t n = 1ull << 33;
  k_small<<<148 * 16, 256>>>(1, n, d);
  k_wide<<<148 * 16, 256>>>(7, n, d + 1);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  printf("{\"markstein_u8_divisor\": {\"samples\": %llu, \"mismatches\": %llu}, "
         "\"markstein_wide\": {\"samples\": %llu, \"mismatches\": %llu}, \"cuda\": \"%s\"}\n",
         (unsigned long long)n, h[0], (unsigned long long)n, h[1], cudaGetErrorString(e));
  return (h[0] || h[1] || e != cudaSuccess) ? 1 : 0;
}
