// Checks that rcp.approx.ftz.f64 + two Newton steps (compress_pair.cu::rcp_faithful)
// is within one ulp of the correctly rounded 1/a: random significands (and the
// all-ones / all-zeros ones) over exponents -960..976.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rcp_check rcp_check.cu && /tmp/rcp_check
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double rcp_faithful(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  return fma(y, e, y);
}

__global__ void k(uint64_t seed, uint64_t n, unsigned long long* bad, unsigned long long* notrn) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = (i + seed) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    uint64_t mant = x & 0xFFFFFFFFFFFFFull;
    if ((i & 1023) == 0) mant = 0xFFFFFFFFFFFFFull;
    if ((i & 1023) == 1) mant = 0;
    const int64_t e = 1023 - 960 + (int64_t)((x >> 52) % 1937);
    const double a = __longlong_as_double((int64_t)(((uint64_t)e << 52) | mant));
    const double y = rcp_faithful(a), r = 1.0 / a;
    const int64_t d = __double_as_longlong(y) - __double_as_longlong(r);
    if (d != 0) atomicAdd(notrn, 1ull);
    if (d > 1 || d < -1) atomicAdd(bad, 1ull);
  }
}

int main() {
  unsigned long long *bad, *notrn;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&notrn, 8);
  *bad = 0;
  *notrn = 0;
  const uint64_t n = 1ull << 32;
  k<<<148 * 16, 256>>>(12345, n, bad, notrn);
  cudaDeviceSynchronize();
  printf("rcp_faithful: %llu samples, %llu not correctly rounded, %llu beyond one ulp\n",
         (unsigned long long)n, *notrn, *bad);
  return *bad != 0;
}
