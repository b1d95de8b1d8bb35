// Checks the rounding semantics of mma.sync.m8n8k4.f64 (DMMA) on B200 against
// host-side candidates: an ascending-k chain of fused multiply-adds
// d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))), the descending chain,
// and a non-fused chain.  Prints mismatch counts over many random tiles.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* D, int tiles) {
  int lane = threadIdx.x;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const double* a = A + t * 32;  // 8x4 row-major
    const double* b = B + t * 32;  // 4x8 row-major
    const double* c = C + t * 64;  // 8x8
    double* d = D + t * 64;
    double fa = a[(lane >> 2) * 4 + (lane & 3)];
    double fb = b[(lane & 3) * 8 + (lane >> 2)];
    int r = lane >> 2, c0 = (lane & 3) * 2;
    double d0 = c[r * 8 + c0], d1 = c[r * 8 + c0 + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(fa), "d"(fb));
    d[r * 8 + c0] = d0;
    d[r * 8 + c0 + 1] = d1;
  }
}

int main() {
  const int T = 20000;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  std::vector<double> A(T * 32), B(T * 32), C(T * 64), D(T * 64);
  for (auto& x : A) x = u(rng) * std::pow(10.0, (int)(rng() % 7) - 3);
  for (auto& x : B) x = u(rng) * std::pow(10.0, (int)(rng() % 7) - 3);
  for (auto& x : C) x = u(rng) * std::pow(10.0, (int)(rng() % 7) - 3);
  double *dA, *dB, *dC, *dD;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dB, B.size() * 8); cudaMalloc(&dC, C.size() * 8); cudaMalloc(&dD, D.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice);
  k<<<256, 32>>>(dA, dB, dC, dD, T);
  cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost);
  long asc = 0, desc = 0, nonf = 0, any_ok = 0, n = 0;
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        const double* a = &A[t * 32 + i * 4];
        double bb[4];
        for (int k2 = 0; k2 < 4; ++k2) bb[k2] = B[t * 32 + k2 * 8 + j];
        double c = C[t * 64 + i * 8 + j], g = D[t * 64 + i * 8 + j];
        double x = c;
        for (int k2 = 0; k2 < 4; ++k2) x = std::fma(a[k2], bb[k2], x);
        double y = c;
        for (int k2 = 3; k2 >= 0; --k2) y = std::fma(a[k2], bb[k2], y);
        volatile double z = c;
        for (int k2 = 0; k2 < 4; ++k2) { volatile double p = a[k2] * bb[k2]; z = z + p; }
        asc += (x != g); desc += (y != g); nonf += ((double)z != g);
        any_ok += (x == g || y == g);
        ++n;
      }
  printf("DMMA m8n8k4 vs host: %ld entries; mismatches ascending-fma %ld, descending-fma %ld, non-fused %ld, neither-chain %ld\n",
         n, asc, desc, nonf, n - any_ok);
  return 0;
}
