// Dependent-chain latency of DADD / DMUL / DFMA and of a constant-bank load feeding a DMUL
// on B200 (one warp, clock64).  Evidence for the decompress analysis in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

struct Basis { double t[64]; };

template <int OP>
__global__ void k_chain(double* out, long long* cyc, double a, double b, int n, const Basis B) {
  double x = a + threadIdx.x * 1e-9;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __dadd_rn(x, b);
      else if (OP == 1) x = __dmul_rn(x, b);
      else if (OP == 2) x = __fma_rn(x, b, a);
      else x = __dmul_rn(x, B.t[(i + k) & 63]);  // constant-bank operand on the chain
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.0) *out = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMallocManaged(&cyc, 8);
  Basis B;
  for (int i = 0; i < 64; ++i) B.t[i] = 1.0 + i * 1e-12;
  const int n = 4096;
  const char* names[4] = {"DADD", "DMUL", "DFMA", "DMUL(c[] operand via LDC)"};
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) k_chain<0><<<1, 32>>>(out, cyc, 1.0, 1e-9, n, B);
      if (op == 1) k_chain<1><<<1, 32>>>(out, cyc, 1.0, 1.0000001, n, B);
      if (op == 2) k_chain<2><<<1, 32>>>(out, cyc, 1.0, 0.999, n, B);
      if (op == 3) k_chain<3><<<1, 32>>>(out, cyc, 1.0, 1.0, n, B);
      cudaDeviceSynchronize();
    }
    printf("%-28s %.2f cycles per dependent op\n", names[op], (double)*cyc / (16.0 * n));
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
