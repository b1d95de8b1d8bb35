// Conversion throughput on B200 (sm_100a): I2F.F64.S32, I2F.F64.S16 (int8/int16 sources),
// and the magic-constant alternative (integer add into the low word + one DADD).
// Prints conversions/clk/SM.  Evidence for the compress kernel's conversion budget.
#include <cstdio>
#include <cuda_runtime.h>
#define CHAINS 8

template <int MODE>
__global__ void k_cvt(unsigned* out, int seed, int iters) {
  int n[CHAINS];
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) n[c] = seed + threadIdx.x * 3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      double d;
      if (MODE == 0) d = (double)(n[c] + it);                 // I2F.F64.S32
      else if (MODE == 1) d = (double)(short)(n[c] + it);     // I2F.F64.S16
      else d = __hiloint2double(0x43300000, (n[c] + it) ^ 0x80000000) - 4503601774854144.0;  // magic
      acc ^= __double2hiint(d) + __double2loint(d);
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned* out;
  cudaMalloc(&out, 4);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  const char* names[3] = {"I2F.F64.S32", "I2F.F64.S16", "magic IADD+DADD"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k_cvt<0><<<blocks, threads>>>(out, 1, iters);
      else if (mode == 1) k_cvt<1><<<blocks, threads>>>(out, 1, iters);
      else k_cvt<2><<<blocks, threads>>>(out, 1, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * threads * iters * CHAINS;
    printf("%-18s %.3f ms  %.2f cvt/clk/SM (at %d MHz)\n", names[mode], ms, n / (ms * 1e-3) / (clk * 1e3) / sms,
           clk / 1000);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
