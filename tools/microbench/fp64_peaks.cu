// FP64 pipe microbenchmarks for B200 (sm_100a): DADD, DMUL, DFMA, DMMA m8n8k4,
// F2I.S64 / I2F.F64 conversions. Prints ops/clk/SM and Tops/s. Evidence for DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
#define CHAINS 8

template <int OP>
__global__ void k_fp64(double* out, double a, double b, int iters) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = a + threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) x[c] = __dadd_rn(x[c], b);
      else if (OP == 1) x[c] = __dmul_rn(x[c], b);
      else x[c] = __fma_rn(x[c], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_cvt(double* out, double a, int iters) {
  double x[CHAINS];
  long long acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = a + threadIdx.x + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      long long t = __double2ll_rz(x[c]);
      x[c] = __ll2double_rn(t + 1);
    }
  }
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc += (long long)x[c];
  if (acc == 12345) out[0] = acc;
}

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock(max) %d MHz\n", p.name, p.multiProcessorCount, clk_khz / 1000);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  double best[3] = {0, 0, 0}, best_dmma = 0, copy_gbs = 0;
  for (int threads : {128, 256, 512}) {
    for (int op = 0; op < 3; ++op) {
      int blocks = sms * (2048 / threads);
      auto launch = [&]() {
        if (op == 0) k_fp64<0><<<blocks, threads>>>(out, 1.0, 1.0000001, N_ITER);
        if (op == 1) k_fp64<1><<<blocks, threads>>>(out, 1.0, 1.0000001, N_ITER);
        if (op == 2) k_fp64<2><<<blocks, threads>>>(out, 1e-3, 0.9999999, N_ITER);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * N_ITER * CHAINS;
      printf("%s threads/blk %d: %.3f ms  %.2f Tops/s  (%.1f ops/clk/SM at %d MHz)\n", names[op], threads, ms,
             ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
      if (ops / ms / 1e9 > best[op]) best[op] = ops / ms / 1e9;
    }
  }
  {
    int threads = 256, blocks = sms * 8;
    k_cvt<<<blocks, threads>>>(out, 1.5, N_ITER / 4); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_cvt<<<blocks, threads>>>(out, 1.5, N_ITER / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * (N_ITER / 4) * CHAINS;
    printf("F2I.S64+I2F pair: %.3f ms %.2f Gpairs/s (%.2f pairs/clk/SM)\n", ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk_khz * 1e3));
  }
  for (int threads : {128, 256}) {
    int blocks = sms * (1024 / threads);
    k_dmma<<<blocks, threads>>>(out, N_ITER / 4); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(out, N_ITER / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = (double)blocks * (threads / 32) * (N_ITER / 4) * CHAINS * 8 * 8 * 4 * 2;
    printf("DMMA m8n8k4 threads %d: %.3f ms %.2f TFLOP/s\n", threads, ms, flops / ms / 1e9);
    if (flops / ms / 1e9 > best_dmma) best_dmma = flops / ms / 1e9;
  }
  {
    size_t bytes = 4ull << 30; double2 *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    size_t n = bytes / 16;
    for (int r = 0; r < 2; ++r) k_copy<<<sms * 8, 512>>>(a, b, n);
    cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) k_copy<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    copy_gbs = 5.0 * 2 * bytes / (ms * 1e-3) / 1e9;
    printf("copy 4GiB: %.1f GB/s (read+write)\n", copy_gbs);
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  // machine-readable line (bench.py reads it): FP64 pipe ops/s and FLOP/s peaks
  printf("{\"dadd_tops\": %.3f, \"dmul_tops\": %.3f, \"dfma_tops\": %.3f, \"dfma_tflops\": %.3f, "
         "\"dmma_tflops\": %.3f, \"copy_gbs\": %.1f, \"sm_clock_max_mhz\": %d, \"ok\": %s}\n",
         best[0], best[1], best[2], 2 * best[2], best_dmma, copy_gbs, clk_khz / 1000,
         err == cudaSuccess ? "true" : "false");
  return 0;
}
