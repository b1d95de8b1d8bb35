// gemm.cu -- K7 dense FP64 product of decompressed operand tiles.
//
// mat_mul_impl (H/matrix.hpp:204-217) accumulates every output entry as
// acc = 0.0; acc += a(i,k) * b(k,j) over the global inner index k ascending
// (accumulate_product_tile, :188-202), padding excluded (k < a.cols).
// Exact mode keeps that order with DMUL+DADD (this TU is built with
// -fmad=false); fused mode uses DFMA in the same order (tolerance parity).
#include "launch.h"

namespace blz {

constexpr int GBM = 64, GBN = 64, GBK = 16, GTM = 4, GTN = 4;

template <bool FUSED>
__global__ void __launch_bounds__(256) k_gemm(const double* __restrict__ A, uint64_t lda,
                                              const double* __restrict__ Bm, uint64_t ldb,
                                              double* __restrict__ Cm, uint64_t ldc, uint64_t M,
                                              uint64_t N, uint64_t K) {
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const uint64_t m0 = (uint64_t)blockIdx.y * GBM, n0 = (uint64_t)blockIdx.x * GBN;
  double acc[GTM][GTN];
#pragma unroll
  for (int i = 0; i < GTM; ++i)
#pragma unroll
    for (int j = 0; j < GTN; ++j) acc[i][j] = 0.0;

  for (uint64_t k0 = 0; k0 < K; k0 += GBK) {
    // A tile: GBM x GBK (transposed into smem), B tile: GBK x GBN
    for (int e = threadIdx.x; e < GBM * GBK; e += 256) {
      const int r = e / GBK, kk = e % GBK;
      const uint64_t gr = m0 + r, gk = k0 + kk;
      As[kk][r] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < GBK * GBN; e += 256) {
      const int kk = e / GBN, cc = e % GBN;
      const uint64_t gk = k0 + kk, gc = n0 + cc;
      Bs[kk][cc] = (gk < K && gc < N) ? Bm[gk * ldb + gc] : 0.0;
    }
    __syncthreads();
    const int kmax = (K - k0) < (uint64_t)GBK ? (int)(K - k0) : GBK;
    for (int kk = 0; kk < kmax; ++kk) {
      double av[GTM], bv[GTN];
#pragma unroll
      for (int i = 0; i < GTM; ++i) av[i] = As[kk][ty * GTM + i];
#pragma unroll
      for (int j = 0; j < GTN; ++j) bv[j] = Bs[kk][tx * GTN + j];
#pragma unroll
      for (int i = 0; i < GTM; ++i)
#pragma unroll
        for (int j = 0; j < GTN; ++j) {
          if (FUSED)
            acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
          else
            acc[i][j] = acc[i][j] + av[i] * bv[j];
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < GTM; ++i)
#pragma unroll
    for (int j = 0; j < GTN; ++j) {
      const uint64_t gr = m0 + ty * GTM + i, gc = n0 + tx * GTN + j;
      if (gr < M && gc < N) Cm[gr * ldc + gc] = acc[i][j];
    }
}

cudaError_t launch_gemm(const LaunchCtx& c, int mode, const double* A, uint64_t lda, const double* Bm,
                        uint64_t ldb, double* Cm, uint64_t ldc, uint64_t M, uint64_t N, uint64_t K) {
  dim3 grid((unsigned)((N + GBN - 1) / GBN), (unsigned)((M + GBM - 1) / GBM));
  if (mode == 1)
    k_gemm<true><<<grid, 256, 0, c.stream>>>(A, lda, Bm, ldb, Cm, ldc, M, N, K);
  else
    k_gemm<false><<<grid, 256, 0, c.stream>>>(A, lda, Bm, ldb, Cm, ldc, M, N, K);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
