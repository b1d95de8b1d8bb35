// gemm.cu -- K7 dense FP64 product of decompressed operand tiles.
//
// mat_mul_impl (H/matrix.hpp:204-217) accumulates every output entry as
// acc = 0.0; acc += a(i,k) * b(k,j) over the global inner index k ascending
// (accumulate_product_tile, :188-202), padding excluded (k < a.cols).
//
//  * BLZ_GEMM_EXACT -- k_gemm_simt<false>: CUDA-core DMUL + DADD (this TU is built
//    with -fmad=false) in exactly that order: bitwise equal to the reference.
//    Tiles beyond K are zero-filled: adding +0.0 to a running sum that starts
//    at +0.0 (and is therefore never -0.0) is the identity.
//  * BLZ_GEMM_FUSED -- acc = fma(a(i,k), b(k,j), acc), k ascending, from +0.0:
//    deterministic, tolerance parity against the exact product.  Two kernels
//    compute this chain bitwise identically (tests/test_gpu_parity.py checks):
//      k_gemm_simt<true> (BLZ_GEMM_FUSED_DFMA): the SIMT kernel with DFMA;
//      k_gemm_dmma2 (BLZ_GEMM_FUSED_DMMA): FP64 tensor cores (mma.sync m8n8k4
//      f64).  On B200 one DMMA equals the ascending-k chain of fused
//      multiply-adds (tools/microbench/dmma_semantics.cu: 0 mismatches in 1.28M
//      entries).
//    BLZ_GEMM_FUSED runs FUSED_KERNEL_DEFAULT, the faster of the two on B200
//    (K7, profiles/r02_ncu_summary.md).
#include <cuda_pipeline_primitives.h>

#include "launch.h"

namespace blz {

// ---------------------------------------------------------------------------
// exact SIMT DGEMM (and its DFMA twin), ascending k, operands staged with
// cp.async; a warp reads 2 rows of A per k (broadcast) and 256 contiguous bytes
// of a B row.
// ---------------------------------------------------------------------------
constexpr int EBK = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  __pipeline_memcpy_async(smem, gmem, 16);
}

// FMA = false: acc + a*b as DMUL then DADD (-fmad=false); true: one DFMA.
// The accumulators start from C when acc_c (a K-panel continuing the chain of
// the previous panels: storing and reloading a double is exact, so the
// per-entry operation sequence is the single-pass one); otherwise from +0.0.
// CTA tile 128 x 64 (128 threads, 8 x 8 outputs each), BK = 16, four cp.async
// stages, two CTAs per SM.  Measured at 8192^3 (TFLOP/s, exact / DFMA): 128x128
// two stages (round 1) 15.3 / 23.2; 128x64 three stages 15.8 / 24.0, four 16.2 /
// 24.8; 64x128 four 15.7 / 24.0; 128x128 three 15.2 / 23.1; 64x64 two / three
// stages (four CTAs per SM) 13.6 / 14.5 exact.
constexpr int SBM = 128, SBN = 64, STHREADS = SBM * SBN / 64, SSTAGES = 4;
constexpr int SSTAGE = SBM * EBK + EBK * SBN;
template <bool FMA>
__global__ void __launch_bounds__(STHREADS, 2) k_gemm_simt(const double* __restrict__ A, uint64_t lda,
                                                             const double* __restrict__ Bm, uint64_t ldb,
                                                             double* __restrict__ Cm, uint64_t ldc, uint64_t M,
                                                             uint64_t N, uint64_t K, bool acc_c) {
  extern __shared__ __align__(16) double esm[];
  const int tid = threadIdx.x;
  const int tx = tid % (SBN / 8), ty = tid / (SBN / 8);
  const uint64_t m0 = (uint64_t)blockIdx.y * SBM, n0 = (uint64_t)blockIdx.x * SBN;
  const bool vecA = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool vecB = ((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(Bm) & 15) == 0);
  auto load_tile = [&](int st, uint64_t k0) {
    double* As = esm + st * SSTAGE;
    double* Bs = As + SBM * EBK;
#pragma unroll
    for (int r = 0; r < SBM * 8 / STHREADS; ++r) {
      const int e = tid + r * STHREADS;
      const int row = e >> 3, kc = (e & 7) * 2;
      const uint64_t gr = m0 + row, gk = k0 + kc;
      double* dst = &As[row * EBK + kc];
      if (gr < M && gk + 1 < K && vecA) {
        cp_async16(dst, A + gr * lda + gk);
      } else {
        dst[0] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.0;
        dst[1] = (gr < M && gk + 1 < K) ? A[gr * lda + gk + 1] : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < 8 * SBN / STHREADS; ++r) {
      const int e = tid + r * STHREADS;
      const int kr = e / (SBN / 2), cc = (e % (SBN / 2)) * 2;
      const uint64_t gk = k0 + kr, gc = n0 + cc;
      double* dst = &Bs[kr * SBN + cc];
      if (gk < K && gc + 1 < N && vecB) {
        cp_async16(dst, Bm + gk * ldb + gc);
      } else {
        dst[0] = (gk < K && gc < N) ? Bm[gk * ldb + gc] : 0.0;
        dst[1] = (gk < K && gc + 1 < N) ? Bm[gk * ldb + gc + 1] : 0.0;
      }
    }
  };
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t gr = m0 + ty * 8 + i, gc = n0 + (j / 2) * (SBN / 4) + 2 * tx + (j % 2);
      acc[i][j] = (acc_c && gr < M && gc < N) ? Cm[gr * ldc + gc] : 0.0;
    }
  const uint64_t ntiles = (K + EBK - 1) / EBK;
#pragma unroll
  for (int st = 0; st < SSTAGES - 1; ++st) {
    if ((uint64_t)st < ntiles) load_tile(st, (uint64_t)st * EBK);
    __pipeline_commit();
  }
  for (uint64_t kt = 0; kt < ntiles; ++kt) {
    __pipeline_wait_prior(SSTAGES - 2);
    __syncthreads();
    const uint64_t nt = kt + SSTAGES - 1;
    if (nt < ntiles) load_tile((int)(nt % SSTAGES), nt * EBK);
    __pipeline_commit();
    const double* As = esm + (int)(kt % SSTAGES) * SSTAGE;
    const double* Bs = As + SBM * EBK;
#pragma unroll
    for (int kk = 0; kk < EBK; kk += 2) {
      double2 av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = *reinterpret_cast<const double2*>(&As[(ty * 8 + i) * EBK + kk]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double bv[8];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(&Bs[(kk + h) * SBN + (j / 2) * (SBN / 4) + 2 * tx]);
          bv[j] = v.x;
          bv[j + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double a = h ? av[i].y : av[i].x;
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = FMA ? fma(a, bv[j], acc[i][j]) : acc[i][j] + a * bv[j];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t gr = m0 + ty * 8 + i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t gc = n0 + (j / 2) * (SBN / 4) + 2 * tx + (j % 2);
      if (gc < N) Cm[gr * ldc + gc] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// fused DGEMM on FP64 tensor cores, small tiles and a deep pipeline (the shape
// cuBLAS's DGEMM picks on this GPU): CTA tile 64 x 64, BK = 16, 4 cp.async
// stages, 4 warps (2 x 2, each 32 x 32 = 4 x 4 MMA tiles), several CTAs per SM.
// Same ascending-k FMA chain per output as k_gemm_simt<true> (bitwise equal
// results).  90 % of the DMMA peak at 8192^3 against 80-82 % for the round-1
// kernel (128 x 128 tile, BK = 32, two stages, one CTA per SM).
// ---------------------------------------------------------------------------
#ifndef G2_STAGES
#define G2_STAGES 4
#endif
// measured at 8192^3 (TFLOP/s): 64x32x16 / 3-6 stages 32.2, 31.5, 32.1, 29.7; 64x64x16 / 3 31.5, / 4 33.0
// (also with 2 CTAs/SM forced: 33.0), / 5-6 31.4;
// 64x128x16 / 4 32.1; 128x32x16 / 3 30.5; 128x64x16 / 4 22.0; 64x32x32 / 3 29.5; 64x64x8 / 8 32.3;
// XOR-swizzled unpadded tiles 32.9; grouped raster orders (4 / 8 / 16 tile-rows) 30.7; the round-1
// 128x128x32 two-stage kernel 29.3; register double-buffered fragments with the next tile's barrier
// before the last k-step 31.5 (184 regs, 2 CTAs/SM) / 32.4 (capped to 3 CTAs/SM); cuBLAS DGEMM 35.5
#ifndef G2_TM
#define G2_TM 64
#endif
#ifndef G2_TN
#define G2_TN 64
#endif
#ifndef G2_TK
#define G2_TK 16
#endif
#ifndef G2_MINB
#define G2_MINB 1
#endif
constexpr int G2M = G2_TM, G2N = G2_TN, G2K = G2_TK;
constexpr int G2MI = G2M / 16, G2NJ = G2N / 16;  // MMA tiles per warp (2 x 2 warps)
constexpr int G2A_CHUNKS = G2M * G2K / 2 / 128, G2B_CHUNKS = G2K * G2N / 2 / 128;
// rows padded by 4 doubles (4 mod 16): the fragment loads of a quarter-warp hit distinct banks
constexpr int G2AS = G2K + 4;  // As[m][k] row stride
constexpr int G2BS = G2N + 4;  // Bs[k][n] row stride
__device__ __forceinline__ int g2a(int row, int k) { return row * G2AS + k; }
__device__ __forceinline__ int g2b(int k, int col) { return k * G2BS + col; }
constexpr int G2_STAGE_DOUBLES = G2M * G2AS + G2K * G2BS;

__global__ void __launch_bounds__(128, G2_MINB) k_gemm_dmma2(const double* __restrict__ A, uint64_t lda,
                                                    const double* __restrict__ Bm, uint64_t ldb,
                                                    double* __restrict__ Cm, uint64_t ldc, uint64_t M,
                                                    uint64_t N, uint64_t K, bool acc_c) {
  extern __shared__ __align__(16) double g2sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // warp tile rows wm*32.., cols wn*16..
  const uint64_t m0 = (uint64_t)blockIdx.y * G2M, n0 = (uint64_t)blockIdx.x * G2N;
  const bool vecA = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool vecB = ((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(Bm) & 15) == 0);

  auto load_tile = [&](int stage, uint64_t k0) {
    double* As = g2sm + stage * G2_STAGE_DOUBLES;
    double* Bs = As + G2M * G2AS;
    // A: G2M rows x G2K k in 16-byte chunks
#pragma unroll
    for (int r = 0; r < G2A_CHUNKS; ++r) {
      const int e = tid + r * 128;
      const int row = e / (G2K / 2), kc = (e % (G2K / 2)) * 2;
      const uint64_t gr = m0 + row, gk = k0 + kc;
      double* dst = As + g2a(row, kc);
      if (vecA && gr < M && gk + 1 < K) {
        cp_async16(dst, A + gr * lda + gk);
      } else {
        dst[0] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.0;
        dst[1] = (gr < M && gk + 1 < K) ? A[gr * lda + gk + 1] : 0.0;
      }
    }
    // B: G2K k x G2N cols in 16-byte chunks
#pragma unroll
    for (int r = 0; r < G2B_CHUNKS; ++r) {
      const int e = tid + r * 128;
      const int kr = e / (G2N / 2), cc = (e % (G2N / 2)) * 2;
      const uint64_t gk = k0 + kr, gc = n0 + cc;
      double* dst = Bs + g2b(kr, cc);
      if (vecB && gk < K && gc + 1 < N) {
        cp_async16(dst, Bm + gk * ldb + gc);
      } else {
        dst[0] = (gk < K && gc < N) ? Bm[gk * ldb + gc] : 0.0;
        dst[1] = (gk < K && gc + 1 < N) ? Bm[gk * ldb + gc + 1] : 0.0;
      }
    }
  };

  double acc[G2MI][G2NJ][2];
#pragma unroll
  for (int i = 0; i < G2MI; ++i)
#pragma unroll
    for (int j = 0; j < G2NJ; ++j) {  // D fragment: row = lane>>2, cols = (lane&3)*2 + {0,1}
      const uint64_t gr = m0 + wm * (G2M / 2) + i * 8 + (lane >> 2);
      const uint64_t gc = n0 + wn * (G2N / 2) + j * 8 + (lane & 3) * 2;
      acc[i][j][0] = (acc_c && gr < M && gc < N) ? Cm[gr * ldc + gc] : 0.0;
      acc[i][j][1] = (acc_c && gr < M && gc + 1 < N) ? Cm[gr * ldc + gc + 1] : 0.0;
    }

  const uint64_t ntiles = (K + G2K - 1) / G2K;
#pragma unroll
  for (int st = 0; st < G2_STAGES - 1; ++st) {
    if ((uint64_t)st < ntiles) load_tile(st, (uint64_t)st * G2K);
    __pipeline_commit();
  }
  for (uint64_t kt = 0; kt < ntiles; ++kt) {
    __pipeline_wait_prior(G2_STAGES - 2);  // tile kt has landed (this thread's copies)
    __syncthreads();                        // ... everyone's; and tile kt-1's stage is free
    const uint64_t nt = kt + G2_STAGES - 1;
    if (nt < ntiles) load_tile((int)(nt % G2_STAGES), nt * G2K);
    __pipeline_commit();
    const double* As = g2sm + (int)(kt % G2_STAGES) * G2_STAGE_DOUBLES;
    const double* Bs = As + G2M * G2AS;
#pragma unroll
    for (int ks = 0; ks < G2K; ks += 4) {
      double fa[G2MI], fb[G2NJ];
#pragma unroll
      for (int i = 0; i < G2MI; ++i) fa[i] = As[g2a(wm * (G2M / 2) + i * 8 + (lane >> 2), ks + (lane & 3))];
#pragma unroll
      for (int j = 0; j < G2NJ; ++j) fb[j] = Bs[g2b(ks + (lane & 3), wn * (G2N / 2) + j * 8 + (lane >> 2))];
#pragma unroll
      for (int i = 0; i < G2MI; ++i)
#pragma unroll
        for (int j = 0; j < G2NJ; ++j)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
              : "d"(fa[i]), "d"(fb[j]));
    }
  }
#pragma unroll
  for (int i = 0; i < G2MI; ++i)
#pragma unroll
    for (int j = 0; j < G2NJ; ++j) {
      const uint64_t gr = m0 + wm * (G2M / 2) + i * 8 + (lane >> 2);
      const uint64_t gc = n0 + wn * (G2N / 2) + j * 8 + (lane & 3) * 2;
      if (gr < M) {
        if (gc < N) Cm[gr * ldc + gc] = acc[i][j][0];
        if (gc + 1 < N) Cm[gr * ldc + gc + 1] = acc[i][j][1];
      }
    }
}

#ifndef FUSED_KERNEL_DEFAULT
#define FUSED_KERNEL_DEFAULT 2  // BLZ_GEMM_FUSED_DMMA
#endif

cudaError_t launch_gemm(const LaunchCtx& c, int mode, const double* A, uint64_t lda, const double* Bm,
                        uint64_t ldb, double* Cm, uint64_t ldc, uint64_t M, uint64_t N, uint64_t K, bool acc_c) {
  if (mode == 1) mode = FUSED_KERNEL_DEFAULT;
  // per call: the smem attribute belongs to the current device (a few microseconds
  // against a GEMM of milliseconds)
  if (mode == 2) {
    dim3 grid((unsigned)((N + G2N - 1) / G2N), (unsigned)((M + G2M - 1) / G2M));
    const size_t smem = (size_t)G2_STAGES * G2_STAGE_DOUBLES * sizeof(double);
    cudaError_t ea = cudaFuncSetAttribute(k_gemm_dmma2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
    k_gemm_dmma2<<<grid, 128, smem, c.stream>>>(A, lda, Bm, ldb, Cm, ldc, M, N, K, acc_c);
  } else {
    dim3 grid((unsigned)((N + SBN - 1) / SBN), (unsigned)((M + SBM - 1) / SBM));
    const size_t smem = (size_t)SSTAGES * SSTAGE * sizeof(double);
    auto kern = mode == 3 ? k_gemm_simt<true> : k_gemm_simt<false>;
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
    kern<<<grid, STHREADS, smem, c.stream>>>(A, lda, Bm, ldb, Cm, ldc, M, N, K, acc_c);
  }
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
