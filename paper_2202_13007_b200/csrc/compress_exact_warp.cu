// compress_exact_warp.cu -- exact compress_block (H/codec.hpp:130-146) with
// one WARP per block, for the verified path's worklist.
//
// The worklist holds the few blocks whose fast-path decisions were not
// certified (a handful per million).  Run one-thread-per-block, each of them is
// a ~3,000-operation dependent chain (~70 us of pure latency); a warp cuts
// that to a few microseconds.  Every value is computed with exactly the
// reference's operations and order (this TU is built with -fmad=false):
//   lane L owns cells L and L + 32 for the elementwise stages, the |delta| sum
//   is one serial chain in row-major order, the DCT outputs are 8-term
//   ascending chains (the reference's acc = 0.0; acc += t*x), reductions are
//   max (order-independent) or exact integer counts.
#include "blaz_device.cuh"
#include "launch.h"

namespace blz {

struct WarpTile {
  double x[64];    // input, then deltas, then snapped values
  double tmp[64];  // first DCT pass
  double d[64];    // transform grid
};

__device__ __forceinline__ double warp_max(double v) {  // std::max semantics on finite values
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = stdmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(128) k_compress_worklist_warp(const Basis B, const double* __restrict__ dense,
                                                                uint64_t rows, uint64_t cols, uint64_t ld, CMat out,
                                                                unsigned long long* err,
                                                                const uint64_t* __restrict__ wl,
                                                                const unsigned long long* __restrict__ wl_count,
                                                                unsigned long long* stats) {
  __shared__ WarpTile tiles[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpTile& T = tiles[warp];
  const uint64_t n = *wl_count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(stats, (unsigned long long)n);
  for (uint64_t q = blockIdx.x * 4ull + warp; q < n; q += gridDim.x * 4ull) {
    const uint64_t t = wl[q];
    const uint64_t bi = t / out.bc, bj = t % out.bc;
    // edge-replicated tile (H/matrix.hpp:72-84)
    double m0, m1;  // cells lane, lane + 32
    {
      const int c0 = lane, c1 = lane + 32;
      const uint64_t r0 = min(bi * BD + c0 / 8, rows - 1), r1 = min(bi * BD + c1 / 8, rows - 1);
      m0 = dense[r0 * ld + min(bj * BD + c0 % 8, cols - 1)];
      m1 = dense[r1 * ld + min(bj * BD + c1 % 8, cols - 1)];
    }
    T.x[lane] = m0;
    T.x[lane + 32] = m1;
    __syncwarp();
    const double f = T.x[0];
    RBlock rb;
    rb.f = f;
    rb.s = 0.0;
    rb.phi = 1;
#pragma unroll
    for (int w = 0; w < 7; ++w) rb.c[w] = 0;
    uint32_t status = DERR_NONE;
    // all_finite (H/block.hpp:83-87)
    if (__any_sync(0xffffffffu, !is_finite(m0) || !is_finite(m1))) status = DERR_NONFINITE;
    if (status == DERR_NONE) {
      // normalize (H/codec.hpp:20-32), from the original values
      double d0, d1;
      {
        auto delta = [&](int k) {
          const int i = k / 8, j = k % 8;
          const double a = T.x[k];
          if (i == 0 && j == 0) return 0.0;
          if (i == 0) return a - T.x[k - 1];
          if (j == 0) return a - T.x[k - 8];
          return ((a - T.x[k - 8]) + (a - T.x[k - 1])) / 2.0;
        };
        d0 = delta(lane);
        d1 = delta(lane + 32);
      }
      __syncwarp();
      T.x[lane] = d0;
      T.x[lane + 32] = d1;
      __syncwarp();
      // mean_slope (H/codec.hpp:47-57): one serial chain, row-major order
      const int nz = __popc(__ballot_sync(0xffffffffu, d0 != 0.0)) + __popc(__ballot_sync(0xffffffffu, d1 != 0.0));
      double s = 0.0;
      if (lane == 0) {
        double sum = 0.0;
        for (int k = 0; k < 64; ++k)
          if (T.x[k] != 0.0) sum += fabs(T.x[k]);
        s = nz == 0 ? 0.0 : sum / (double)nz;
      }
      s = __shfl_sync(0xffffffffu, s, 0);
      rb.s = s;
      if (s != 0.0) {
        if (!(s > 0.0)) {
          status = DERR_PREDICT;
        } else {
          // slopes, s_max (H/codec.hpp:88, :138-139)
          const double v0 = d0 / s, v1 = d1 / s;
          const double smax = warp_max(stdmax(stdmax(0.0, fabs(v0)), fabs(v1)));  // never NaN, as the serial std::max
          const double lo = s - smax;
          const double step = 2.0 * smax / 256;
          const int q0 = (step == 0.0) ? 0 : clamp_index((v0 - lo) / step);
          const int q1 = (step == 0.0) ? 0 : clamp_index((v1 - lo) / step);
          __syncwarp();
          T.x[lane] = lo + (double)q0 * step;
          T.x[lane + 32] = lo + (double)q1 * step;
          __syncwarp();
          // dct2 pass 1 (H/dct.hpp:35-40): tmp(i,v) = sum_u t(i,u) x(u,v)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = lane + 32 * h, i = k / 8, v = k % 8;
            double acc = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += B.t[i * 8 + u] * T.x[u * 8 + v];
            T.tmp[k] = acc;
          }
          __syncwarp();
          // pass 2 (:42-47): d(i,j) = sum_v tmp(i,v) t(j,v); m = max |d|
          double mloc = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = lane + 32 * h, i = k / 8, j = k % 8;
            double acc = 0.0;
#pragma unroll
            for (int v = 0; v < 8; ++v) acc += T.tmp[i * 8 + v] * B.t[j * 8 + v];
            T.d[k] = acc;
            mloc = stdmax(mloc, fabs(acc));
          }
          const double mx = warp_max(mloc);
          __syncwarp();
          // quantize_coeffs (H/codec.hpp:108-125)
          if (mx != 0.0) {
            double phi = floor(127.0 / mx);
            if (phi < 1.0) phi = 1.0;
            if (phi > 255.0) phi = 255.0;
            rb.phi = (uint32_t)phi;
            int c = 0;
            if (lane < KEPT) c = clamp_coeff(phi * T.d[krow(lane) * 8 + kcol(lane)]);
            // gather the 28 bytes into 7 words
#pragma unroll
            for (int w = 0; w < 7; ++w) {
              uint32_t word = 0;
#pragma unroll
              for (int b = 0; b < 4; ++b) word |= (uint32_t)(__shfl_sync(0xffffffffu, c, 4 * w + b) & 0xff) << (8 * b);
              rb.c[w] = word;
            }
          }
        }
      }
    }
    if (lane == 0) {
      if (status != DERR_NONE) latch_error(err, t, status);
      store_block(out, t, rb);
    }
    __syncwarp();
  }
}

cudaError_t launch_compress_worklist_warp(const LaunchCtx& c, const Basis& B, const double* dense, uint64_t rows,
                                          uint64_t cols, uint64_t ld, const CMat& out) {
  k_compress_worklist_warp<<<c.sm_count, 128, 0, c.stream>>>(B, dense, rows, cols, ld, out, c.err, c.wl,
                                                             c.wl_count, c.stats + 0);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
