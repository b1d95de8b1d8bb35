// stages.cu -- the codec's stage functions as batched device calls (SURVEY.md 8(b):
// "the stage functions in H/codec.hpp / H/dct.hpp" are public API, called by the
// reference's codec and dct tests).  One thread per 8x8 block, each stage exactly
// as the reference writes it (-fmad=false, reference order):
//
//   normalize / denormalize   H/codec.hpp:20-44
//   mean_slope                H/codec.hpp:47-57
//   predict                   H/codec.hpp:61-98 (slope_quantizer encode / decode)
//   quantize_coeffs           H/codec.hpp:108-125
//   dct2 / idct2              H/dct.hpp:32-70
//
// compress / decompress do not use these kernels: they run the fused kernels of
// codec.cu / compress_pair.cu.
#include "blaz_device.cuh"
#include "launch.h"

namespace blz {

namespace {

__device__ __forceinline__ void load64(const double* __restrict__ p, uint64_t t, double (&m)[BC]) {
#pragma unroll
  for (int k = 0; k < BC; ++k) m[k] = p[t * BC + k];
}
__device__ __forceinline__ void store64(double* __restrict__ p, uint64_t t, const double (&m)[BC]) {
#pragma unroll
  for (int k = 0; k < BC; ++k) p[t * BC + k] = m[k];
}

#define BLZ_FOR_BLOCKS(n) \
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < (n); t += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_normalize(const double* __restrict__ in, uint64_t n, double* __restrict__ first,
                            double* __restrict__ deltas, unsigned long long* err) {
  BLZ_FOR_BLOCKS(n) {
    double m[BC], d[BC];
    load64(in, t, m);
    bool fin = true;
#pragma unroll
    for (int k = 0; k < BC; ++k) fin &= is_finite(m[k]);
    if (!fin) {
      latch_error(err, t, DERR_NONFINITE);
      continue;
    }
    first[t] = m[0];
    d[0] = 0.0;
#pragma unroll
    for (int j = 1; j < BD; ++j) d[j] = m[j] - m[j - 1];
#pragma unroll
    for (int i = 1; i < BD; ++i) d[i * BD] = m[i * BD] - m[(i - 1) * BD];
#pragma unroll
    for (int i = 1; i < BD; ++i)
#pragma unroll
      for (int j = 1; j < BD; ++j)
        d[i * BD + j] = ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) / 2.0;
    store64(deltas, t, d);
  }
}

__global__ void k_denormalize(const double* __restrict__ first, const double* __restrict__ deltas, uint64_t n,
                              double* __restrict__ out) {
  BLZ_FOR_BLOCKS(n) {
    double d[BC], m[BC];
    load64(deltas, t, d);
    m[0] = first[t];
#pragma unroll
    for (int j = 1; j < BD; ++j) m[j] = m[j - 1] + d[j];
#pragma unroll
    for (int i = 1; i < BD; ++i) m[i * BD] = m[(i - 1) * BD] + d[i * BD];
#pragma unroll
    for (int i = 1; i < BD; ++i)
#pragma unroll
      for (int j = 1; j < BD; ++j) m[i * BD + j] = (m[(i - 1) * BD + j] + m[i * BD + j - 1]) / 2.0 + d[i * BD + j];
    store64(out, t, m);
  }
}

__global__ void k_mean_slope(const double* __restrict__ deltas, uint64_t n, double* __restrict__ out) {
  BLZ_FOR_BLOCKS(n) {
    double sum = 0.0;
    int nz = 0;
    for (int k = 0; k < BC; ++k) {
      const double v = deltas[t * BC + k];
      if (v != 0.0) {
        sum += fabs(v);
        ++nz;
      }
    }
    out[t] = nz == 0 ? 0.0 : sum / (double)nz;
  }
}

__global__ void k_predict(const double* __restrict__ slopes, const double* __restrict__ mean, uint64_t n,
                          uint8_t* __restrict__ idx, double* __restrict__ snapped, double* __restrict__ lo_out,
                          double* __restrict__ step_out, unsigned long long* err) {
  BLZ_FOR_BLOCKS(n) {
    const double sm = mean[t];
    if (!(sm > 0.0)) {
      latch_error(err, t, DERR_PREDICT);
      continue;
    }
    double v[BC];
    load64(slopes, t, v);
    double smax = 0.0;
#pragma unroll
    for (int k = 0; k < BC; ++k) smax = stdmax(smax, fabs(v[k]));
    const double lo = sm - smax;
    const double step = 2.0 * smax / 256;
    lo_out[t] = lo;
    step_out[t] = step;
#pragma unroll
    for (int k = 0; k < BC; ++k) {
      const int q = (step == 0.0) ? 0 : clamp_index((v[k] - lo) / step);
      idx[t * BC + k] = (uint8_t)q;
      snapped[t * BC + k] = lo + (double)q * step;
    }
  }
}

__global__ void k_quantize_coeffs(const double* __restrict__ dgrid, uint64_t n, uint8_t* __restrict__ scale,
                                  int8_t* __restrict__ coeffs) {
  BLZ_FOR_BLOCKS(n) {
    double d[BC];
    load64(dgrid, t, d);
    double mx = 0.0;
#pragma unroll
    for (int k = 0; k < BC; ++k) mx = stdmax(mx, fabs(d[k]));
    if (mx == 0.0) {
      scale[t] = 1;
#pragma unroll
      for (int k = 0; k < KEPT; ++k) coeffs[t * KEPT + k] = 0;
      continue;
    }
    double phi = floor(127.0 / mx);
    if (phi < 1.0) phi = 1.0;
    if (phi > 255.0) phi = 255.0;
    scale[t] = (uint8_t)phi;
    // keep set: rows 0-1 (k 0-15), then column 0 / column 1 of rows 2-7 (H/block.hpp:48-56)
#pragma unroll
    for (int k = 0; k < KEPT; ++k) {
      const int r = k < 16 ? k / 8 : (k < 22 ? k - 14 : k - 20);
      const int c = k < 16 ? k % 8 : (k < 22 ? 0 : 1);
      coeffs[t * KEPT + k] = (int8_t)clamp_coeff(phi * d[r * BD + c]);
    }
  }
}

// dct2: d = T x T' (tmp = T x, then d = tmp T'); idct2: x = T' d T.
template <bool INVERSE>
__global__ void k_dct(const Basis B, const double* __restrict__ in, uint64_t n, double* __restrict__ out) {
  BLZ_FOR_BLOCKS(n) {
    double x[BC], tmp[BC], y[BC];
    load64(in, t, x);
#pragma unroll
    for (int a = 0; a < BD; ++a)
#pragma unroll
      for (int b = 0; b < BD; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < BD; ++c)
          acc += INVERSE ? B.t[c * BD + a] * x[c * BD + b] : B.t[a * BD + c] * x[c * BD + b];
        tmp[a * BD + b] = acc;
      }
#pragma unroll
    for (int a = 0; a < BD; ++a)
#pragma unroll
      for (int b = 0; b < BD; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < BD; ++c) acc += INVERSE ? tmp[a * BD + c] * B.t[c * BD + b] : tmp[a * BD + c] * B.t[b * BD + c];
        y[a * BD + b] = acc;
      }
    store64(out, t, y);
  }
}

unsigned grid(const LaunchCtx& c, uint64_t n) {
  const uint64_t want = (n + 127) / 128;
  const uint64_t cap = (uint64_t)c.sm_count * 16;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_stage(const LaunchCtx& c, const Basis& B, int stage, const double* in0, const double* in1,
                         uint64_t n, double* out0, double* out1, double* out2, void* out3) {
  const unsigned g = grid(c, n);
  switch (stage) {
    case STAGE_NORMALIZE: k_normalize<<<g, 128, 0, c.stream>>>(in0, n, out1, out0, c.err); break;
    case STAGE_DENORMALIZE: k_denormalize<<<g, 128, 0, c.stream>>>(in1, in0, n, out0); break;
    case STAGE_MEAN_SLOPE: k_mean_slope<<<g, 128, 0, c.stream>>>(in0, n, out0); break;
    case STAGE_PREDICT:
      k_predict<<<g, 128, 0, c.stream>>>(in0, in1, n, (uint8_t*)out3, out0, out1, out2, c.err);
      break;
    case STAGE_QUANTIZE:
      k_quantize_coeffs<<<g, 128, 0, c.stream>>>(in0, n, (uint8_t*)out3, (int8_t*)out1);
      break;
    case STAGE_DCT2: k_dct<false><<<g, 128, 0, c.stream>>>(B, in0, n, out0); break;
    case STAGE_IDCT2: k_dct<true><<<g, 128, 0, c.stream>>>(B, in0, n, out0); break;
    default: return cudaErrorInvalidValue;
  }
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
