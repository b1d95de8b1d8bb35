// blaz_device.cuh -- per-8x8-block device arithmetic for sm_100a.
//
// Exact mode: this header is only compiled with nvcc -fmad=false, so every
// a*b+c below is a DMUL followed by a DADD, matching the reference built with
// -ffp-contract=off (proj/CMakeLists.txt:15-18).  The evaluation order of
// each expression follows the reference line cited next to it.
//
// Deliberate, proven-equivalent deviations:
//  * acc = 0.0; acc += p0; ...  is computed as acc = p0; ... wherever p0 can
//    never be -0.0 (0.0 + p0 == p0 for every p0 != -0.0).  Holds for all four
//    DCT passes: t(i,0) > 0 and the other factor is never -0.0.
//  * products with a structurally-zero factor (the 36 discarded coefficient
//    positions) are skipped: a running sum that starts at +0.0 is never -0.0,
//    so adding +-0.0 to it is the identity.
#pragma once
#include <cstdint>

#include "blaz_types.h"

#ifndef DEC_V4
#define DEC_V4 1
#endif

namespace blz {

constexpr int BD = 8;
constexpr int BC = 64;
constexpr int KEPT = 28;

// Reference status codes latched on device (first failing block wins).
enum DevErr : uint32_t {
  DERR_NONE = 0,
  DERR_NONFINITE = DERR_NONFINITE_CODE,
  DERR_PREDICT = DERR_PREDICT_CODE,
  DERR_DOT_RANGE = DERR_DOT_RANGE_CODE,
};

// H/block.hpp:48-56: keep-set position of coefficient k.
__host__ __device__ constexpr int krow(int k) { return k < 8 ? 0 : k < 16 ? 1 : k < 22 ? k - 14 : k - 20; }
__host__ __device__ constexpr int kcol(int k) { return k < 8 ? k : k < 16 ? k - 8 : k < 22 ? 0 : 1; }

// std::max(a, b) == (a < b) ? b : a  -- a NaN b leaves a unchanged.
__device__ __forceinline__ double stdmax(double a, double b) { return (a < b) ? b : a; }

// H/block.hpp:61-67.  (double)(long long)x with the x86-64 conversion result
// for out-of-range/NaN inputs (INT64_MIN), which the reference build executes.
__device__ __forceinline__ double round_half_away(double x) {
  double t;
  if (x >= -9223372036854775808.0 && x < 9223372036854775808.0)
    t = __ll2double_rn(__double2ll_rz(x));
  else
    t = -9223372036854775808.0;
  const double frac = x - t;
  if (frac >= 0.5) return t + 1.0;
  if (frac <= -0.5) return t - 1.0;
  return t;
}

// H/block.hpp:69-74
__device__ __forceinline__ int clamp_index(double x) {
  const double r = round_half_away(x);
  if (r <= 0.0) return 0;
  if (r >= 255.0) return 255;
  return (int)r;
}

// H/block.hpp:76-81
__device__ __forceinline__ int clamp_coeff(double x) {
  const double r = round_half_away(x);
  if (r <= -127.0) return -127;
  if (r >= 127.0) return 127;
  return (int)r;
}

__device__ __forceinline__ bool is_finite(double v) {
  return (__double_as_longlong(v) & 0x7ff0000000000000ll) != 0x7ff0000000000000ll;
}

// Packs coefficient k (int in [-128,127]) into 7 little-endian words.
__device__ __forceinline__ void put_coeff(uint32_t (&w)[7], int k, int c) {
  w[k >> 2] |= (uint32_t)(c & 0xff) << (8 * (k & 3));
}
// Byte q of w as a signed int8, converted to double: one I2F.F64.S8 with a byte
// selector (byte 0 through PTX cvt.s8, which C++ sign extension would turn into
// two PRMTs and an I2F.S16).
__device__ __forceinline__ double i8_byte_to_f64(uint32_t w, int q) {
  if (q == 0) {
    double d;
    asm("cvt.rn.f64.s8 %0, %1;" : "=d"(d) : "h"((unsigned short)w));
    return d;
  }
  return (double)(int8_t)(uint8_t)(w >> (8 * q));
}

__device__ __forceinline__ int get_coeff(const uint32_t (&w)[7], int k) {
  return (int)(int8_t)(uint8_t)(w[k >> 2] >> (8 * (k & 3)));
}

// One 8-double output row to global memory: two 32-byte stores (st.global.v4.f64,
// STG.E.ENL2.256 -- whole 32-byte sectors) when v4 (dst 32-byte aligned), else four
// 16-byte stores (dst 16-byte aligned).
__device__ __forceinline__ void store_row8(double* dst, const double (&row)[BD], bool v4) {
  if (v4) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * h), "d"(row[4 * h]),
                   "d"(row[4 * h + 1]), "d"(row[4 * h + 2]), "d"(row[4 * h + 3])
                   : "memory");
  } else {
    double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d2[q] = make_double2(row[2 * q], row[2 * q + 1]);
  }
}

// One 8-double input row through the read-only path: two 32-byte loads
// (ld.global.nc.v4.f64, LDG.E.ENL2.256) when v4 (src 32-byte aligned), else four 16-byte loads.
__device__ __forceinline__ void load_row8(const double* src, double (&row)[BD], bool v4) {
  if (v4) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
          : "=d"(row[4 * h]), "=d"(row[4 * h + 1]), "=d"(row[4 * h + 2]), "=d"(row[4 * h + 3])
          : "l"(src + 4 * h));
  } else {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 x = __ldg(s2 + q);
      row[2 * q] = x.x;
      row[2 * q + 1] = x.y;
    }
  }
}

// Whether rows of a dense output at `dense` with leading dimension ld take 32-byte stores.
__device__ __host__ __forceinline__ bool rows_v4(const double* dense, uint64_t ld) {
  return DEC_V4 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(dense) & 31) == 0;
}

// Compressed block in registers.
struct RBlock {
  double f, s;
  uint32_t phi;
  uint32_t c[7];
};

// ---------------------------------------------------------------------------
// compress_block (H/codec.hpp:130-146), exact.  m is overwritten.
// Returns a DevErr.  The constant-block path returns {f, s(=+-0), 1, 0s}.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t compress_exact(double (&m)[BC], const Basis& B, RBlock& out) {
  bool fin = true;
#pragma unroll
  for (int k = 0; k < BC; ++k) fin &= is_finite(m[k]);
  out.phi = 1;
#pragma unroll
  for (int w = 0; w < 7; ++w) out.c[w] = 0;
  out.f = m[0];
  out.s = 0.0;
  if (!fin) return DERR_NONFINITE;

  // normalize (H/codec.hpp:20-32), in place, reverse order so that the
  // up/left neighbours read are still the original values.
#pragma unroll
  for (int i = BD - 1; i >= 1; --i)
#pragma unroll
    for (int j = BD - 1; j >= 1; --j)
      m[i * BD + j] = ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) / 2.0;
#pragma unroll
  for (int i = BD - 1; i >= 1; --i) m[i * BD] = m[i * BD] - m[(i - 1) * BD];
#pragma unroll
  for (int j = BD - 1; j >= 1; --j) m[j] = m[j] - m[j - 1];
  m[0] = 0.0;

  // mean_slope (H/codec.hpp:47-57): serial row-major sum over nonzero deltas.
  double sum = 0.0;
  int nz = 0;
#pragma unroll
  for (int k = 0; k < BC; ++k) {
    if (m[k] != 0.0) {
      sum += fabs(m[k]);
      ++nz;
    }
  }
  const double s = nz == 0 ? 0.0 : sum / (double)nz;
  out.s = s;
  if (s == 0.0) return DERR_NONE;
  if (!(s > 0.0)) return DERR_PREDICT;

  // slopes = deltas / s (H/codec.hpp:138-139), s_max (:88)
  double smax = 0.0;
#pragma unroll
  for (int k = 0; k < BC; ++k) {
    m[k] = m[k] / s;
    smax = stdmax(smax, fabs(m[k]));
  }
  // slope_quantizer (H/codec.hpp:61-71, :90-96)
  const double lo = s - smax;
  const double step = 2.0 * smax / 256;
#pragma unroll
  for (int k = 0; k < BC; ++k) {
    const int q = (step == 0.0) ? 0 : clamp_index((m[k] - lo) / step);
    m[k] = lo + (double)q * step;
  }

  // dct2 (H/dct.hpp:32-49) fused with quantize_coeffs' max (H/codec.hpp:110):
  // row i of tmp = T x needs all of x; row i of d = tmp T' needs tmp row i.
  double dk[KEPT];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < BD; ++i) {
    double tr[BD];
#pragma unroll
    for (int v = 0; v < BD; ++v) {
      double acc = B.t[i * BD + 0] * m[0 * BD + v];
#pragma unroll
      for (int u = 1; u < BD; ++u) acc += B.t[i * BD + u] * m[u * BD + v];
      tr[v] = acc;
    }
#pragma unroll
    for (int j = 0; j < BD; ++j) {
      double acc = tr[0] * B.t[j * BD + 0];
#pragma unroll
      for (int v = 1; v < BD; ++v) acc += tr[v] * B.t[j * BD + v];
      mx = stdmax(mx, fabs(acc));
      if (i < 2) dk[i * 8 + j] = acc;
      else if (j == 0) dk[14 + i] = acc;
      else if (j == 1) dk[20 + i] = acc;
    }
  }
  // quantize_coeffs (H/codec.hpp:108-125)
  if (mx == 0.0) return DERR_NONE;
  double phi = floor(127.0 / mx);
  if (phi < 1.0) phi = 1.0;
  if (phi > 255.0) phi = 255.0;
  out.phi = (uint32_t)phi;
#pragma unroll
  for (int k = 0; k < KEPT; ++k) put_coeff(out.c, k, clamp_coeff(phi * dk[k]));
  return DERR_NONE;
}

// ---------------------------------------------------------------------------
// decompress_block (H/codec.hpp:150-185), exact, streamed row by row:
// emit(u, row[8]) is called for u = 0..7 in order.
// ---------------------------------------------------------------------------
// C / phi, correctly rounded, for integer C in [-128, 127] and phi in [1, 255]:
// r = RN(1/phi), q = RN(C*r), e = C - phi*q (exact in one FMA), RN(q + e*r).
// Equal to the IEEE quotient over the whole 256 x 255 domain (checked
// exhaustively, tests/test_oracle_golden.py::test_markstein_dequant_exhaustive).
__device__ __forceinline__ double dequant_d(double cd, double phi, double r) {
  const double q = cd * r;
  const double e = fma(-phi, q, cd);
  return fma(e, r, q);
}
__device__ __forceinline__ double dequant(int c, double phi, double r) {
  const double cd = (double)c;
  const double q = cd * r;
  const double e = fma(-phi, q, cd);
  return fma(e, r, q);
}

// SYM: the basis has the bitwise repeats of the reference's (glibc) basis --
// row 0 constant, and t(1,7) = -t(1,0), t(2,3) = -t(2,0), t(3,5) = -t(3,2),
// t(4,4) = -t(4,2) (checked on the host, analyse_basis).  Equal factors give
// equal (or exactly negated) rounded products, so those products are formed
// once; every sum keeps the reference's order.
#ifndef DEC_DQSEL
#define DEC_DQSEL 0  // the output select alone yields the +0.0 grid for s == 0
#endif
template <bool SLOPES_ONLY, bool SYM = false, class Emit>
__device__ __forceinline__ void decompress_rows_impl(const RBlock& b, const Basis& B, Emit&& emit) {
  const double s = b.s;
  double dq[KEPT];
  const bool zero = (s == 0.0);  // dequantize_prediction returns a zero grid (:151)
  const double fphi = (double)b.phi;
  // phi in [1,255] (the reference reader rejects 0, H/io.hpp:129-130); other
  // values take the IEEE division so that the result is still C / phi.
  if (b.phi - 1u < 255u) {
    const double r = 1.0 / fphi;
#pragma unroll
    for (int k = 0; k < KEPT; ++k) dq[k] = DEC_DQSEL && zero ? 0.0 : dequant_d(i8_byte_to_f64(b.c[k >> 2], k & 3), fphi, r);
  } else {
#pragma unroll
    for (int k = 0; k < KEPT; ++k) dq[k] = zero ? 0.0 : (double)get_coeff(b.c, k) / fphi;
  }

  if (SYM) {  // t(0,u) d(0,j) is the same for every u
#pragma unroll
    for (int j = 0; j < BD; ++j) dq[j] = B.t[0] * dq[j];
  }

  double prev[BD];
#pragma unroll
  for (int u = 0; u < BD; ++u) {
    // idct2 pass 1 (H/dct.hpp:56-61): tmp(u,j) = sum_i t(i,u) d(i,j), the
    // discarded positions (rows>=2 x cols>=2) are structural zeros.
    double tr[BD];
#pragma unroll
    for (int j = 0; j < BD; ++j) {
      double acc = SYM ? dq[j] : B.t[0 * BD + u] * dq[j];  // d(0,j) = dq[j]
      acc += B.t[1 * BD + u] * dq[8 + j];                // d(1,j) = dq[8+j]
      if (j == 0) {
#pragma unroll
        for (int i = 2; i < BD; ++i) acc += B.t[i * BD + u] * dq[14 + i];
      } else if (j == 1) {
#pragma unroll
        for (int i = 2; i < BD; ++i) acc += B.t[i * BD + u] * dq[20 + i];
      }
      tr[j] = acc;
    }
    // idct2 pass 2 (H/dct.hpp:62-68): x(u,v) = sum_j tmp(u,j) t(j,v)
    double p[BD];
    if (SYM) {
      const double p0 = tr[0] * B.t[0];
      const double q1 = tr[1] * B.t[1 * BD + 0], q2 = tr[2] * B.t[2 * BD + 0];
      const double q3 = tr[3] * B.t[3 * BD + 2], q4 = tr[4] * B.t[4 * BD + 2];
#pragma unroll
      for (int v = 0; v < BD; ++v) {
        double acc = p0;
        acc += v == 0 ? q1 : (v == 7 ? -q1 : tr[1] * B.t[1 * BD + v]);
        acc += v == 0 ? q2 : (v == 3 ? -q2 : tr[2] * B.t[2 * BD + v]);
        acc += v == 2 ? q3 : (v == 5 ? -q3 : tr[3] * B.t[3 * BD + v]);
        acc += v == 2 ? q4 : (v == 4 ? -q4 : tr[4] * B.t[4 * BD + v]);
#pragma unroll
        for (int j = 5; j < BD; ++j) acc += tr[j] * B.t[j * BD + v];
        p[v] = zero ? 0.0 : acc;
      }
    } else {
#pragma unroll
      for (int v = 0; v < BD; ++v) {
        double acc = tr[0] * B.t[0 * BD + v];
#pragma unroll
        for (int j = 1; j < BD; ++j) acc += tr[j] * B.t[j * BD + v];
        p[v] = zero ? 0.0 : acc;
      }
    }
    if (SLOPES_ONLY) {
      emit(u, p);
      continue;
    }
    // integrate_rows (H/codec.hpp:164-174)
    double row[BD];
    if (u == 0) {
      row[0] = b.f;
#pragma unroll
      for (int j = 1; j < BD; ++j) row[j] = row[j - 1] + s * p[j];
    } else {
      row[0] = prev[0] + s * p[0];
#pragma unroll
      for (int j = 1; j < BD; ++j) row[j] = (prev[j] + row[j - 1]) / 2.0 + s * p[j];
    }
    emit(u, row);
#pragma unroll
    for (int j = 0; j < BD; ++j) prev[j] = row[j];
  }
}

template <bool SYM = false, class Emit>
__device__ __forceinline__ void decompress_exact(const RBlock& b, const Basis& B, Emit&& emit) {
  decompress_rows_impl<false, SYM>(b, B, emit);
}

// dequantize_prediction (H/codec.hpp:150-158) streamed row by row: emit(u, p[8])
// with p = row u of idct2(d), d the dequantized coefficient grid; zeros for s == 0.
template <class Emit>
__device__ __forceinline__ void slope_grid_exact(const RBlock& b, const Basis& B, Emit&& emit) {
  decompress_rows_impl<true>(b, B, emit);
}

// Full 8x8 decompression into registers.
__device__ __forceinline__ void decompress_exact_full(const RBlock& b, const Basis& B, double (&out)[BC]) {
  decompress_exact(b, B, [&](int u, const double (&row)[BD]) {
#pragma unroll
    for (int j = 0; j < BD; ++j) out[u * BD + j] = row[j];
  });
}

// H/block_ops.hpp:12-15 (phi1 + phi2 == 0 only for invalid blocks; defined as 1)
__device__ __forceinline__ uint32_t merge_scale_factor(uint32_t p1, uint32_t p2) {
  const uint32_t den = p1 + p2;
  if (den == 0) return 1;
  const uint32_t phi = (p1 * p2) / den;
  return phi < 1 ? 1 : (phi > 255 ? 255 : phi);
}

// The same for scale factors in [0, 255] (every record the kernels produce or
// read; the callers route others to merge_scale_factor): floor(N / D) with
// N = p1 p2 <= 65025, D = p1 + p2 <= 510 through one approximate fp32 division
// instead of the integer division sequence.  N and D are exact in fp32;
// __fdividef is within 2 ulp, i.e. a relative error below 2^-21, so the fp32
// quotient is within 255 * 2^-21 < 1.3e-4 of N / D, while a non-integer N / D is
// at least 1 / D >= 1 / 510 > 1.9e-3 away from the next integer above it and the
// quotient of a multiple is exact to 1.3e-4 (floor of q in [k - 1.3e-4, k + 1.3e-4]
// is taken after adding 1/1024, which keeps k and stays below the next integer).
__device__ __forceinline__ uint32_t merge_scale_factor_u8(uint32_t p1, uint32_t p2) {
  const uint32_t den = p1 + p2;
  const float q = __fdividef((float)(p1 * p2), (float)den) + (1.0f / 1024.0f);
  const uint32_t phi = den == 0 ? 1u : (uint32_t)__float2int_rz(q);
  return phi < 1 ? 1 : (phi > 255 ? 255 : phi);
}

// H/block_ops.hpp:20-58 without the dense fallback.  Returns false when the
// s1 + s2 == 0 dense fallback (:36-44) is required.
template <bool SUB>
__device__ __forceinline__ bool combine_fast(const RBlock& b1, const RBlock& b2, RBlock& out) {
  const double rhs = SUB ? -1.0 : 1.0;
  const double f = b1.f + rhs * b2.f;
  if (b2.s == 0.0) {  // :27
    out = b1;
    out.f = f;
    return true;
  }
  if (b1.s == 0.0) {  // :28-33
    out = b2;
    out.f = f;
    if (SUB) {
#pragma unroll
      for (int w = 0; w < 7; ++w) {
        uint32_t r = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = (int)(int8_t)(uint8_t)(b2.c[w] >> (8 * q));
          const int n = (c == -127) ? 127 : -c;
          r |= (uint32_t)(n & 0xff) << (8 * q);
        }
        out.c[w] = r;
      }
    }
    return true;
  }
  const double s = b1.s + b2.s;  // :35
  if (s == 0.0) return false;    // :36-44
  out.f = f;
  out.s = s;
  const uint32_t phi = merge_scale_factor(b1.phi, b2.phi);
  out.phi = phi;
  const double a1 = b1.s / s;                                 // :51
  const double a2 = rhs * b2.s / s;                           // :52
  const double w1 = a1 / (double)b1.phi * (double)phi;        // :53
  const double w2 = a2 / (double)b2.phi * (double)phi;        // :54
#pragma unroll
  for (int w = 0; w < 7; ++w) out.c[w] = 0;
#pragma unroll
  for (int k = 0; k < KEPT; ++k)                              // :55-56
    put_coeff(out.c, k, clamp_coeff(w1 * (double)get_coeff(b1.c, k) + w2 * (double)get_coeff(b2.c, k)));
  return true;
}

// Block coordinates (row-major block grid) of t, t + S, t + 2S, ... for a
// grid-stride loop: one division at the start, then an add with carry per step
// instead of a 64-bit division per iteration.  bi may run past the grid for
// lanes beyond the last block; callers clamp those (coords()).
struct BlockCursor {
  uint64_t bi, bj, sq, sr;
  __device__ __forceinline__ BlockCursor(uint64_t t, uint64_t stride, uint64_t bc)
      : bi(t / bc), bj(t % bc), sq(stride / bc), sr(stride % bc) {}
  // stride quotient / remainder precomputed by the host
  __device__ __forceinline__ BlockCursor(uint64_t t, uint64_t bc, uint64_t sq_, uint64_t sr_)
      : bi(t / bc), sq(sq_), sr(sr_) {
    bj = t - bi * bc;
  }
  __device__ __forceinline__ void advance(uint64_t bc) {
    bj += sr;
    bi += sq;
    if (bj >= bc) {
      bj -= bc;
      ++bi;
    }
  }
};

// ---- SoA global access -------------------------------------------------------
__device__ __forceinline__ RBlock load_block(const CMat& m, uint64_t t) {
  RBlock b;
  b.f = m.first[t];
  b.s = m.slope[t];
  b.phi = m.scale[t];
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(m.coeffs + t * KEPT);
#pragma unroll
  for (int w = 0; w < 7; ++w) b.c[w] = cw[w];
  return b;
}

__device__ __forceinline__ void store_block(const CMat& m, uint64_t t, const RBlock& b) {
  m.first[t] = b.f;
  m.slope[t] = b.s;
  m.scale[t] = (uint8_t)b.phi;
  uint32_t* cw = reinterpret_cast<uint32_t*>(m.coeffs + t * KEPT);
#pragma unroll
  for (int w = 0; w < 7; ++w) cw[w] = b.c[w];
}

// Latches the error of the lowest failing block index.
__device__ __forceinline__ void latch_error(unsigned long long* err, uint64_t block, uint32_t code) {
  atomicMin(err, (unsigned long long)((block << 8) | code));
}

}  // namespace blz
