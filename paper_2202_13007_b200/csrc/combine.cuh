// combine.cuh -- the arithmetic of add / sub (H/block_ops.hpp:20-71) on one
// block's record, shared by k_addsub_v2 (addsub.cu) and the fused op+decompress
// kernels (fused.cu).  Exactly the reference's operations; the coefficient
// rounding is branch-free (see below).
#pragma once
#include "blaz_device.cuh"
#include "fastpath.cuh"  // hi32
#include "rcp_table.cuh"

namespace blz {

struct CombineOut {
  double f, s;
  uint32_t phi;
  uint32_t c[7];
  bool fallback;  // s1 + s2 == 0: dense fallback (:36-44), recomputed elsewhere
  bool slow;      // huge / NaN weights: coefficients need the reference rounding sequence
  double w1, w2;  // the weights (for the slow path)
};

// clamp_coeff(round_half_away(v)) (H/block.hpp:61-81) for |v| < 2^30: the
// reference's round_half_away is sign(v) * trunc(RZ(|v| + 1/2)) exactly (RZ never
// crosses the representable integer floor(|v| + 1/2)), and clamping the magnitude
// to 127 before applying the sign is clamp_coeff's [-127, 127].  This returns the
// magnitude; trunc(t) for t in [1/2, 2^30) is the low word of RZ(t + 2^52), an FP64
// add instead of a conversion-unit F2I (the conversion unit was the busiest pipe).
__device__ __forceinline__ int round_magnitude(double v) {
  return min(__double2loint(__dadd_rz(__dadd_rz(fabs(v), 0.5), 4503599627370496.0)), 127);
}

// bytes 0, 1 = 0xff where the sign bit of a (resp. b) is set, else 0 (PRMT sign replication)
__device__ __forceinline__ uint32_t prmt_sign2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x00fb;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// a / b for b > 0 given y = RN(1/b): q = RN(a y), e = a - b q (exact), RN(q + e y)
// is RN(a / b) (Markstein) when a, b and the quotient stay clear of underflow /
// overflow -- the callers guard the exponent range.
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q = a * y;
  const double e = fma(-b, q, a);
  return fma(e, y, q);
}

// |x| in [2^-400, 2^400] (NaN / inf excluded), from the high word read as a float
__device__ __forceinline__ bool mid_range(double x) {
  const float h = fabsf(__int_as_float((int)hi32(x)));
  return h > __int_as_float(0x26f00000) && h < __int_as_float(0x58f00000);
}

// The coefficient words come as arrays in registers or as a view of shared
// memory (SmemWords): each branch then loads the words it uses, instead of the
// compiler moving register copies between the branches.
struct SmemWords {
  const uint32_t* p;
  __device__ __forceinline__ uint32_t operator[](int w) const { return p[w]; }
};

template <bool SUB, class W1, class W2>
__device__ __forceinline__ CombineOut combine_record(double f1, double s1, uint32_t p1, const W1& c1, double f2,
                                                     double s2, uint32_t p2, const W2& c2) {
  CombineOut o;
  const double rhs = SUB ? -1.0 : 1.0;
  o.f = f1 + rhs * f2;  // (:22)
  o.fallback = false;
  o.slow = false;
  o.w1 = 0.0;
  o.w2 = 0.0;
  if (s2 == 0.0) {  // (:27)
    o.s = s1;
    o.phi = p1;
#pragma unroll
    for (int w = 0; w < 7; ++w) o.c[w] = c1[w];
  } else if (s1 == 0.0) {  // (:28-33)
    o.s = s2;
    o.phi = p2;
#pragma unroll
    for (int w = 0; w < 7; ++w) {
      uint32_t r = c2[w];
      if (SUB) {
        r = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = (int)(int8_t)(uint8_t)(c2[w] >> (8 * q));
          const int n = (c == -127) ? 127 : -c;
          r |= (uint32_t)(n & 0xff) << (8 * q);
        }
      }
      o.c[w] = r;
    }
  } else {
    o.s = s1 + s2;               // (:35)
    o.fallback = (o.s == 0.0);   // (:36-44)
    const uint32_t phi = merge_scale_factor_u8(p1, p2);  // p1, p2 are bytes (u8 fields)
    o.phi = phi;
    // Slopes in [2^-400, 2^400] keep every quotient below clear of underflow /
    // overflow, so one IEEE reciprocal of s serves both divisions by s and the
    // divisions by the (nonzero) scale factors use the table of RN(1/p); each
    // quotient is then RN(a / b) (div_rcp, tools/microbench/markstein_check.cu).
    // Otherwise (phi = 0 included) the plain IEEE divisions.
    if (mid_range(s1) && mid_range(s2) && mid_range(o.s) && p1 != 0u && p2 != 0u) {
      const double ys = 1.0 / o.s;
      const double a1 = div_rcp(s1, o.s, ys);        // (:51)
      const double a2 = div_rcp(rhs * s2, o.s, ys);  // (:52)
      const double2 t1 = __ldg(&k_rcp_u8[p1]), t2 = __ldg(&k_rcp_u8[p2]);
      const double fphi = __ldg(&k_rcp_u8[phi].y);
      o.w1 = div_rcp(a1, t1.y, t1.x) * fphi;  // (:53)
      o.w2 = div_rcp(a2, t2.y, t2.x) * fphi;  // (:54)
    } else {
      const double a1 = s1 / o.s;
      const double a2 = rhs * s2 / o.s;
      o.w1 = a1 / (double)p1 * (double)phi;
      o.w2 = a2 / (double)p2 * (double)phi;
    }
    // |v| <= 127 (|w1| + |w2|) < 2^30 unless the weights are huge (s1 + s2 nearly
    // cancelling) or NaN: those blocks take the reference sequence (caller).
    o.slow = !(fabs(o.w1) + fabs(o.w2) < 4194304.0);
#pragma unroll
    for (int w = 0; w < 7; ++w) {
      // magnitudes packed, then the four signs applied bytewise: (m ^ s) - s with
      // s in {0, 0xff} per byte, as ((m ^ s) & 0x7f) + (s & 1), then bit 7 ^ s
      // (m <= 127, so no carry leaves a byte)
      int m[4];
      uint32_t h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double x1 = i8_byte_to_f64(c1[w], q);  // I2F.F64.S8 on a byte lane
        const double x2 = i8_byte_to_f64(c2[w], q);
        const double v = o.w1 * x1 + o.w2 * x2;      // (:55-56)
        m[q] = round_magnitude(v);
        h[q] = hi32(v);
      }
      const uint32_t M = __byte_perm(__byte_perm(m[0], m[1], 0x0040), __byte_perm(m[2], m[3], 0x0040), 0x5410);
      const uint32_t S = __byte_perm(prmt_sign2(h[0], h[1]), prmt_sign2(h[2], h[3]), 0x5410);
      const uint32_t L = ((M ^ S) & 0x7f7f7f7fu) + (S & 0x01010101u);
      o.c[w] = L ^ (S & 0x80808080u);
    }
  }
  return o;
}

}  // namespace blz
