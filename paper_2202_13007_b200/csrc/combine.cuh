// combine.cuh -- the arithmetic of add / sub (H/block_ops.hpp:20-71) on one
// block's record, shared by k_addsub_v2 (addsub.cu) and the fused op+decompress
// kernels (fused.cu).  Exactly the reference's operations; the coefficient
// rounding is branch-free (see below).
#pragma once
#include "blaz_device.cuh"
#include "fastpath.cuh"  // hi32

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
// to 127 before applying the sign is clamp_coeff's [-127, 127].
__device__ __forceinline__ int round_clamp_coeff(double v) {
  const int m = min(__double2int_rz(__dadd_rz(fabs(v), 0.5)), 127);
  const int sg = (int)hi32(v) >> 31;
  return (m ^ sg) - sg;
}

template <bool SUB>
__device__ __forceinline__ CombineOut combine_record(double f1, double s1, uint32_t p1, const uint32_t (&c1)[7],
                                                     double f2, double s2, uint32_t p2, const uint32_t (&c2)[7]) {
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
    const double a1 = s1 / o.s;        // (:51)
    const double a2 = rhs * s2 / o.s;  // (:52)
    o.w1 = a1 / (double)p1 * (double)phi;  // (:53)
    o.w2 = a2 / (double)p2 * (double)phi;  // (:54)
    // |v| <= 127 (|w1| + |w2|) < 2^30 unless the weights are huge (s1 + s2 nearly
    // cancelling) or NaN: those blocks take the reference sequence (caller).
    o.slow = !(fabs(o.w1) + fabs(o.w2) < 4194304.0);
#pragma unroll
    for (int w = 0; w < 7; ++w) {
      int n[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double x1 = i8_byte_to_f64(c1[w], q);  // I2F.F64.S8 on a byte lane
        const double x2 = i8_byte_to_f64(c2[w], q);
        n[q] = round_clamp_coeff(o.w1 * x1 + o.w2 * x2);  // (:55-56)
      }
      o.c[w] = __byte_perm(__byte_perm(n[0], n[1], 0x0040), __byte_perm(n[2], n[3], 0x0040), 0x5410);
    }
  }
  return o;
}

}  // namespace blz
