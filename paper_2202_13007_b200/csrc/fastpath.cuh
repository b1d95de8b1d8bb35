// fastpath.cuh -- helpers of the verified fast path for compress_block
// (H/codec.hpp:130-146); the kernel is compress_pair.cu.
//
// Bit-exactness argument:
//   * f (a copy) and s (serial row-major sum / count) are computed EXACTLY as
//     the reference does, with -fmad=false DADDs in the reference order.
//   * Everything after s only influences the output through integer decisions:
//     the 64 quantizer indices idx = clamp(rhaz(x)), phi = clamp(floor(127/m))
//     and the 28 coefficients C = clamp(rhaz(phi*d)).  Those are computed here
//     with fused arithmetic (DFMA, reciprocals, a DCT of the integer index grid)
//     together with a rigorous bound on |fast - reference| for every decision
//     variable.  If any decision variable lies within its bound of a decision
//     boundary, the block is handed to the exact kernel (compress_exact,
//     reference order), otherwise both computations provably take the same
//     branch and produce the same integers.
//   * Exotic values (inf/NaN deltas, subnormal or huge s, s_max, step) also go
//     to the exact kernel.
// The result is therefore identical to the reference bit for bit; the exact
// kernel is the rare path (its block count is reported by blz_ctx_stats).
#pragma once
#include "blaz_device.cuh"

namespace blz {

constexpr uint32_t NEED_EXACT = 0x80u;

// Kernel parameter block: basis plus ss00 = RN(sigma_0^2), sigma_0 = sum_u t(0,u)
// evaluated in extended precision on the host (only the DC term of
// T J T' is kept; the others are < 12 u |lo| and are part of the bound).
struct FastParams {
  Basis B;
  double ss00;
  uint32_t zero;  // always 0; keeps ptxas from merging the two halves' conversions
};

__device__ __forceinline__ uint32_t hi32(double x) { return (uint32_t)__double2hiint(x); }
__device__ __forceinline__ uint32_t lo32(double x) { return (uint32_t)__double2loint(x); }

// Decision helper.  For |y| < 2^19 returns n = floor(y + 0.5) (== rhaz(y)
// away from ties) and the distance of y + 0.5 to the nearest integer in units
// of 2^-32 (dist32).  t = y + (1.5*2^20 + 0.5) lies in [2^20, 2^21) where the
// ulp is 2^-32: its low word is frac(y + 0.5) * 2^32 and the low 20 bits of
// its high word are floor(y + 0.5) + 2^19 (exact up to the rounding of t,
// <= 2^-33, which the margins include).  Callers treat |y| >= 2^19 separately.
// Integer index -> double, volatile so the two DCT halves re-convert instead
// of keeping 64 converted doubles live (conversion pipe, not the FP64 pipe).
__device__ __forceinline__ double u8_to_double(uint32_t v) {
  double r;
  asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(r) : "r"(v));
  return r;
}

struct Decision {
  int n;
  uint32_t dist32;
};
__device__ __forceinline__ Decision decide(double y) {
  const double t = y + 1572864.5;
  Decision d;
  d.n = (int)(hi32(t) & 0xFFFFFu) - (1 << 19);
  const uint32_t fr = lo32(t);
  d.dist32 = min(fr, 0u - fr);
  return d;
}
__device__ __forceinline__ bool is_big(double y) {  // |y| >= 2^19, inf or NaN
  return (hi32(y) & 0x7FFFFFFFu) >= 0x41200000u;
}

// Margin (value units) -> 2^-32 units, +1 for the rounding of t.  Huge
// margins saturate so that every decision reads as "near".
__device__ __forceinline__ uint32_t margin32(double m) {
  if (!(m < 0.25)) return 0xFFFFFFFFu;
  return (uint32_t)__double2uint_ru(m * 4294967296.0) + 1u;
}

}  // namespace blz
