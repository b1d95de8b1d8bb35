// fastpath.cuh -- verified fast path for compress_block (H/codec.hpp:130-146).
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

// Rows 4*HALF .. 4*HALF+3 of G = T K T' (column-outer), keeping the retained
// entries in gk and the high-word max of |G| (k != 0) in gh.
template <int HALF>
__device__ __forceinline__ void dct_half(const Basis& B, const uint32_t (&idx)[16], uint32_t zero, double (&gk)[KEPT],
                                         uint32_t& gh) {
  double G[32];
#pragma unroll
  for (int v = 0; v < BD; ++v) {
    double kc[BD];
#pragma unroll
    for (int u = 0; u < BD; ++u)
      kc[u] = u8_to_double(((idx[(u * BD + v) >> 2] >> (8 * ((u * BD + v) & 3))) & 0xffu) + (HALF ? zero : 0u));
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = HALF * 4 + ii;
      double tg = B.t[i * BD] * kc[0];
#pragma unroll
      for (int u = 1; u < BD; ++u) tg = fma(B.t[i * BD + u], kc[u], tg);
#pragma unroll
      for (int j = 0; j < BD; ++j) {
        if (v == 0)
          G[ii * BD + j] = tg * B.t[j * BD + v];
        else
          G[ii * BD + j] = fma(tg, B.t[j * BD + v], G[ii * BD + j]);
      }
    }
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = HALF * 4 + ii;
#pragma unroll
    for (int j = 0; j < BD; ++j) {
      if (i != 0 || j != 0) gh = max(gh, hi32(G[ii * BD + j]) & 0x7FFFFFFFu);
      if (i < 2) gk[i * 8 + j] = G[ii * BD + j];
      else if (j == 0) gk[14 + i] = G[ii * BD + j];
      else if (j == 1) gk[20 + i] = G[ii * BD + j];
    }
  }
}

__device__ __forceinline__ uint32_t compress_fast(double (&m)[BC], const FastParams& P, RBlock& out) {
  const Basis& B = P.B;
  out.phi = 1;
#pragma unroll
  for (int w = 0; w < 7; ++w) out.c[w] = 0;
  out.f = m[0];
  out.s = 0.0;

  // normalize (H/codec.hpp:20-32): exact, reverse order in place; x/2.0 == x*0.5.
#pragma unroll
  for (int i = BD - 1; i >= 1; --i)
#pragma unroll
    for (int j = BD - 1; j >= 1; --j)
      m[i * BD + j] = ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) * 0.5;
#pragma unroll
  for (int i = BD - 1; i >= 1; --i) m[i * BD] = m[i * BD] - m[(i - 1) * BD];
#pragma unroll
  for (int j = BD - 1; j >= 1; --j) m[j] = m[j] - m[j - 1];
  m[0] = 0.0;

  // mean_slope (H/codec.hpp:47-57).  Adding |delta| = +0.0 to the running sum
  // (which starts at +0.0 and is never -0.0) is the identity, so the serial
  // sum over all 64 entries equals the reference's sum over nonzero entries.
  double sum = 0.0, amax = 0.0;
  int nz = 0;
#pragma unroll
  for (int k = 0; k < BC; ++k) {
    const double a = fabs(m[k]);
    sum += a;
    nz += ((lo32(m[k]) | (hi32(m[k]) << 1)) != 0u);
    amax = a > amax ? a : amax;
  }
  // A non-finite input always leaves a non-finite delta, hence a non-finite
  // sum; such blocks (and overflowing finite ones) take the exact kernel, which
  // performs the reference's all_finite check (H/codec.hpp:21).
  if (!(sum <= 1.7976931348623157e308)) return NEED_EXACT;
  const double s = nz == 0 ? 0.0 : sum / (double)nz;
  out.s = s;
  if (s == 0.0) return DERR_NONE;  // constant block (:136)
  const uint32_t es = (hi32(s) >> 20) & 0x7ff;
  if (es < 64 || es > 2000) return NEED_EXACT;

  // s_max = max_k RN(|delta_k| / s) = RN(max|delta| / s)  (RN and /s are monotone)
  const double smax = amax / s;
  const double lo = s - smax;                 // (:90) the reference's operation
  const double step = 2.0 * smax / 256;       // (:91) the reference's operation
  const uint32_t em = (hi32(smax) >> 20) & 0x7ff;
  if (em < 64 || em > 2000) return NEED_EXACT;
  const double inv_s = 1.0 / s;
  const double inv_step = 1.0 / step;
  const double A = inv_s * inv_step;
  const double Bc = -lo * inv_step;
  // |x_fast - x_ref| <= 2^-42 (1 + |lo|/s_max)
  const uint32_t mq_x = margin32(2.2737367544323206e-13 * (1.0 + fabs(lo) / smax));
  bool near = false;

  // quantizer indices (H/codec.hpp:61-71, :92-96): idx = clamp(rhaz(x), 0, 255).
  // Boundaries that can change the clamped index: x + 0.5 = N, 1 <= N <= 255;
  // flagging "near" for n in [0, 255] covers them (and two harmless extras).
  uint32_t idx[16];
#pragma unroll
  for (int w = 0; w < 16; ++w) idx[w] = 0;
#pragma unroll
  for (int k = 0; k < BC; ++k) {
    const double x = fma(m[k], A, Bc);
    const Decision d = decide(x);
    const bool big = is_big(x);
    near |= !big && d.dist32 <= mq_x && (uint32_t)d.n <= 255u;
    int n = min(max(d.n, 0), 255);
    n = big ? ((hi32(x) >> 31) ? 0 : 255) : n;
    idx[k >> 2] |= (uint32_t)n << (8 * (k & 3));
  }

  // DCT of the integer index grid, G = T K T', in two halves of 4 rows
  // (column-outer within a half) so that only 32 accumulators are live; the
  // retained entries and the high-word max of |G| (k != 0) are kept.
  double gk[KEPT];
  uint32_t gh = 0;
  dct_half<0>(B, idx, P.zero, gk, gh);
  dct_half<1>(B, idx, P.zero, gk, gh);
  // d = lo*sigma sigma' + step*G; only the DC term of sigma sigma' is kept.
  const double d00 = fma(step, gk[0], lo * P.ss00);
  // m = max|d| (H/codec.hpp:110) bracketed from the high words of |G|:
  // gmax_lo <= max|G_k| (k != 0) < gmax_hi, relative width < 2^-19.
  const double gmax_lo = __hiloint2double((int)gh, 0);
  const double gmax_hi = __hiloint2double((int)(gh + 1u), 0);
  const double ad00 = fabs(d00);
  // |d_fast - d_ref| <= Ed per entry
  const double Ed = 4.440892098500626e-16 * (256.0 * fabs(lo) + 512.0 * smax);
  const double m_lo = fmax(ad00, step * gmax_lo) * (1.0 - 2.3e-16) - Ed;
  const double m_hi = fmax(ad00, step * gmax_hi) * (1.0 + 2.3e-16) + Ed;
  if (!(m_lo > 4.0 * Ed) || !(m_hi < 4.6e18)) return NEED_EXACT;

  // phi = clamp(floor(127 / m), 1, 255) (:116-119): certified when the whole
  // interval [127/m_hi, 127/m_lo] floors to the same clamped integer.
  const double q_lo = (127.0 / m_hi) * (1.0 - 4.5e-16);
  const double q_hi = (127.0 / m_lo) * (1.0 + 4.5e-16);
  double phi = floor(q_lo);
  phi = phi < 1.0 ? 1.0 : (phi > 255.0 ? 255.0 : phi);
  double phi_hi = floor(q_hi);
  phi_hi = phi_hi < 1.0 ? 1.0 : (phi_hi > 255.0 ? 255.0 : phi_hi);
  if (phi != phi_hi) return NEED_EXACT;
  out.phi = (uint32_t)phi;

  // C[k] = clamp_coeff(rhaz(phi * d(keep_k)))  (:120-123).  Boundaries that
  // can change the clamped value: y + 0.5 = N, -126 <= N <= 127; flagging
  // n in [-127, 127] covers them.
  const double ps = phi * step;
  const uint32_t mq_c = margin32(phi * 2.0 * Ed + 5.6843418860808015e-14);
#pragma unroll
  for (int k = 0; k < KEPT; ++k) {
    const int r = krow(k), c = kcol(k);
    (void)r;
    (void)c;
    const double y = (r == 0 && c == 0) ? phi * d00 : gk[k] * ps;
    const Decision d = decide(y);
    const bool big = is_big(y);
    near |= !big && d.dist32 <= mq_c && (uint32_t)(d.n + 127) <= 254u;
    int n = min(max(d.n, -127), 127);
    n = big ? ((hi32(y) >> 31) ? -127 : 127) : n;
    put_coeff(out.c, k, n);
  }
  if (near) return NEED_EXACT;
  return DERR_NONE;
}

}  // namespace blz
