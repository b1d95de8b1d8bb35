// compress_pair.cu -- K1 compress, verified fast path, two threads per block.
//
// Work split: a warp pair owns 32 consecutive blocks of the row-major block
// grid; lane L of the "upper" warp (h = 0) holds rows 0-3 of block L, lane L of
// the "lower" warp (h = 1) rows 4-7.  h is warp-uniform, and both halves run
// ONE code path (per-half constants come from a parameter table), which keeps
// the kernel's instruction footprint small.  Everything the reference computes
// serially stays serial and in order:
//   * the mean-slope sum (H/codec.hpp:50-55) runs over rows 0-3 in the upper
//     thread, whose partial sum is handed to the lower thread which continues
//     over rows 4-7 -- the identical sequence of DADDs;
//   * the rest is the certified decision pipeline of fastpath.cuh: quantizer
//     indices, a butterfly DCT of the integer index grid (outputs 0-3 of every
//     column in the upper thread, 4-7 in the lower one), phi and the retained
//     coefficients, with the shared quantities exchanged through shared memory.
// Records of the 32 blocks are staged in shared memory and written with
// coalesced 16-byte stores.  Blocks whose decisions are not certified are
// appended to the exact worklist (k_compress_worklist overwrites them).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "blaz_device.cuh"
#include "fastpath.cuh"
#include "launch.h"

#ifndef CMP_V4
#define CMP_V4 1  // 32-byte tile-row loads when the input allows them
#endif

namespace blz {

#ifndef CP_PAIR_WARPS
#define CP_PAIR_WARPS 2
#endif
#ifndef CP_MINB
#define CP_MINB 8
#endif
constexpr int PAIR_WARPS = CP_PAIR_WARPS;  // 64-thread CTA = one warp pair (8 CTAs / SM)

// Butterfly constants (exact-math DCT-II, correctly rounded on the host):
// c[0] = 1/sqrt(8), c[k] = cos(k pi/16)/2.  half[h] holds the pass-1
// coefficients of outputs 4h..4h+3 (see dct8_int_half).
struct Butterfly {
  double c[8];
  double half[2][11];
  double c2[2][8];  // pass-2 constants per half; the lower half's odd ones negated
};

#ifndef CP_GRID_MULT
#define CP_GRID_MULT 128  // CTAs per SM in the grid (8 resident): short-lived CTAs desynchronise the pairs
#endif
#ifndef CP_SIMD_P1
#define CP_SIMD_P1 1
#endif
#ifndef CP_COLSPLIT
#define CP_COLSPLIT 1
#endif
// CP_TMA: rows 0..CP_TMA_ROWS-1 of each warp's half tile of the NEXT group (32
// blocks = 256 columns) arrive by one TMA copy -- a 3-D view of the matrix, 16
// doubles x 16 column chunks x CP_TMA_ROWS rows, 128-byte swizzle so that the
// lanes' 16-byte reads 64 bytes apart are conflict-free -- completing on a
// per-warp mbarrier, issued as soon as the warp has read the current group's
// rows; the remaining row(s) and the lower half's row 3 are loaded directly.
// Three rows fit next to the pass-1 exchange buffer at 8 CTAs per SM
// (0.540 against 0.545 ms per 16384^2 without TMA; K1).  Used when the
// columns are a multiple of 256 (every group lies in one block-row).
#ifndef CP_TMA
#define CP_TMA 1
#endif
#ifndef CP_TMA_ROWS
#define CP_TMA_ROWS 3
#endif


struct PairShared {
  double sumA[32];
  double amax[2][32];
  int nz[2][32];
  double s[32];
  uint32_t idx[32][17];     // 16 words + 1 pad
  uint32_t gh[2][32];
  double d00[32];
  uint32_t nearL[32];
  uint8_t cbytes[32 * 28];  // staged coefficient records of the 32 blocks
#if CP_COLSPLIT
  double2 zx[2][8][32];     // pass-1 outputs for the other half's rows [writer][slot][lane]
#endif
};

// 1/a within 2u (faithful) for normal a in the ranges the status checks admit:
// the hardware approximation (~2^-22) refined by two Newton steps.  Blocks outside
// those ranges are marked NEED_EXACT, so their values here do not matter.
__device__ __forceinline__ double rcp_faithful(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// Certified decision on y (see fastpath.cuh::decide): t = y + 1.5*2^20 + 0.5
// lies in [2^20, 2^21) for |y| < 2^19, where its high word is
// 0x41380000 + floor(y + 0.5) and its low word frac(y + 0.5) * 2^32.
//  * the clamped result (range [LO, HI] around 0x41380000) is
//    min(max(hi, 0x41380000 + LO), 0x41380000 + HI); its LOW BYTE is the
//    two's-complement byte of the clamped integer (0x41380000 has a zero low
//    byte), and every out-of-range t (negative, < 2^20, >= 2^21) clamps to the
//    correct end;
//  * near: key = frac + m (mod 2^32) is < 2m exactly when the fraction is within
//    m of 0 or 1; the caller keeps the minimum key.  Keys of decisions whose high
//    word lies outside [LO, HI] are kept as well: they can only raise a spurious
//    "near" (a slower exact recompute), never hide one.  Such a decision cannot
//    differ from the reference's: the fast value is >= HI + 1/2 (resp. < LO - 1/2),
//    so with the certified error m < 1/2 the reference rounds to >= HI (<= LO) and
//    clamps to the same end.  (Magnitudes stay far below the int64 range where the
//    reference's conversion misbehaves: see the exponent and m_hi guards.)
//
// Callers pass t itself, formed by ONE fused operation: t = fma(g, ps, M) for a
// coefficient (one rounding to the 2^-32 grid instead of RN(y) then RN(y + M):
// strictly less error than the margin assumes) and t = fma(delta, A, Bc + M) for
// a quantizer index (RN(Bc + M) adds at most 2^-33, so that margin carries one
// more unit of 2^-32).
constexpr double kDecideM = 1572864.5;  // 1.5 * 2^20 + 0.5
template <int LO, int HI>
__device__ __forceinline__ uint32_t decide_byte(double t, uint32_t mq, uint32_t& kmin) {
  const int hi = (int)hi32(t);
  const int c = min(max(hi, 0x41380000 + LO), 0x41380000 + HI);
  kmin = min(kmin, lo32(t) + mq);
  return (uint32_t)c;  // callers take the low byte
}

// Outputs 4h..4h+3 of the 8-point transform of the integer vector k[0..7]:
// the butterflies run in exact integer arithmetic, then
//   y0 = hc0 (p +- q), y1 = odd row (hc3..6), y2 = hc1 e0 + hc2 e1, y3 = odd row (hc7..10).
__device__ __forceinline__ void dct8_int_half(const double (&hc)[11], int h, const int (&k)[8], double (&y)[4]) {
  const int s0 = k[0] + k[7], s1 = k[1] + k[6], s2 = k[2] + k[5], s3 = k[3] + k[4];
  const double d0 = (double)(k[0] - k[7]), d1 = (double)(k[1] - k[6]);
  const double d2 = (double)(k[2] - k[5]), d3 = (double)(k[3] - k[4]);
  const double e0 = (double)(s0 - s3), e1 = (double)(s1 - s2);
  const int p = s0 + s3, q = s1 + s2;
  y[0] = hc[0] * (double)(h ? p - q : p + q);
  y[1] = fma(hc[3], d0, fma(hc[4], d1, fma(hc[5], d2, hc[6] * d3)));
  y[2] = fma(hc[1], e0, hc[2] * e1);
  y[3] = fma(hc[7], d0, fma(hc[8], d1, fma(hc[9], d2, hc[10] * d3)));
}

// The FP64 part of dct8_int_half on converted butterfly values (pq = p + q for
// the upper outputs, p - q for the lower ones): the same operations, same order.
__device__ __forceinline__ void dct8_f64_half(const double (&hc)[11], double pq, const double (&d)[4], double e0,
                                              double e1, double (&y)[4]) {
  y[0] = hc[0] * pq;
  y[1] = fma(hc[3], d[0], fma(hc[4], d[1], fma(hc[5], d[2], hc[6] * d[3])));
  y[2] = fma(hc[1], e0, hc[2] * e1);
  y[3] = fma(hc[7], d[0], fma(hc[8], d[1], fma(hc[9], d[2], hc[10] * d[3])));
}

// Signed 16-bit lane l of w as a double (I2F.F64.S16 with a half selector).
__device__ __forceinline__ double s16_lane_to_f64(uint32_t w, int l) {
  unsigned short lo, hi;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(w));
  double d;
  asm("cvt.rn.f64.s16 %0, %1;" : "=d"(d) : "h"(l ? hi : lo));
  return d;
}

// All 8 outputs of the transform of a double vector z[0..7].
__device__ __forceinline__ void dct8_f64(const double (&c)[8], const double (&z)[8], double (&y)[8]) {
  const double s0 = z[0] + z[7], s1 = z[1] + z[6], s2 = z[2] + z[5], s3 = z[3] + z[4];
  const double d0 = z[0] - z[7], d1 = z[1] - z[6], d2 = z[2] - z[5], d3 = z[3] - z[4];
  const double p = s0 + s3, q = s1 + s2, e0 = s0 - s3, e1 = s1 - s2;
  y[0] = c[0] * (p + q);
  y[4] = c[4] * (p - q);
  y[2] = fma(c[2], e0, c[6] * e1);
  y[6] = fma(c[6], e0, -(c[2] * e1));
  y[1] = fma(c[1], d0, fma(c[3], d1, fma(c[5], d2, c[7] * d3)));
  y[3] = fma(c[3], d0, -fma(c[7], d1, fma(c[1], d2, c[5] * d3)));
  y[5] = fma(c[5], d0, fma(-c[1], d1, fma(c[7], d2, c[3] * d3)));
  y[7] = fma(c[7], d0, fma(-c[5], d1, fma(c[3], d2, -(c[1] * d3))));
}

__global__ void __launch_bounds__(PAIR_WARPS * 32, CP_MINB)
    k_compress_pair(const FastParams P, const Butterfly W, const double* __restrict__ dense, uint64_t rows,
                    uint64_t cols, uint64_t ld, CMat out, uint64_t* __restrict__ wl,
                    unsigned long long* __restrict__ wl_count, uint64_t step_q, uint64_t step_r
#if CP_TMA
                    , const __grid_constant__ CUtensorMap tmap, int use_tma
#endif
                    ) {
  __shared__ PairShared shared[PAIR_WARPS / 2];
#if CP_TMA
  constexpr int TR = CP_TMA_ROWS;
  __shared__ __align__(1024) double stile[PAIR_WARPS][TR * 256];
  __shared__ __align__(8) unsigned long long tbar[PAIR_WARPS];
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1;
  const int h = __shfl_sync(0xffffffffu, warp & 1, 0);  // warp-uniform half
  const int bar = 1 + pair;
  PairShared& sh = shared[pair];
  const uint64_t nb = out.nb();
  const uint64_t groups = (nb + 31) / 32;
  const bool aligned = ((ld & 1) == 0) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  const bool v4 = CMP_V4 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(dense) & 31) == 0;

  const uint64_t g0 = (uint64_t)blockIdx.x * (PAIR_WARPS / 2) + pair;
  const uint64_t gstep = (uint64_t)gridDim.x * (PAIR_WARPS / 2);
  BlockCursor cur(g0 * 32 + lane, out.bc, step_q, step_r);
#if CP_TMA
  const unsigned my_bar = (unsigned)__cvta_generic_to_shared(&tbar[warp]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(my_bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t tphase = 0;
  // group gg starts at lane 0's cursor block (bi0, bj0)
  auto tma_ok = [&](uint64_t gg, uint64_t bi0) -> bool {
    return use_tma && gg < groups && gg * 32 + 32 <= nb && bi0 * BD + BD <= rows;
  };
  auto tma_issue = [&](uint64_t bi0, uint64_t bj0) {
    if (lane == 0) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&stile[warp][0]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(my_bar), "r"(TR * 2048) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"((int)(bj0 / 2)), "r"((int)(bi0 * BD + 4 * h)),
          "r"(my_bar)
          : "memory");
    }
  };
  bool staged;
  {
    const uint64_t bi0 = __shfl_sync(0xffffffffu, cur.bi, 0), bj0 = __shfl_sync(0xffffffffu, cur.bj, 0);
    staged = tma_ok(g0, bi0);
    if (staged) tma_issue(bi0, bj0);
  }
  const int swz_line = lane >> 1, swz_x = (lane >> 1) & 7, swz_c = (lane & 1) * 4;
#endif
  for (uint64_t g = g0; g < groups; g += gstep, cur.advance(out.bc)) {
    const uint64_t t = g * 32 + lane;
    const bool valid = t < nb;
    const uint64_t bi = valid ? cur.bi : out.br - 1, bj = valid ? cur.bj : out.bc - 1;
    const uint64_t c0 = bj * BD;
    const bool vec = aligned && bi * BD + BD <= rows && c0 + BD <= cols;

    // ---- own rows + (lower half) row 3, original values, edge-replicated ---
    double m[32], up[8];
#if CP_TMA
    if (staged) {
      // rows TR.. and (lower half) row 3 straight from global memory, the rest from the TMA buffer
      const double* p = dense + (bi * BD + 4 * h) * ld + c0;
#pragma unroll
      for (int i = TR; i < 5; ++i) {
        if (i == 4 && h == 0) break;
        double x[BD];
        load_row8(i < 4 ? p + i * ld : p - ld, x, v4);
#pragma unroll
        for (int j = 0; j < BD; ++j) {
          if (i < 4) m[i * BD + j] = x[j];
          else up[j] = x[j];
        }
      }
      asm volatile(
          "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(
              my_bar),
          "r"(tphase)
          : "memory");
      const double* base = &stile[warp][0];
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 x = *reinterpret_cast<const double2*>(base + (i * 16 + swz_line) * 16 + ((swz_c + q) ^ swz_x) * 2);
          m[i * BD + 2 * q] = x.x;
          m[i * BD + 2 * q + 1] = x.y;
        }
      tphase ^= 1u;
    } else
#endif
    if (vec) {  // whole tile inside: one row pointer, rows at +ld
      const double* p = dense + (bi * BD + 4 * h) * ld + c0;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i == 4 && h == 0) break;
        double x[BD];
        load_row8(i < 4 ? p + i * ld : p - ld, x, v4);
#pragma unroll
        for (int j = 0; j < BD; ++j) {
          if (i < 4) m[i * BD + j] = x[j];
          else up[j] = x[j];
        }
      }
    } else {    // edge tile: clamped rows / columns (edge replication)
      const uint64_t r0 = bi * BD + 4 * h;
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i == 4 && h == 0) break;
        const uint64_t r = (i < 4) ? min(r0 + i, rows - 1) : min(bi * BD + 3, rows - 1);
        double v[8];
#pragma unroll
        for (int j = 0; j < BD; ++j) v[j] = __ldg(dense + r * ld + min(c0 + j, cols - 1));
#pragma unroll
        for (int j = 0; j < BD; ++j) {
          if (i < 4) m[i * BD + j] = v[j];
          else up[j] = v[j];
        }
      }
    }
    const double first = m[0];
#if CP_TMA
    BlockCursor tnx = cur;
    tnx.advance(out.bc);
    const uint64_t nbi0 = __shfl_sync(0xffffffffu, tnx.bi, 0), nbj0 = __shfl_sync(0xffffffffu, tnx.bj, 0);
    const bool staged_next = tma_ok(g + gstep, nbi0);
    if (staged_next) {  // own buffer: free once every lane has read it
      __syncwarp();
      tma_issue(nbi0, nbj0);
    }
#endif

    // ---- normalize (H/codec.hpp:20-32), reverse order in place ------------
#pragma unroll
    for (int i = 3; i >= 1; --i)
#pragma unroll
      for (int j = BD - 1; j >= 1; --j)
        m[i * BD + j] = ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) * 0.5;
#pragma unroll
    for (int i = 3; i >= 1; --i) m[i * BD] = m[i * BD] - m[(i - 1) * BD];
    if (h == 0) {  // global row 0: single predecessor, delta(0,0) = 0
#pragma unroll
      for (int j = BD - 1; j >= 1; --j) m[j] = m[j] - m[j - 1];
      m[0] = 0.0;
    } else {       // global row 4: the up neighbour is row 3
#pragma unroll
      for (int j = BD - 1; j >= 1; --j) m[j] = ((m[j] - up[j]) + (m[j] - m[j - 1])) * 0.5;
      m[0] = m[0] - up[0];
    }

    // ---- mean_slope: serial sum, rows 0-3 then rows 4-7 --------------------
    // (adding |delta| = +0.0 to the never -0.0 running sum is the identity, so
    // summing all entries equals the reference's sum over nonzero entries)
    // The upper thread runs its half of the sum first so that the lower one can
    // continue it while the upper computes max |delta| and the count.
    double sum = 0.0, amax = 0.0;
    if (h == 0) {
#pragma unroll
      for (int k = 0; k < 32; ++k) sum += fabs(m[k]);
      sh.sumA[lane] = sum;
      pair_bar(bar);  // B1: upper partial sum ready
    }
    // max |delta| (exact), and a zero test: the minimum of (|hi| | lo) over the
    // cells is 0 iff some delta is +-0 (delta(0,0) = 0 of the upper half is known).
    // The running maximum is kept as words: one FP64 compare and two 32-bit
    // selects per cell, the high word's sign cleared by the select's |.|.
    // Two independent chains (even / odd cells), merged at the end: the maximum
    // is exact in any order, and the split halves the compare-select latency.
    // zero test on the high words only, as floats (|hi| is monotone as a float bit
    // pattern; NaN patterns, |delta| >= 2^1017, are nonzero and ignored by fminf).
    // A zero high word with a nonzero low word (subnormal delta) only sends the
    // block through the exact count below.
    float zminf = 3.0e38f;
    float amax_h[2] = {0.0f, 0.0f};
    uint32_t amax_l[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int c = k & 1;
      const bool gt = fabs(m[k]) > __hiloint2double(__float_as_int(amax_h[c]), (int)amax_l[c]);
      amax_h[c] = gt ? fabsf(__int_as_float((int)hi32(m[k]))) : amax_h[c];
      amax_l[c] = gt ? lo32(m[k]) : amax_l[c];
      zminf = (k == 0 && h == 0) ? zminf : fminf(zminf, fabsf(__int_as_float((int)hi32(m[k]))));
    }
    {
      const bool gt = __hiloint2double(__float_as_int(amax_h[1]), (int)amax_l[1]) >
                      __hiloint2double(__float_as_int(amax_h[0]), (int)amax_l[0]);
      amax_h[0] = gt ? amax_h[1] : amax_h[0];
      amax_l[0] = gt ? amax_l[1] : amax_l[0];
    }
    amax = __hiloint2double(__float_as_int(amax_h[0]), (int)amax_l[0]);
    int nz = 32 - (h == 0);
    if (zminf == 0.0f) {  // some zero deltas (rare on real data): count them
      nz = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) nz += fabs(m[k]) > 0.0;
    }
    if (h == 1) {
      pair_bar(bar);  // B1
      sum = sh.sumA[lane];
#pragma unroll
      for (int k = 0; k < 32; ++k) sum += fabs(m[k]);
    }
    sh.amax[h][lane] = amax;
    sh.nz[h][lane] = nz;
    if (h == 1) sh.s[lane] = sum;  // the lower thread holds the complete serial sum
    pair_bar(bar);    // B2
    amax = fmax(sh.amax[0][lane], sh.amax[1][lane]);
    nz = sh.nz[0][lane] + sh.nz[1][lane];
    const double fullsum = sh.s[lane];
    const double s = (nz == 0) ? 0.0 : fullsum / (double)nz;

    // status shared by both halves (identical inputs -> identical decisions)
    uint32_t status = DERR_NONE;
    const uint32_t es = (hi32(s) >> 20) & 0x7ff;
    if (!(fullsum <= 1.7976931348623157e308)) status = NEED_EXACT;  // non-finite input / overflow
    else if (s == 0.0) status = 0x40u;                              // constant block (:136)
    else if (es < 64 || es > 2000) status = NEED_EXACT;
    const double smax = amax / s;              // = max_k RN(|delta_k| / s)
    const double lo = s - smax;                // (:90)
    const double step = 2.0 * smax / 256;      // (:91)
    const uint32_t em = (hi32(smax) >> 20) & 0x7ff;
    if (status == DERR_NONE && (em < 64 || em > 2000)) status = NEED_EXACT;
    // Faithful reciprocals (within 2u) for the fast-path factors; the margin below
    // is 2^-41 (1 + L), twice what correctly rounded ones need.
    const double inv_step = rcp_faithful(step);
    const double A = rcp_faithful(s) * inv_step;
    const double Bc = -lo * inv_step;
    const double BcM = Bc + kDecideM;  // rounded: <= 2^-33, the extra unit below
    // L = |lo| / s_max enters only the margin: |lo| * inv_step / 128 is within 3u of
    // it, far inside the bound's >= 2x slack (2^-42 (1 + L) against u (512 + 384 L)).
    uint32_t mq_x = margin32(4.547473508864641e-13 * (1.0 + fabs(lo) * inv_step * 0.0078125));
    mq_x += mq_x < 0x7FFFFFFFu ? 1u : 0u;
    if (mq_x >= 0x7FFFFFFFu) status = (status == DERR_NONE) ? NEED_EXACT : status;
    // min over decisions of (frac + m) mod 2^32, in two chains (odd / even cells)
    uint32_t kmin = 0xFFFFFFFFu, kmin2 = 0xFFFFFFFFu;

    // ---- quantizer indices for the 32 own cells ---------------------------
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = decide_byte<0, 255>(fma(m[w * 4 + q], A, BcM), mq_x, (q & 1) ? kmin2 : kmin);
      // low byte of each decision into one word (three byte permutes)
      sh.idx[lane][h * 8 + w] = __byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410);
    }
    kmin = min(kmin, kmin2);
    bool near = kmin < 2u * mq_x;
    pair_bar(bar);    // B3: full index grid visible

#if CP_COLSPLIT
    // ---- DCT of the index grid: pass 1 over this half's 4 columns ----------
    // Columns are taken in the order col(c) = h ? 7 - c : c.  All 8 outputs of a
    // column share one set of integer butterflies: the own rows' outputs use
    // half[h], the other half's rows half[1 - h] (the same formulas as
    // dct8_int_half, so every value is the one the row-split version computed).
    // own[ii][c] = Z(4h + ii, col(c)); the other rows' outputs go to shared memory.
    double own[4][4];
    {
      double ho[11], hx[11];
#pragma unroll
      for (int k = 0; k < 11; ++k) {
        ho[k] = W.half[h][k];
        hx[k] = W.half[1 - h][k];
      }
      uint32_t wv[8];
#pragma unroll
      for (int u = 0; u < BD; ++u) wv[u] = sh.idx[lane][u * 2 + h];
      double oth[4][4];
#if CP_SIMD_P1
      // Two columns per pass through the integer butterflies: 16-bit lanes of
      // one register (VIADD.16x2 / IADD3), each difference formed with a bias that
      // keeps the lower lane from borrowing and removed per lane; the lanes then
      // convert with I2F.F64.S16 (.H0 / .H1).  The integers are the same, so every
      // double is the one the scalar version computed.
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const uint32_t i0 = (uint32_t)(h ? 3 - 2 * pr : 2 * pr), i1 = (uint32_t)(h ? 2 - 2 * pr : 2 * pr + 1);
        const uint32_t sel = 0x4040u | (i1 << 8) | i0;  // bytes col(c0), col(c1) into lanes 0, 1
        uint32_t kw[8];
#pragma unroll
        for (int u = 0; u < BD; ++u) kw[u] = __byte_perm(wv[u], 0u, sel);
        uint32_t sw[4], dw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sw[j] = kw[j] + kw[7 - j];
          dw[j] = __vadd2(kw[j] - kw[7 - j] + 0x01000100u, 0xFF00FF00u);
        }
        const uint32_t e0w = __vadd2(sw[0] - sw[3] + 0x02000200u, 0xFE00FE00u);
        const uint32_t e1w = __vadd2(sw[1] - sw[2] + 0x02000200u, 0xFE00FE00u);
        const uint32_t pw = sw[0] + sw[3], qw = sw[1] + sw[2];
        const uint32_t ppq = pw + qw, pmq = __vadd2(pw - qw + 0x04000400u, 0xFC00FC00u);
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          double d[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) d[j] = s16_lane_to_f64(dw[j], l);
          const double e0 = s16_lane_to_f64(e0w, l), e1 = s16_lane_to_f64(e1w, l);
          const double vpq = s16_lane_to_f64(ppq, l), vmq = s16_lane_to_f64(pmq, l);
          double yo[4], yx[4];
          dct8_f64_half(ho, h ? vmq : vpq, d, e0, e1, yo);
          dct8_f64_half(hx, h ? vpq : vmq, d, e0, e1, yx);
          const int c = 2 * pr + l;
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) {
            own[ii][c] = yo[ii];
            oth[ii][c] = yx[ii];
          }
        }
      }
#else
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t sel = 0x4440u | (uint32_t)(h ? 3 - c : c);  // byte col(c) & 3, zero-extended
        int kk[8];
#pragma unroll
        for (int u = 0; u < BD; ++u) kk[u] = (int)__byte_perm(wv[u], 0u, sel);
        double yo[4], yx[4];
        dct8_int_half(ho, h, kk, yo);
        dct8_int_half(hx, 1 - h, kk, yx);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          own[ii][c] = yo[ii];
          oth[ii][c] = yx[ii];
        }
      }
#endif
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int q = 0; q < 2; ++q) sh.zx[h][ii * 2 + q][lane] = make_double2(oth[ii][2 * q], oth[ii][2 * q + 1]);
    }
    pair_bar(bar);    // B3b: the other half's pass-1 outputs visible
    // ---- pass 2 (own rows), max|G| and the retained entries ---------------
    // Row ii of Z in butterfly form: z[j] + z[7-j] = own[j] + B[j] and
    // z[j] - z[7-j] = +-(own[j] - B[j]) (sign - for h = 1, folded into c2[1]).
    float ghf = 0.0f;  // max over |G| high words, as a float (|G| < 2^12: never a NaN pattern)
    double G[20];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      double B[4];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 x = sh.zx[1 - h][ii * 2 + q][lane];
        B[2 * q] = x.x;
        B[2 * q + 1] = x.y;
      }
      double z[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        z[j] = own[ii][j];
        z[7 - j] = B[j];
      }
      double gr[8];
      dct8_f64(W.c2[h], z, gr);
#pragma unroll
      for (int j = 0; j < BD; ++j) {
        ghf = (ii == 0 && j == 0 && h == 0) ? ghf : fmaxf(ghf, fabsf(__int_as_float((int)hi32(gr[j]))));
        if (ii < 2) G[ii * 8 + j] = gr[j];
        else if (j < 2) G[16 + (ii - 2) * 2 + j] = gr[j];
      }
    }
#else
    // ---- DCT of the index grid: pass 1 (columns, outputs 4h..4h+3) --------
    double hc[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) hc[k] = W.half[h][k];
    double tg[4][8];
#pragma unroll
    for (int v = 0; v < BD; ++v) {
      int kk[8];
#pragma unroll
      for (int u = 0; u < BD; ++u) {
        const uint32_t wv = sh.idx[lane][(u * BD + v) >> 2];
        kk[u] = (int)((wv >> (8 * ((u * BD + v) & 3))) & 0xffu);
      }
      double y[4];
      dct8_int_half(hc, h, kk, y);
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) tg[ii][v] = y[ii];
    }
    // ---- pass 2 (own rows), max|G| and the retained entries ---------------
    // G[0..15]: local rows 0,1 (all columns); G[16..19]: local rows 2,3, cols 0,1
    uint32_t gh = 0;
    double G[20];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      double gr[8];
      dct8_f64(W.c, tg[ii], gr);
#pragma unroll
      for (int j = 0; j < BD; ++j) {
        const uint32_t a = hi32(gr[j]) & 0x7FFFFFFFu;
        gh = (ii == 0 && j == 0 && h == 0) ? gh : max(gh, a);
        if (ii < 2) G[ii * 8 + j] = gr[j];
        else if (j < 2) G[16 + (ii - 2) * 2 + j] = gr[j];
      }
    }
#endif
#if CP_COLSPLIT
    uint32_t gh = (uint32_t)__float_as_int(ghf);
#endif
    sh.gh[h][lane] = gh;
    if (h == 0) sh.d00[lane] = fma(step, G[0], lo * P.ss00);
    pair_bar(bar);    // B4
    gh = max(sh.gh[0][lane], sh.gh[1][lane]);
    const double d00 = sh.d00[lane];
    const double ad00 = fabs(d00);
    // |d_fast - d_ref| <= Ed per entry
    const double Ed = 4.440892098500626e-16 * (256.0 * fabs(lo) + 1024.0 * smax);
    const double m_lo = fmax(ad00, step * __hiloint2double((int)gh, 0)) * (1.0 - 2.3e-16) - Ed;
    const double m_hi = fmax(ad00, step * __hiloint2double((int)(gh + 1u), 0)) * (1.0 + 2.3e-16) + Ed;
    if (status == DERR_NONE && (!(m_lo > 4.0 * Ed) || !(m_hi < 4.6e18))) status = NEED_EXACT;
    // No division: 127/m_lo = (127/m_hi) / (1 - x), x = (m_hi - m_lo)/m_hi, is at
    // most R (1 + x + 2x^2) for x <= 1/2; x is taken from R as (m_hi - m_lo) R / 127.
    // The computed upper end carries every rounding (<= 14u) and the reference's own
    // rounding of 127/m (u) inside the factor 1 + 2e-15 (18u); the lower end's factor
    // 1 - 1e-15 (9u) covers R's 3u, one multiply and the reference's rounding.
    const double R = 127.0 * rcp_faithful(m_hi);  // within 3u of 127 / m_hi
    double phi = floor(R * (1.0 - 1e-15));
    phi = phi < 1.0 ? 1.0 : (phi > 255.0 ? 255.0 : phi);
    const double xq = (m_hi - m_lo) * R * 0.007874015748031496;
    if (status == DERR_NONE && !(xq < 0.25)) status = NEED_EXACT;
    double phi_hi = floor(R * (1.0 + fma(2.0 * xq, xq, xq)) * (1.0 + 2e-15));
    phi_hi = phi_hi < 1.0 ? 1.0 : (phi_hi > 255.0 ? 255.0 : phi_hi);
    if (status == DERR_NONE && phi != phi_hi) status = NEED_EXACT;

    // ---- retained coefficients (H/codec.hpp:120-123) -----------------------
    const double ps = phi * step;
    const uint32_t mq_c = margin32(phi * 2.0 * Ed + 5.6843418860808015e-14);
    if (mq_c >= 0x7FFFFFFFu) status = (status == DERR_NONE) ? NEED_EXACT : status;
    const bool zero_c = (status == 0x40u);  // constant block: all coefficients 0
    uint8_t* cb = sh.cbytes + lane * 28;
    kmin = 0xFFFFFFFFu;
    // Decisions of local rows 0..3, columns 0,1 (both halves) and, in the upper
    // half, rows 0,1, columns 2..7; the low byte of each is the coefficient byte.
    // Keep-set positions (global row r = 4h + ii): k = 8r + c for r < 2,
    // 14 + r (c = 0) and 20 + r (c = 1) otherwise.  Bytes are packed with PRMT and
    // stored as words / half-words.
    uint32_t cbv[4][2];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double gv = ii < 2 ? G[ii * 8 + c] : G[16 + (ii - 2) * 2 + c];
        const double t = (h == 0 && ii == 0 && c == 0) ? fma(phi, d00, kDecideM) : fma(gv, ps, kDecideM);
        cbv[ii][c] = decide_byte<-127, 127>(t, mq_c, kmin);
      }
    const uint32_t zm = zero_c ? 0u : 0xFFFFFFFFu;
    auto pack4 = [](uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
      return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
    };
    if (h == 0) {
      uint32_t rb[2][8];
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        rb[ii][0] = cbv[ii][0];
        rb[ii][1] = cbv[ii][1];
#pragma unroll
        for (int c = 2; c < 8; ++c) rb[ii][c] = decide_byte<-127, 127>(fma(G[ii * 8 + c], ps, kDecideM), mq_c, kmin);
      }
      uint32_t* cw = reinterpret_cast<uint32_t*>(cb);
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        cw[2 * ii] = pack4(rb[ii][0], rb[ii][1], rb[ii][2], rb[ii][3]) & zm;
        cw[2 * ii + 1] = pack4(rb[ii][4], rb[ii][5], rb[ii][6], rb[ii][7]) & zm;
      }
      *reinterpret_cast<uint16_t*>(cb + 16) = (uint16_t)(__byte_perm(cbv[2][0], cbv[3][0], 0x0040) & zm);
      *reinterpret_cast<uint16_t*>(cb + 22) = (uint16_t)(__byte_perm(cbv[2][1], cbv[3][1], 0x0040) & zm);
    } else {
      *reinterpret_cast<uint16_t*>(cb + 18) = (uint16_t)(__byte_perm(cbv[0][0], cbv[1][0], 0x0040) & zm);
      *reinterpret_cast<uint16_t*>(cb + 20) = (uint16_t)(__byte_perm(cbv[2][0], cbv[3][0], 0x0040) & zm);
      *reinterpret_cast<uint32_t*>(cb + 24) = pack4(cbv[0][1], cbv[1][1], cbv[2][1], cbv[3][1]) & zm;
    }
    near |= kmin < 2u * mq_c;
    if (h == 1) sh.nearL[lane] = near ? 1u : 0u;
    pair_bar(bar);    // B5: coefficient bytes and the lower near flag visible

    // ---- store the 32 records (coalesced) ----------------------------------
    if (h == 0) {
      near |= sh.nearL[lane] != 0u;
      if (status == DERR_NONE && near) status = NEED_EXACT;
      if (valid) {
        if (status == NEED_EXACT) wl[atomicAdd(wl_count, 1ull)] = t;
        out.first[t] = first;
        out.slope[t] = s;
        out.scale[t] = (uint8_t)(zero_c ? 1u : (uint32_t)phi);
      }
    }
    const uint64_t t0 = g * 32;
    if (t0 + 32 <= nb) {  // 32 x 28 = 896 bytes = 56 16-byte chunks
      const int chunk = h * 32 + lane;
      if (chunk < 56)
        reinterpret_cast<uint4*>(out.coeffs + t0 * 28)[chunk] = reinterpret_cast<const uint4*>(sh.cbytes)[chunk];
    } else if (h == 0 && valid) {
      for (int k = 0; k < 28; ++k) out.coeffs[t * 28 + k] = cb[k];
    }
    pair_bar(bar);    // B6: staging buffer free for the next group
#if CP_TMA
    staged = staged_next;
#endif
  }
}

cudaError_t launch_compress_pair(const LaunchCtx& c, const FastParams& P, const double* dense, uint64_t rows,
                                 uint64_t cols, uint64_t ld, const CMat& out) {
  Butterfly W;
  for (int k = 0; k < 8; ++k) W.c[k] = c.fast->bfly[k];
  const double* C = W.c;
  // upper half: outputs 0,1,2,3 ; lower half: outputs 4,5,6,7 (as in dct8_f64)
  const double up[11] = {C[0], C[2], C[6], C[1], C[3], C[5], C[7], C[3], -C[7], -C[1], -C[5]};
  const double lw[11] = {C[4], C[6], -C[2], C[5], -C[1], C[7], C[3], C[7], -C[5], C[3], -C[1]};
  for (int k = 0; k < 11; ++k) {
    W.half[0][k] = up[k];
    W.half[1][k] = lw[k];
  }
  for (int k = 0; k < 8; ++k) {
    W.c2[0][k] = C[k];
    W.c2[1][k] = (k & 1) ? -C[k] : C[k];
  }
  const uint64_t groups = (out.nb() + 31) / 32;
  const uint64_t want = (groups + PAIR_WARPS / 2 - 1) / (PAIR_WARPS / 2);
  const uint64_t cap = (uint64_t)c.sm_count * CP_GRID_MULT;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  const uint64_t stride = (uint64_t)g * (PAIR_WARPS / 2) * 32;  // blocks per grid-stride step
#if CP_TMA
  CUtensorMap tmap{};
  int use_tma = 0;
  if (cols % 256 == 0 && (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(dense) & 15) == 0 && rows >= 8) {
    // the driver's tensor-map encoder, looked up once (thread-safe static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (encode) {
      const cuuint64_t dims[3] = {16, cols / 16, rows};
      const cuuint64_t strides[2] = {128, ld * 8};
      const cuuint32_t box[3] = {16, 16, CP_TMA_ROWS};
      const cuuint32_t estr[3] = {1, 1, 1};
      use_tma = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(dense), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  k_compress_pair<<<g, PAIR_WARPS * 32, 0, c.stream>>>(P, W, dense, rows, cols, ld, out, c.wl, c.wl_count,
                                                       stride / out.bc, stride % out.bc, tmap, use_tma);
#else
  k_compress_pair<<<g, PAIR_WARPS * 32, 0, c.stream>>>(P, W, dense, rows, cols, ld, out, c.wl, c.wl_count,
                                                       stride / out.bc, stride % out.bc);
#endif
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
