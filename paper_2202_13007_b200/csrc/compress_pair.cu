// compress_pair.cu -- K1 compress, verified fast path, two threads per block.
//
// Work split: a warp pair owns 32 consecutive blocks of the row-major block
// grid; lane L of the "upper" warp (h = 0) holds rows 0-3 of block L, lane L of
// the "lower" warp (h = 1) rows 4-7.  Everything the reference computes
// serially stays serial and in order:
//   * the mean-slope sum (H/codec.hpp:50-55) runs over rows 0-3 in the upper
//     thread, whose partial sum is handed to the lower thread which continues
//     over rows 4-7 -- the identical sequence of DADDs;
//   * the rest is the certified decision pipeline of fastpath.cuh, split by
//     rows of the transform (rows 0-3 of G = T K T' in the upper thread, rows
//     4-7 in the lower one) with the few shared quantities (s, s_max, the index
//     grid, max|d|) exchanged through shared memory between named barriers.
// Blocks whose decisions are not certified go to the exact worklist kernel.
// Halving the per-thread tile keeps the kernel at <= 128 registers (no
// spills), doubling resident warps versus one thread per block.
#include "blaz_device.cuh"
#include "fastpath.cuh"
#include "launch.h"

namespace blz {

constexpr int PAIR_WARPS = 4;  // 128-thread CTA = 2 warp pairs

struct PairShared {
  double sumA[32];
  double amax[2][32];
  int nz[2][32];
  double s[32];
  double smax[32];
  uint32_t idx[32][17];    // padded: 16 words + 1
  uint32_t gh[2][32];
  double d00[32];
  uint32_t cw[32][4];      // lower half coefficient words 4..6 + near flag
};

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

template <int H>
__device__ __forceinline__ void load_rows(const double* __restrict__ dense, uint64_t rows, uint64_t cols,
                                          uint64_t ld, uint64_t bi, uint64_t bj, bool vec, double (&m)[32]) {
  const uint64_t r0 = bi * BD + 4 * H, c0 = bj * BD;
  if (vec) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2* row = reinterpret_cast<const double2*>(dense + (r0 + i) * ld + c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = __ldg(row + q);
        m[i * BD + 2 * q] = v.x;
        m[i * BD + 2 * q + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t r = min(r0 + i, rows - 1);
#pragma unroll
      for (int j = 0; j < BD; ++j) m[i * BD + j] = __ldg(dense + r * ld + min(c0 + j, cols - 1));
    }
  }
}

// Fast 8-point DCT-II with exact-math constants (even/odd butterfly):
//   c[0] = 1/sqrt(8), c[k] = cos(k pi/16)/2 (k = 1..7), correctly rounded on the host.
// The fast path only needs |G_fast - T_hat K T_hat'| bounded: the
// glibc basis T_hat is within 4.3u of the exact cosines, which the bound E_d
// covers together with the butterfly's own rounding.
struct Butterfly {
  double c[8];
};

// Outputs 4H..4H+3 of the transform of the integer vector k[0..7].
template <int H>
__device__ __forceinline__ void dct8_int_half(const Butterfly& W, const int (&k)[8], double (&y)[4]) {
  const int s0 = k[0] + k[7], s1 = k[1] + k[6], s2 = k[2] + k[5], s3 = k[3] + k[4];
  const double d0 = (double)(k[0] - k[7]), d1 = (double)(k[1] - k[6]);
  const double d2 = (double)(k[2] - k[5]), d3 = (double)(k[3] - k[4]);
  const double e0 = (double)(s0 - s3), e1 = (double)(s1 - s2);
  const int p = s0 + s3, q = s1 + s2;
  if (H == 0) {
    y[0] = W.c[0] * (double)(p + q);
    y[1] = fma(W.c[1], d0, fma(W.c[3], d1, fma(W.c[5], d2, W.c[7] * d3)));
    y[2] = fma(W.c[2], e0, W.c[6] * e1);
    y[3] = fma(W.c[3], d0, -fma(W.c[7], d1, fma(W.c[1], d2, W.c[5] * d3)));
  } else {
    y[0] = W.c[4] * (double)(p - q);
    y[1] = fma(W.c[5], d0, fma(-W.c[1], d1, fma(W.c[7], d2, W.c[3] * d3)));
    y[2] = fma(W.c[6], e0, -(W.c[2] * e1));
    y[3] = fma(W.c[7], d0, fma(-W.c[5], d1, fma(W.c[3], d2, -(W.c[1] * d3))));
  }
}

// All 8 outputs of the transform of a double vector z[0..7].
__device__ __forceinline__ void dct8_f64(const Butterfly& W, const double (&z)[8], double (&y)[8]) {
  const double s0 = z[0] + z[7], s1 = z[1] + z[6], s2 = z[2] + z[5], s3 = z[3] + z[4];
  const double d0 = z[0] - z[7], d1 = z[1] - z[6], d2 = z[2] - z[5], d3 = z[3] - z[4];
  const double p = s0 + s3, q = s1 + s2, e0 = s0 - s3, e1 = s1 - s2;
  y[0] = W.c[0] * (p + q);
  y[4] = W.c[4] * (p - q);
  y[2] = fma(W.c[2], e0, W.c[6] * e1);
  y[6] = fma(W.c[6], e0, -(W.c[2] * e1));
  y[1] = fma(W.c[1], d0, fma(W.c[3], d1, fma(W.c[5], d2, W.c[7] * d3)));
  y[3] = fma(W.c[3], d0, -fma(W.c[7], d1, fma(W.c[1], d2, W.c[5] * d3)));
  y[5] = fma(W.c[5], d0, fma(-W.c[1], d1, fma(W.c[7], d2, W.c[3] * d3)));
  y[7] = fma(W.c[7], d0, fma(-W.c[5], d1, fma(W.c[3], d2, -(W.c[1] * d3))));
}

// One pass of the pipeline for the H half of block t (valid = t < nb).
template <int H>
__device__ __forceinline__ void pair_step(const FastParams& P, const Butterfly& W, const double* __restrict__ dense, uint64_t rows,
                                          uint64_t cols, uint64_t ld, const CMat& out, unsigned long long* err,
                                          uint64_t* __restrict__ wl, unsigned long long* __restrict__ wl_count,
                                          PairShared& sh, int lane, int bar, uint64_t t, bool valid) {
  const Basis& B = P.B;
  const uint64_t tt = valid ? t : 0;
  const uint64_t bi = tt / out.bc, bj = tt % out.bc;
  const bool vec = bi * BD + BD <= rows && bj * BD + BD <= cols && ((ld | (bj * BD)) & 1) == 0 &&
                   (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  double m[32];
  load_rows<H>(dense, rows, cols, ld, bi, bj, vec, m);
  double first = m[0];

  // ---- normalize (H/codec.hpp:20-32), reverse order in place -------------
  if (H == 0) {
#pragma unroll
    for (int i = 3; i >= 1; --i)
#pragma unroll
      for (int j = BD - 1; j >= 1; --j)
        m[i * BD + j] = ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) * 0.5;
#pragma unroll
    for (int i = 3; i >= 1; --i) m[i * BD] = m[i * BD] - m[(i - 1) * BD];
#pragma unroll
    for (int j = BD - 1; j >= 1; --j) m[j] = m[j] - m[j - 1];
    m[0] = 0.0;
  } else {
    double up[BD];  // row 3 (original values), an L1 hit after the upper warp's load
    {
      const uint64_t r3 = min(bi * BD + 3, rows - 1);
      if (vec) {
        const double2* row = reinterpret_cast<const double2*>(dense + r3 * ld + bj * BD);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 v = __ldg(row + q);
          up[2 * q] = v.x;
          up[2 * q + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < BD; ++j) up[j] = __ldg(dense + r3 * ld + min(bj * BD + j, cols - 1));
      }
    }
#pragma unroll
    for (int i = 3; i >= 0; --i)
#pragma unroll
      for (int j = BD - 1; j >= 1; --j) {
        const double a = m[i * BD + j];
        const double u = i ? m[(i - 1) * BD + j] : up[j];
        m[i * BD + j] = ((a - u) + (a - m[i * BD + j - 1])) * 0.5;
      }
#pragma unroll
    for (int i = 3; i >= 0; --i) m[i * BD] = m[i * BD] - (i ? m[(i - 1) * BD] : up[0]);
  }

  // ---- mean_slope: serial sum, rows 0-3 then rows 4-7 ----------------------
  double sum = 0.0, amax = 0.0;
  int nz = 0;
  if (H == 1) {
    pair_bar(bar);  // B1: upper partial sum ready
    sum = sh.sumA[lane];
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double a = fabs(m[k]);
    sum += a;
    nz += ((lo32(m[k]) | (hi32(m[k]) << 1)) != 0u);
    amax = a > amax ? a : amax;
  }
  sh.amax[H][lane] = amax;
  sh.nz[H][lane] = nz;
  if (H == 0) {
    sh.sumA[lane] = sum;
    pair_bar(bar);  // B1
  }
  pair_bar(bar);    // B2: both partial amax / nz visible
  amax = fmax(sh.amax[0][lane], sh.amax[1][lane]);
  nz = sh.nz[0][lane] + sh.nz[1][lane];
  if (H == 1) {
    // the lower thread holds the complete serial sum
    sh.s[lane] = (nz == 0) ? 0.0 : sum / (double)nz;
    sh.smax[lane] = sum;  // carry the sum itself for the finiteness test
  }
  pair_bar(bar);    // B3: s visible
  const double s = sh.s[lane];
  const double fullsum = sh.smax[lane];

  // status shared by both halves (identical inputs -> identical decisions)
  uint32_t status = DERR_NONE;
  const uint32_t es = (hi32(s) >> 20) & 0x7ff;
  if (!(fullsum <= 1.7976931348623157e308)) status = NEED_EXACT;  // non-finite input / overflow
  else if (s == 0.0) status = 0x40u;                              // constant block
  else if (es < 64 || es > 2000) status = NEED_EXACT;
  const double smax = amax / s;
  const double lo = s - smax;
  const double step = 2.0 * smax / 256;
  const uint32_t em = (hi32(smax) >> 20) & 0x7ff;
  if (status == DERR_NONE && (em < 64 || em > 2000)) status = NEED_EXACT;
  const double inv_s = 1.0 / s;
  const double inv_step = 1.0 / step;
  const double A = inv_s * inv_step;
  const double Bc = -lo * inv_step;
  const uint32_t mq_x = margin32(2.2737367544323206e-13 * (1.0 + fabs(lo) / smax));
  bool near = false;

  // ---- quantizer indices for the 32 own cells -----------------------------
  uint32_t idx[16];
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double x = fma(m[w * 4 + q], A, Bc);
      const Decision d = decide(x);
      const bool big = is_big(x);
      near |= !big && d.dist32 <= mq_x && (uint32_t)d.n <= 255u;
      int n = min(max(d.n, 0), 255);
      n = big ? ((hi32(x) >> 31) ? 0 : 255) : n;
      word |= (uint32_t)n << (8 * q);
    }
    sh.idx[lane][H * 8 + w] = word;
  }
  pair_bar(bar);    // B4: full index grid visible
#pragma unroll
  for (int w = 0; w < 16; ++w) idx[w] = sh.idx[lane][w];

  // ---- DCT of the index grid: pass 1 (columns, outputs 4H..4H+3), -------
  //      pass 2 (own rows), max|G| and the retained entries ----------------
  double tg[4][8];
#pragma unroll
  for (int v = 0; v < BD; ++v) {
    int kk[8];
#pragma unroll
    for (int u = 0; u < BD; ++u) kk[u] = (int)((idx[(u * BD + v) >> 2] >> (8 * ((u * BD + v) & 3))) & 0xffu);
    double y[4];
    dct8_int_half<H>(W, kk, y);
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) tg[ii][v] = y[ii];
  }
  uint32_t gh = 0;
  double G[20];  // retained entries of the own rows (H=0: 20, H=1: 8)
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    double g[8];
    dct8_f64(W, tg[ii], g);
    const int i = 4 * H + ii;
#pragma unroll
    for (int j = 0; j < BD; ++j) {
      if (i != 0 || j != 0) gh = max(gh, hi32(g[j]) & 0x7FFFFFFFu);
      if (H == 0) {
        if (i < 2) G[i * 8 + j] = g[j];
        else if (j < 2) G[16 + (i - 2) * 2 + j] = g[j];
      } else if (j < 2) {
        G[ii * 2 + j] = g[j];
      }
    }
  }
  sh.gh[H][lane] = gh;
  if (H == 0) sh.d00[lane] = fma(step, G[0], lo * P.ss00);
  pair_bar(bar);    // B5
  gh = max(sh.gh[0][lane], sh.gh[1][lane]);
  const double d00 = sh.d00[lane];
  const double gmax_lo = __hiloint2double((int)gh, 0);
  const double gmax_hi = __hiloint2double((int)(gh + 1u), 0);
  const double ad00 = fabs(d00);
  const double Ed = 4.440892098500626e-16 * (256.0 * fabs(lo) + 1024.0 * smax);
  const double m_lo = fmax(ad00, step * gmax_lo) * (1.0 - 2.3e-16) - Ed;
  const double m_hi = fmax(ad00, step * gmax_hi) * (1.0 + 2.3e-16) + Ed;
  if (status == DERR_NONE && (!(m_lo > 4.0 * Ed) || !(m_hi < 4.6e18))) status = NEED_EXACT;
  const double q_lo = (127.0 / m_hi) * (1.0 - 4.5e-16);
  const double q_hi = (127.0 / m_lo) * (1.0 + 4.5e-16);
  double phi = floor(q_lo);
  phi = phi < 1.0 ? 1.0 : (phi > 255.0 ? 255.0 : phi);
  double phi_hi = floor(q_hi);
  phi_hi = phi_hi < 1.0 ? 1.0 : (phi_hi > 255.0 ? 255.0 : phi_hi);
  if (status == DERR_NONE && phi != phi_hi) status = NEED_EXACT;

  // ---- coefficients of the own rows ----------------------------------------
  const double ps = phi * step;
  const uint32_t mq_c = margin32(phi * 2.0 * Ed + 5.6843418860808015e-14);
  uint32_t cw[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < KEPT; ++k) {
    const int r = krow(k), c = kcol(k);
    if ((r >> 2) != H) continue;
    const int gi = H == 0 ? (r < 2 ? r * 8 + c : 16 + (r - 2) * 2 + c) : (r - 4) * 2 + c;
    const double y = (r == 0 && c == 0) ? phi * d00 : G[gi] * ps;
    const Decision d = decide(y);
    const bool big = is_big(y);
    near |= !big && d.dist32 <= mq_c && (uint32_t)(d.n + 127) <= 254u;
    int n = min(max(d.n, -127), 127);
    n = big ? ((hi32(y) >> 31) ? -127 : 127) : n;
    put_coeff(cw, k, n);
  }
  if (H == 1) {
    sh.cw[lane][0] = cw[4];
    sh.cw[lane][1] = cw[5];
    sh.cw[lane][2] = cw[6];
    sh.cw[lane][3] = near ? 1u : 0u;
  }
  pair_bar(bar);    // B6
  if (H == 0 && valid) {
    cw[4] |= sh.cw[lane][0];
    cw[5] |= sh.cw[lane][1];
    cw[6] |= sh.cw[lane][2];
    near |= sh.cw[lane][3] != 0u;
    if (status == DERR_NONE && near) status = NEED_EXACT;
    RBlock rb;
    rb.f = first;
    rb.s = s;
    if (status == 0x40u) {  // constant block (:136)
      rb.phi = 1;
#pragma unroll
      for (int w = 0; w < 7; ++w) rb.c[w] = 0;
      store_block(out, t, rb);
    } else if (status == NEED_EXACT) {
      wl[atomicAdd(wl_count, 1ull)] = t;
    } else {
      rb.phi = (uint32_t)phi;
#pragma unroll
      for (int w = 0; w < 7; ++w) rb.c[w] = cw[w];
      store_block(out, t, rb);
    }
  }
  (void)err;
}

__global__ void __launch_bounds__(PAIR_WARPS * 32, 4) k_compress_pair(const FastParams P, const Butterfly W, const double* __restrict__ dense,
                                                                   uint64_t rows, uint64_t cols, uint64_t ld, CMat out,
                                                                   unsigned long long* err, uint64_t* __restrict__ wl,
                                                                   unsigned long long* __restrict__ wl_count) {
  __shared__ PairShared sh[PAIR_WARPS / 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, h = warp & 1;
  const int bar = 1 + pair;
  const uint64_t nb = out.nb();
  const uint64_t groups = (nb + 31) / 32;
  for (uint64_t g = (uint64_t)blockIdx.x * (PAIR_WARPS / 2) + pair; g < groups;
       g += (uint64_t)gridDim.x * (PAIR_WARPS / 2)) {
    const uint64_t t = g * 32 + lane;
    const bool valid = t < nb;
    if (h == 0)
      pair_step<0>(P, W, dense, rows, cols, ld, out, err, wl, wl_count, sh[pair], lane, bar, t, valid);
    else
      pair_step<1>(P, W, dense, rows, cols, ld, out, err, wl, wl_count, sh[pair], lane, bar, t, valid);
  }
}

cudaError_t launch_compress_pair(const LaunchCtx& c, const FastParams& P, const double* dense, uint64_t rows,
                                 uint64_t cols, uint64_t ld, const CMat& out) {
  Butterfly W;
  for (int k = 0; k < 8; ++k) W.c[k] = c.fast->bfly[k];
  const uint64_t groups = (out.nb() + 31) / 32;
  const uint64_t want = (groups + PAIR_WARPS / 2 - 1) / (PAIR_WARPS / 2);
  const uint64_t cap = (uint64_t)c.sm_count * 32;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  k_compress_pair<<<g, PAIR_WARPS * 32, 0, c.stream>>>(P, W, dense, rows, cols, ld, out, c.err, c.wl, c.wl_count);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
