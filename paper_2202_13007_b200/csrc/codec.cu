// codec.cu -- K1 compress / K2 decompress kernels (exact mode).
//
// compress_matrix (H/matrix.hpp:97-111) and decompress_matrix (:113-126):
// one thread owns one 8x8 block of the row-major block grid; the per-block
// arithmetic is blaz_device.cuh.
#include "blaz_device.cuh"
#include "fastpath.cuh"  // FastParams, NEED_EXACT
#include "launch.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#ifndef DEC_UB
#define DEC_UB 1  // k_decompress_ub for aligned outputs (0: k_decompress everywhere; A/B builds)
#endif
#ifndef DEC_UB_THREADS
#define DEC_UB_THREADS 32  // one-warp CTAs: 32 / 64 / 128 / 256 threads 0.4365 / 0.4386 / 0.442 / 0.463 ms
#endif
#ifndef DEC_UB_MINB
#define DEC_UB_MINB (640 / DEC_UB_THREADS)  // CTAs per SM the register allocation targets: 20 warps (16: 0.4327 ms, 20: 0.4293; 24 spills)
#endif
#ifndef DEC_UB_STORE_AFTER
#define DEC_UB_STORE_AFTER 2  // row stores from the shared row: 0 in the pair loop 0.558 ms, 1 after it 0.540, 2 row u-1 during row u 0.531
#endif
#ifndef DEC_UB_V4
#define DEC_UB_V4 1  // 32-byte row stores (STG.E.ENL2.256) when the output allows them: 0.531 -> 0.442 ms
#endif
#ifndef DEC_UB_PF
#define DEC_UB_PF 1184  // L2 prefetch distance of the records in CTAs (0: none; 592-2368: 0.4325 ms, none 0.4366, 4736: 0.4405)
#endif
#ifndef DEC_UB_PER_THREAD
#define DEC_UB_PER_THREAD 1  // blocks per thread of k_decompress_ub (straight-line copies; 2 / 3: 0.599 / 0.615 ms against 0.558)
#endif
#ifndef DEC_GRID_PER_SM
#define DEC_GRID_PER_SM 128  // short-lived CTAs: 4 / 8 / 32 / 64 / 128 / 256 per SM: 0.589 / 0.586 / 0.575 / 0.561 / 0.560 / 0.568 ms
#endif

namespace blz {

// Edge-replicated tile load (H/matrix.hpp:72-84).
__device__ __forceinline__ void load_tile(const double* __restrict__ dense, uint64_t rows, uint64_t cols,
                                          uint64_t ld, uint64_t bi, uint64_t bj, double (&m)[BC]) {
  const uint64_t r0 = bi * BD, c0 = bj * BD;
  if (r0 + BD <= rows && c0 + BD <= cols && ((ld | c0) & 1) == 0 &&
      (reinterpret_cast<uintptr_t>(dense) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < BD; ++i) {
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
    for (int i = 0; i < BD; ++i) {
      const uint64_t r = min(r0 + i, rows - 1);
#pragma unroll
      for (int j = 0; j < BD; ++j) {
        const uint64_t c = min(c0 + j, cols - 1);
        m[i * BD + j] = __ldg(dense + r * ld + c);
      }
    }
  }
}

// Exact compress (reference order) of every block -- mode BLZ_MODE_EXACT.
__global__ void __launch_bounds__(128) k_compress(const Basis B, const double* __restrict__ dense,
                                                  uint64_t rows, uint64_t cols, uint64_t ld, CMat out,
                                                  unsigned long long* err) {
  const uint64_t nb = out.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t bi = t / out.bc, bj = t % out.bc;
    double m[BC];
    load_tile(dense, rows, cols, ld, bi, bj, m);
    RBlock rb;
    const uint32_t e = compress_exact(m, B, rb);
    if (e != DERR_NONE) latch_error(err, t, e);
    store_block(out, t, rb);
  }
}

// Warp-uniform loop (valid lanes predicated) so that the basis streams through
// uniform registers (LDCU.128) rather than per-thread constant loads.
template <bool SYM>
__global__ void __launch_bounds__(128, 4) k_decompress(const Basis B, CMat in, double* __restrict__ dense,
                                                       uint64_t ld, uint64_t crop_rows, uint64_t crop_cols) {
  const uint64_t nb = in.nb();
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool aligned = ((ld & 1) == 0) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  const bool v4 = rows_v4(dense, ld);
  for (uint64_t base = warp0 * 32; base < nb; base += nwarps * 32) {
    const uint64_t t = base + lane;
    const bool valid = t < nb;
    const uint64_t tt = valid ? t : nb - 1;
    const uint64_t bi = tt / in.bc, bj = tt % in.bc;
    const RBlock rb = load_block(in, tt);
    const uint64_t r0 = bi * BD, c0 = bj * BD;
    const bool full = valid && aligned && r0 + BD <= crop_rows && c0 + BD <= crop_cols;
    decompress_exact<SYM>(rb, B, [&](int u, const double (&row)[BD]) {
      if (full) {
        store_row8(dense + (r0 + u) * ld + c0, row, v4);
      } else if (valid && r0 + u < crop_rows) {
#pragma unroll
        for (int j = 0; j < BD; ++j)
          if (c0 + j < crop_cols) dense[(r0 + u) * ld + c0 + j] = row[j];
      }
    });
  }
}

// Fused all-gather + decompress: the same per-block work as k_decompress, the
// record of block (bi, bj) read from the shard owning block-row bi -- a peer
// GPU's memory over NVLink when the shards are other ranks' arrays.
template <bool SYM>
__global__ void __launch_bounds__(128, 4) k_decompress_gather(const Basis B, const ShardSet S, uint64_t bc,
                                                              double* __restrict__ dense, uint64_t ld,
                                                              uint64_t crop_rows, uint64_t crop_cols) {
  const uint64_t nb = S.lo[S.n] * bc;
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool aligned = ((ld & 1) == 0) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  const bool v4 = rows_v4(dense, ld);
  for (uint64_t base = warp0 * 32; base < nb; base += nwarps * 32) {
    const uint64_t t = base + lane;
    const bool valid = t < nb;
    const uint64_t tt = valid ? t : nb - 1;
    const uint64_t bi = tt / bc, bj = tt % bc;
    int r = 0;
    while (r + 1 < S.n && bi >= S.lo[r + 1]) ++r;
    const RBlock rb = load_block(S.part[r], (bi - S.lo[r]) * bc + bj);
    const uint64_t r0 = bi * BD, c0 = bj * BD;
    const bool full = valid && aligned && r0 + BD <= crop_rows && c0 + BD <= crop_cols;
    decompress_exact<SYM>(rb, B, [&](int u, const double (&row)[BD]) {
      if (full) {
        store_row8(dense + (r0 + u) * ld + c0, row, v4);
      } else if (valid && r0 + u < crop_rows) {
#pragma unroll
        for (int j = 0; j < BD; ++j)
          if (c0 + j < crop_cols) dense[(r0 + u) * ld + c0 + j] = row[j];
      }
    });
  }
}

// dequantize_prediction (H/codec.hpp:150-158): the 8x8 slope grid of each
// block (IDCT of the dequantized coefficients), tile-major output.
__global__ void __launch_bounds__(128) k_dequantize(const Basis B, CMat in, double* __restrict__ tiles) {
  const uint64_t nb = in.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    RBlock rb = load_block(in, t);
    // decompress_exact with f = 0, s = 1 integrates; undo by emitting p directly:
    // run the same pass 1 / pass 2 through slope_grid_exact.
    slope_grid_exact(rb, B, [&](int u, const double (&p)[BD]) {
#pragma unroll
      for (int v = 0; v < BD; ++v) tiles[t * 64 + u * BD + v] = p[v];
    });
  }
}

// K2 main kernel: the basis operands of pass 2 through uniform registers.
//
// The record's arithmetic is decompress_rows_impl's, in the same order; what changes is
// where the operands live.  Pass 2 walks each row in column pairs, the pair's 16 basis
// values read from c_basis_pairs with a loop-uniform index (LDCU into uniform registers,
// used directly as DMUL operands), so no vector registers hold basis values; the
// integration carries the row above through a per-thread shared-memory slot.  Two things
// keep the code in uniform control flow, which ptxas needs before it places loads in
// uniform registers: one block per thread with no grid-stride loop, and the first column
// pair peeled out of the rolled loop (a grid-stride loop, or the select of the first
// pair inside it, turns the loads back into per-thread LDC).  Blocks not fully inside
// the crop go to k_decompress_edges; an output that is not 16-byte aligned, or a context
// whose basis is not the device's bound one, takes k_decompress (launch_decompress).
//
// The zero grid of s == 0 (H/codec.hpp:151) comes from the dequantized coefficients:
// with every d(i,j) = +0.0 each pass-1 and pass-2 sum is a +0.0 first term plus +-0.0
// products, i.e. +0.0, exactly the reference's grid.
__constant__ double2 c_basis_pairs[4][8];  // (t(j, 2k), t(j, 2k+1)), bound per device

// 32-byte global store (STG.E.ENL2.256, sm_100): dst 32-byte aligned.
__device__ __forceinline__ void st_global_v4(double* dst, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

// Row u-1 of the block (in the shared row) to global memory: 16- or 32-byte stores.
template <bool V4>
__device__ __forceinline__ void store_row(double* dst, const double2 (&above)[4][DEC_UB_THREADS]) {
  if (V4) {
    st_global_v4(dst, above[0][threadIdx.x], above[1][threadIdx.x]);
    st_global_v4(dst + 4, above[2][threadIdx.x], above[3][threadIdx.x]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) reinterpret_cast<double2*>(dst)[k] = above[k][threadIdx.x];
  }
}

// L2 prefetch of the 16-byte-aligned part of [p, p + n) (cp.async.bulk.prefetch.L2; never
// outside the range), by the threads with `on`, without a branch.
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t n, bool on) {
  const uint64_t a = (reinterpret_cast<uint64_t>(p) + 15) & ~15ull;
  const uint64_t e = (reinterpret_cast<uint64_t>(p) + n) & ~15ull;
  const uint32_t sz = e > a ? (uint32_t)(e - a) : 0u;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
      "@q cp.async.bulk.prefetch.L2.global [%0], %1;\n\t}" ::"l"(a), "r"(sz), "r"((uint32_t)(on && sz > 0))
      : "memory");
}

template <bool SYM, bool V4>
__global__ void __launch_bounds__(DEC_UB_THREADS, DEC_UB_MINB) k_decompress_ub(const Basis B, CMat in, double* __restrict__ dense,
                                                                    uint64_t ld, uint64_t crop_rows, uint64_t crop_cols) {
  __shared__ double2 above[4][DEC_UB_THREADS];  // row u-1 of this thread's block, column pairs
  const uint64_t nb = in.nb();
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x * DEC_UB_PER_THREAD + threadIdx.x;
#if DEC_UB_PF
  {  // the records of the CTA DEC_UB_PF CTAs ahead, into L2
    const uint64_t p0 = (blockIdx.x + (uint64_t)DEC_UB_PF) * blockDim.x;
    const uint64_t n = p0 < nb ? min((uint64_t)blockDim.x, nb - p0) : 0;
    const bool on = threadIdx.x == 0 && n > 0;
    prefetch_l2(in.first + p0, n * 8, on);
    prefetch_l2(in.slope + p0, n * 8, on);
    prefetch_l2(in.scale + p0, n, on);
    prefetch_l2(in.coeffs + p0 * KEPT, n * KEPT, on);
  }
#endif
  RBlock recs[DEC_UB_PER_THREAD];  // every record loaded up front: the later blocks' loads
#pragma unroll                    // overlap the earlier blocks' arithmetic
  for (int q = 0; q < DEC_UB_PER_THREAD; ++q) recs[q] = load_block(in, min(t0 + q * blockDim.x, nb - 1));
#pragma unroll
  for (int q = 0; q < DEC_UB_PER_THREAD; ++q) {
  const uint64_t t = t0 + q * blockDim.x;
  const uint64_t tt = t < nb ? t : nb - 1;
  const uint64_t bi = tt / in.bc, bj = tt % in.bc;
  const RBlock& b = recs[q];
  const uint64_t r0 = bi * BD, c0 = bj * BD;
  const bool full = t < nb && r0 + BD <= crop_rows && c0 + BD <= crop_cols;

  const double s = b.s;
  const bool zero = (s == 0.0);
  const double fphi = (double)b.phi;
  double dq[KEPT];
  if (b.phi - 1u < 255u) {
    const double r = 1.0 / fphi;
#pragma unroll
    for (int k = 0; k < KEPT; ++k) dq[k] = zero ? 0.0 : dequant_d(i8_byte_to_f64(b.c[k >> 2], k & 3), fphi, r);
  } else {
#pragma unroll
    for (int k = 0; k < KEPT; ++k) dq[k] = zero ? 0.0 : (double)get_coeff(b.c, k) / fphi;
  }
  if (SYM) {  // t(0,u) d(0,j) is the same for every u
#pragma unroll
    for (int j = 0; j < BD; ++j) dq[j] = B.t[0] * dq[j];
  }
  double* rowp = dense + r0 * ld + c0;
#pragma unroll
  for (int u = 0; u < BD; ++u) {
    // idct2 pass 1 (H/dct.hpp:56-61), as decompress_rows_impl
    double tr[BD];
#pragma unroll
    for (int j = 0; j < BD; ++j) {
      double acc = SYM ? dq[j] : B.t[0 * BD + u] * dq[j];
      acc += B.t[1 * BD + u] * dq[8 + j];
      if (j == 0) {
#pragma unroll
        for (int i = 2; i < BD; ++i) acc += B.t[i * BD + u] * dq[14 + i];
      } else if (j == 1) {
#pragma unroll
        for (int i = 2; i < BD; ++i) acc += B.t[i * BD + u] * dq[20 + i];
      }
      tr[j] = acc;
    }
#if DEC_UB_STORE_AFTER == 2
    if (u > 0 && full) store_row<V4>(rowp - ld, above);  // row u-1, until this row's pairs replace it
#endif
    const double p0 = SYM ? tr[0] * B.t[0] : 0.0;  // row 0 of the basis is constant
    double left = 0.0;
    // idct2 pass 2 (H/dct.hpp:62-68) for columns 2k, 2k+1, then integrate_rows
    // (H/codec.hpp:164-174) for them
    auto pair = [&](const int k, const bool first) {
      double a0, a1;
      if (SYM) {
        a0 = p0;
        a1 = p0;
      } else {
        const double2 c = c_basis_pairs[k][0];
        a0 = tr[0] * c.x;
        a1 = tr[0] * c.y;
      }
#pragma unroll
      for (int j = 1; j < BD; ++j) {
        const double2 c = c_basis_pairs[k][j];
        a0 += tr[j] * c.x;
        a1 += tr[j] * c.y;
      }
      double x0, x1;
      if (u == 0) {
        x0 = first ? b.f : left + s * a0;
        x1 = x0 + s * a1;
      } else {
        const double2 up = above[k][threadIdx.x];
        x0 = first ? up.x + s * a0 : (up.x + left) / 2.0 + s * a0;
        x1 = (up.y + x0) / 2.0 + s * a1;
      }
#if DEC_UB_STORE_AFTER
      above[k][threadIdx.x] = make_double2(x0, x1);
      left = x1;
#else
      if (u < BD - 1) above[k][threadIdx.x] = make_double2(x0, x1);
      left = x1;
      if (full) reinterpret_cast<double2*>(rowp)[k] = make_double2(x0, x1);
#endif
    };
    pair(0, true);
#pragma unroll 1
    for (int k = 1; k < 4; ++k) pair(k, false);
#if DEC_UB_STORE_AFTER == 1
    if (full) {
#pragma unroll
      for (int k = 0; k < 4; ++k) reinterpret_cast<double2*>(rowp)[k] = above[k][threadIdx.x];
    }
#endif
    rowp += ld;
  }
#if DEC_UB_STORE_AFTER == 2
  if (full) store_row<V4>(rowp - ld, above);
#endif
  }
}

// The blocks k_decompress_ub leaves out: those partly inside the crop (the last partial
// block-row and block-column), through the streamed per-block code with masked stores.
template <bool SYM>
__global__ void __launch_bounds__(128) k_decompress_edges(const Basis B, CMat in, double* __restrict__ dense,
                                                          uint64_t ld, uint64_t crop_rows, uint64_t crop_cols,
                                                          uint64_t er, uint64_t ec, uint64_t nvr, uint64_t nvc) {
  // edge set: block-row er (if er < in.br) over block-columns [0, nvc), then block-column
  // ec (if ec < in.bc) over block-rows [0, nvr) other than er
  const uint64_t n_row = er < in.br ? nvc : 0;
  const uint64_t n_col = ec < in.bc ? nvr - (er < nvr ? 1 : 0) : 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_row + n_col;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t bi, bj;
    if (i < n_row) {
      bi = er;
      bj = i;
    } else {
      bi = i - n_row;
      if (bi >= er) ++bi;
      bj = ec;
    }
    const RBlock rb = load_block(in, bi * in.bc + bj);
    const uint64_t r0 = bi * BD, c0 = bj * BD;
    decompress_exact<SYM>(rb, B, [&](int u, const double (&row)[BD]) {
      if (r0 + u < crop_rows) {
#pragma unroll
        for (int j = 0; j < BD; ++j)
          if (c0 + j < crop_cols) dense[(r0 + u) * ld + c0 + j] = row[j];
      }
    });
  }
}

// Binds the basis to c_basis_pairs of the current device: the first basis bound on a
// device keeps the symbol (it is never rewritten, so no running kernel sees it change);
// *bound tells whether B is that basis.
cudaError_t bind_decompress_basis(const Basis& B, bool* bound) {
  static std::mutex mu;
  static std::map<int, Basis> held;
  *bound = false;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto it = held.find(dev);
  if (it == held.end()) {
    double2 pairs[4][8];
    for (int k = 0; k < 4; ++k)
      for (int j = 0; j < BD; ++j) pairs[k][j] = make_double2(B.t[j * BD + 2 * k], B.t[j * BD + 2 * k + 1]);
    e = cudaMemcpyToSymbol(c_basis_pairs, pairs, sizeof(pairs));
    if (e != cudaSuccess) return e;
    it = held.emplace(dev, B).first;
  }
  *bound = std::memcmp(it->second.t, B.t, sizeof B.t) == 0;
  return cudaSuccess;
}

static unsigned grid_for(uint64_t n, unsigned threads, int sms, unsigned per_sm = 64) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sms * per_sm;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_compress(const LaunchCtx& c, const Basis& B, const double* dense, uint64_t rows,
                            uint64_t cols, uint64_t ld, const CMat& out) {
  const unsigned g = grid_for(out.nb(), 128, c.sm_count);
  // the fast path stores coefficient records as 16-byte chunks (k_compress_pair):
  // a caller view whose coefficient array is not 16-byte aligned takes the exact kernel
  const bool coeffs_aligned = (reinterpret_cast<uintptr_t>(out.coeffs) & 15) == 0;
  if (c.exact_only || !c.fast || !coeffs_aligned) {
    k_compress<<<g, 128, 0, c.stream>>>(B, dense, rows, cols, ld, out, c.err);
    ++*c.launches;
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(c.wl_count, 0, sizeof(unsigned long long), c.stream);
  if (e != cudaSuccess) return e;
  FastParams P;
  P.B = B;
  P.ss00 = c.fast->ss00;
  P.zero = 0;
  e = launch_compress_pair(c, P, dense, rows, cols, ld, out);
  if (e != cudaSuccess) return e;
  return launch_compress_worklist_warp(c, B, dense, rows, cols, ld, out);
}

cudaError_t launch_dequantize(const LaunchCtx& c, const Basis& B, const CMat& in, double* tiles) {
  k_dequantize<<<grid_for(in.nb(), 128, c.sm_count), 128, 0, c.stream>>>(B, in, tiles);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_decompress_gather(const LaunchCtx& c, const Basis& B, const ShardSet& S, uint64_t bc,
                                     double* dense, uint64_t ld, uint64_t crop_rows, uint64_t crop_cols) {
  const unsigned g = grid_for(S.lo[S.n] * bc, 128, c.sm_count, DEC_GRID_PER_SM);
  if (c.basis_sym && !c.exact_only)
    k_decompress_gather<true><<<g, 128, 0, c.stream>>>(B, S, bc, dense, ld, crop_rows, crop_cols);
  else
    k_decompress_gather<false><<<g, 128, 0, c.stream>>>(B, S, bc, dense, ld, crop_rows, crop_cols);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_decompress(const LaunchCtx& c, const Basis& B, const CMat& in, double* dense,
                              uint64_t ld, uint64_t crop_rows, uint64_t crop_cols) {
  const unsigned g = grid_for(in.nb(), 128, c.sm_count, DEC_GRID_PER_SM);
  const bool aligned = ((ld & 1) == 0) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  if (DEC_UB && c.basis_bound && aligned && in.nb() > 0 && in.nb() / DEC_UB_THREADS < (1ull << 31)) {
    const bool sym = c.basis_sym && !c.exact_only;
    constexpr uint64_t per_cta = (uint64_t)DEC_UB_THREADS * DEC_UB_PER_THREAD;
    const unsigned g1 = (unsigned)((in.nb() + per_cta - 1) / per_cta);
    const bool v4 = DEC_UB_V4 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(dense) & 31) == 0;
    if (sym && v4)
      k_decompress_ub<true, true><<<g1, DEC_UB_THREADS, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
    else if (sym)
      k_decompress_ub<true, false><<<g1, DEC_UB_THREADS, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
    else if (v4)
      k_decompress_ub<false, true><<<g1, DEC_UB_THREADS, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
    else
      k_decompress_ub<false, false><<<g1, DEC_UB_THREADS, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
    ++*c.launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // partial blocks: block-row crop_rows/8 and block-column crop_cols/8 when the crop
    // ends inside them
    const uint64_t er = (crop_rows % BD) ? crop_rows / BD : ~0ull;
    const uint64_t ec = (crop_cols % BD) ? crop_cols / BD : ~0ull;
    if ((er < in.br) || (ec < in.bc)) {
      const uint64_t nvr = std::min<uint64_t>(in.br, (crop_rows + BD - 1) / BD);
      const uint64_t nvc = std::min<uint64_t>(in.bc, (crop_cols + BD - 1) / BD);
      const uint64_t n = nvr + nvc;
      if (sym)
        k_decompress_edges<true><<<grid_for(n, 128, c.sm_count), 128, 0, c.stream>>>(B, in, dense, ld, crop_rows,
                                                                                     crop_cols, er, ec, nvr, nvc);
      else
        k_decompress_edges<false><<<grid_for(n, 128, c.sm_count), 128, 0, c.stream>>>(B, in, dense, ld, crop_rows,
                                                                                      crop_cols, er, ec, nvr, nvc);
      ++*c.launches;
      e = cudaGetLastError();
    }
    return e;
  }
  if (c.basis_sym && !c.exact_only)  // exact mode keeps the plain product-per-term kernel
    k_decompress<true><<<g, 128, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
  else
    k_decompress<false><<<g, 128, 0, c.stream>>>(B, in, dense, ld, crop_rows, crop_cols);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
