// dot.cu -- K5 row-wise dots / Frobenius, K6 batched mat_dot (exact mode).
//
// mat_dot (H/matrix.hpp:157-173): entry (i,j) of Ahat*Bhat accumulated over
// the inner block index t ascending, then k ascending (padding excluded),
// from +0.0, one DMUL + DADD per term.  reconstruct_rows/_cols
// (H/block_ops.hpp:87-115) are bitwise prefixes of decompress_block, so row
// ri / column cj are taken from the full exact decompression.
//
// Row dots (config 2, restated in SURVEY.md 8c): r_i = sum_j Ahat(i,j) *
// Bhat(i,j) ascending j from +0.0 -- the ref::dot loop (H/matrix.hpp:280-286)
// applied along rows of two decompress_matrix outputs.
#include "blaz_device.cuh"
#include "launch.h"

#include <algorithm>

namespace blz {

cudaError_t launch_sum(const LaunchCtx& c, const double* v, uint64_t n, double* out);

// a holds rows [row0, row0 + a.rows) of a matrix with rows_total rows (a row
// shard; row0 = 0 and rows_total = a.rows for a whole matrix).  Queries on rows
// of other shards get +0.0 (all bits zero), so the shards' results combine
// exactly by an integer sum of their bit patterns.
template <bool SYM>
__global__ void __launch_bounds__(128) k_dot_entries(const Basis B, CMat a, CMat b,
                                                     const uint64_t* __restrict__ qi,
                                                     const uint64_t* __restrict__ qj, uint64_t n,
                                                     double* __restrict__ out,
                                                     unsigned long long* err, uint64_t row0, uint64_t rows_total) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ig = qi[q], j = qj[q];
    if (ig >= rows_total || j >= b.cols) {
      latch_error(err, q, DERR_DOT_RANGE);
      out[q] = 0.0;
      continue;
    }
    if (ig < row0 || ig - row0 >= a.rows) {  // another shard's row
      out[q] = 0.0;
      continue;
    }
    const uint64_t i = ig - row0;
    const uint64_t bi = i / BD, bj = j / BD;
    const int ri = (int)(i % BD), cj = (int)(j % BD);
    double r = 0.0;
    for (uint64_t t = 0; t < a.bc; ++t) {
      double arow[BD], bcol[BD];
      const RBlock ba = load_block(a, bi * a.bc + t);
      const RBlock bb = load_block(b, t * b.bc + bj);
      decompress_exact<SYM>(ba, B, [&](int u, const double (&row)[BD]) {
        if (u == ri) {
#pragma unroll
          for (int k = 0; k < BD; ++k) arow[k] = row[k];
        }
      });
      decompress_exact<SYM>(bb, B, [&](int u, const double (&row)[BD]) {
        double v = row[0];
#pragma unroll
        for (int k = 1; k < BD; ++k) v = (cj == k) ? row[k] : v;
        bcol[u] = v;
      });
      const uint64_t rem = a.cols - t * BD;
      const int klim = rem < BD ? (int)rem : BD;
#pragma unroll
      for (int k = 0; k < BD; ++k)
        if (k < klim) r += arow[k] * bcol[k];
    }
    out[q] = r;
  }
}

// Few queries: one warp per query.  Lanes decompress the pairs (A(bi, t), B(t, bj))
// for 32 consecutive t at once and form the products a(ri, k) * b(k, cj) (each
// rounded, as the reference's r += a * b); lane 0 then adds them in the
// reference's order (t ascending, then k < klim) -- the same operation sequence
// as the thread-per-query kernel, with the decompressions spread over the warp.
template <bool SYM>
__global__ void __launch_bounds__(128) k_dot_warp(const Basis B, CMat a, CMat b, const uint64_t* __restrict__ qi,
                                                 const uint64_t* __restrict__ qj, uint64_t n,
                                                 double* __restrict__ out, unsigned long long* err, uint64_t row0,
                                                 uint64_t rows_total) {
  __shared__ double prod[4][32 * 9];  // per warp: 8 products per lane (+1 pad)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* pw = prod[warp];
  for (uint64_t q = blockIdx.x * (uint64_t)4 + warp; q < n; q += (uint64_t)gridDim.x * 4) {
    const uint64_t ig = qi[q], j = qj[q];
    if (ig >= rows_total || j >= b.cols) {  // warp-uniform
      if (lane == 0) {
        latch_error(err, q, DERR_DOT_RANGE);
        out[q] = 0.0;
      }
      continue;
    }
    if (ig < row0 || ig - row0 >= a.rows) {  // another shard's row (k_dot_entries)
      if (lane == 0) out[q] = 0.0;
      continue;
    }
    const uint64_t i = ig - row0;
    const uint64_t bi = i / BD, bj = j / BD;
    const int ri = (int)(i % BD), cj = (int)(j % BD);
    double r = 0.0;
    for (uint64_t t0 = 0; t0 < a.bc; t0 += 32) {
      const uint64_t t = min(t0 + lane, a.bc - 1);
      double arow[BD], bcol[BD];
      const RBlock ba = load_block(a, bi * a.bc + t);
      const RBlock bb = load_block(b, t * b.bc + bj);
      decompress_exact<SYM>(ba, B, [&](int u, const double (&row)[BD]) {
        if (u == ri) {
#pragma unroll
          for (int k = 0; k < BD; ++k) arow[k] = row[k];
        }
      });
      decompress_exact<SYM>(bb, B, [&](int u, const double (&row)[BD]) {
        double v = row[0];
#pragma unroll
        for (int k = 1; k < BD; ++k) v = (cj == k) ? row[k] : v;
        bcol[u] = v;
      });
#pragma unroll
      for (int k = 0; k < BD; ++k) pw[lane * 9 + k] = arow[k] * bcol[k];
      __syncwarp();
      if (lane == 0) {
        const uint64_t left = a.bc - t0;
        const uint64_t cnt = left < 32 ? left : 32;
        for (uint64_t tl = 0; tl < cnt; ++tl) {
          const uint64_t rem = a.cols - (t0 + tl) * BD;
          const int klim = rem < BD ? (int)rem : BD;
          for (int k = 0; k < klim; ++k) r += pw[tl * 9 + k];
        }
      }
      __syncwarp();
    }
    if (lane == 0) out[q] = r;
  }
}

// Row dots r_i = sum_j Ahat(i,j) Bhat(i,j), ascending j from +0.0.
// A warp covers 4 block-rows.  Per chunk of 4 block-columns, lanes 0-15
// decompress the 16 A blocks and lanes 16-31 the 16 matching B blocks (exact,
// one decompression per lane) into shared memory; then lane L advances the
// serial chain of row (L & 7) of block-row (L >> 3) over the chunk's 4 blocks
// x 8 columns in ascending order: acc += a*b (DMUL then DADD) -- the identical
// operation sequence as the single-threaded restatement.  Row stride 9 and
// slot stride 74 doubles keep the chain reads bank-conflict-free.
constexpr int RD_WARPS = 2;
constexpr int RD_SLOT = 74;

template <bool SYM>
__global__ void __launch_bounds__(RD_WARPS * 32) k_rowdot(const Basis B, CMat a, CMat b, double* __restrict__ r) {
  __shared__ double P[RD_WARPS][32 * RD_SLOT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* S = P[warp];
  const uint64_t groups = (a.br + 3) / 4;
  // decompression role of this lane
  const bool is_b = lane >= 16;
  const int dl = lane & 15;
  const int dgrp = dl >> 2, dcol = dl & 3;
  // chain role of this lane
  const int cgrp = lane >> 3, u_own = lane & 7;
  for (uint64_t g = blockIdx.x * (uint64_t)RD_WARPS + warp; g < groups; g += (uint64_t)gridDim.x * RD_WARPS) {
    const uint64_t drow = g * 4 + dgrp, crow = g * 4 + cgrp;
    double acc = 0.0;
    for (uint64_t t0 = 0; t0 < a.bc; t0 += 4) {
      // no divergent branch around the decompression (keeps the basis in
      // uniform registers): out-of-range lanes decompress a clamped block
      // into their own slot, which the chain phase never reads
      {
        const uint64_t t = min(t0 + dcol, a.bc - 1), dr = min(drow, a.br - 1);
        const uint64_t idx = dr * a.bc + t;
        RBlock blk;
        blk.f = is_b ? b.first[idx] : a.first[idx];
        blk.s = is_b ? b.slope[idx] : a.slope[idx];
        blk.phi = is_b ? b.scale[idx] : a.scale[idx];
        const uint32_t* cw = reinterpret_cast<const uint32_t*>((is_b ? b.coeffs : a.coeffs) + idx * KEPT);
#pragma unroll
        for (int w = 0; w < 7; ++w) blk.c[w] = cw[w];
        double* slot = S + lane * RD_SLOT;
        decompress_exact<SYM>(blk, B, [&](int u, const double (&row)[BD]) {
#pragma unroll
          for (int v = 0; v < BD; ++v) slot[u * 9 + v] = row[v];
        });
      }
      __syncwarp();
      if (crow < a.br) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t tk = t0 + k;
          if (tk < a.bc) {
            const uint64_t rem = a.cols - tk * BD;
            const int jlim = rem < BD ? (int)rem : BD;
            const double* sa = S + (cgrp * 4 + k) * RD_SLOT + u_own * 9;
            const double* sb = S + (16 + cgrp * 4 + k) * RD_SLOT + u_own * 9;
#pragma unroll
            for (int v = 0; v < BD; ++v)
              if (v < jlim) acc += sa[v] * sb[v];
          }
        }
      }
      __syncwarp();
    }
    const uint64_t row = crow * BD + u_own;
    if (crow < a.br && row < a.rows) r[row] = acc;
  }
}

// The same row dots as a persistent kernel over split work items: a group's
// block-columns are cut into RD_SPLIT consecutive ranges, and item (q, g) advances
// group g's 32 row chains over range q, starting from the accumulators item
// (q-1, g) left in global memory (storing and reloading a double is exact, so
// every chain is the same single operation sequence).  Items are claimed in
// order from an atomic counter -- all first ranges, then all second ranges, ... --
// so an item's predecessor was claimed earlier by a running warp and the wait
// for it is short; finer items fill the last wave of resident warps (2,048
// groups at 65536^2 are 1.73 waves of the 1,184 resident warps; 8,192 quarter
// items are 6.9 waves).
#ifndef RD_SPLIT
#define RD_SPLIT 16  // 65536^2: 21.2 ms unsplit, 16.7 / 16.4 / 16.5 ms with 8 / 16 / 32 ranges
#endif

#ifndef RD_SPLIT_MINB
#define RD_SPLIT_MINB 1  // (64, 1): 255 registers, 16.8-17.0 ms; plain (64): 220-248 registers, 17.5-17.7 ms
#endif
#define RD_SPLIT_BOUNDS __launch_bounds__(RD_WARPS * 32, RD_SPLIT_MINB)
// Record slot of one lane (the block it decompresses next), filled by cp.async.
struct RecSlot {
  double f, s;
  uint32_t c[7];
  uint32_t phiw;  // the 4-byte word holding the scale byte
};

__device__ __forceinline__ void cpa(void* smem, const void* gmem, int bytes_const8) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes_const8 == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}

#ifndef RD_PREFETCH
#define RD_PREFETCH 1
#endif

constexpr int SUM_BATCH = 1024;

// The ascending total of the row dots (the restated oracle's order: one dependent
// DADD chain from +0.0) run by warp 0 of CTA 0 while the other warps still
// produce row dots: batches of 32 groups (1,024 rows) are staged in shared memory
// with cp.async as soon as their final flags are up, and lane 0 adds the previous
// batch meanwhile.  Bitwise the separate k_sum.
__device__ __noinline__ void rowdot_total_warp(const double* __restrict__ r, uint64_t nrows, uint64_t groups,
                                  const int* __restrict__ flags, int nsplit, double* __restrict__ buf,
                                  double* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const uint64_t nb = (groups + 31) / 32;
  double s = 0.0;
  auto chain = [&](uint64_t bidx) {
    if (lane == 0) {
      const double* p = buf + (bidx & 1) * SUM_BATCH;
      const uint64_t lo = bidx * SUM_BATCH, n = min((uint64_t)SUM_BATCH, nrows - lo);
      for (uint64_t k = 0; k < n; ++k) s += p[k];
    }
  };
  for (uint64_t bidx = 0; bidx < nb; ++bidx) {
    const uint64_t g = bidx * 32 + lane;
    if (g < groups)
      while (*(volatile const int*)(flags + g) < nsplit) __nanosleep(256);
    __syncwarp();
    __threadfence();
    const uint64_t lo = bidx * SUM_BATCH;
    double* dst = buf + (bidx & 1) * SUM_BATCH;
#pragma unroll 4
    for (int k = 0; k < SUM_BATCH / 32; ++k) {
      const uint64_t i = lo + (uint64_t)k * 32 + lane;
      if (i < nrows) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + k * 32 + lane);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(r + i) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (bidx > 0) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      chain(bidx - 1);
      __syncwarp();  // slot (bidx - 1) & 1 is refilled by batch bidx + 1
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  if (nb) chain(nb - 1);
  if (lane == 0) *total = s;
}

template <bool SYM>
__global__ void RD_SPLIT_BOUNDS
    k_rowdot_split(const Basis B, CMat a, CMat b, double* __restrict__ r, unsigned long long* __restrict__ counter,
                   int* __restrict__ flags, double* __restrict__ state, int nsplit, double* __restrict__ total) {
  __shared__ double P[RD_WARPS][32 * RD_SLOT];
#if RD_PREFETCH
  // the next chunk's records, prefetched with cp.async while the current chunk is
  // decompressed (no registers held in flight)
  __shared__ RecSlot R[RD_WARPS][2][32];
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* S = P[warp];
  const uint64_t groups = (a.br + 3) / 4;
  const uint64_t items = groups * nsplit;
  const bool is_b = lane >= 16;
  const int dl = lane & 15;
  const int dgrp = dl >> 2, dcol = dl & 3;
  const int cgrp = lane >> 3, u_own = lane & 7;
  const CMat& src = is_b ? b : a;
  if (total && blockIdx.x == 0 && warp == 0) {  // the total, overlapped with the row dots
    rowdot_total_warp(r, a.rows, groups, flags, nsplit, S, total);
    return;
  }
  for (;;) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(counter, 1ull);
    w = __shfl_sync(0xffffffffu, w, 0);
    if (w >= items) break;
    const int q = (int)(w / groups);
    const uint64_t g = w % groups;
    // block-column range of item q: cut points at multiples of 4 (one chunk)
    const uint64_t c0 = (a.bc * (uint64_t)q / nsplit) / 4 * 4;
    const uint64_t c1 = q == nsplit - 1 ? a.bc : (a.bc * (uint64_t)(q + 1) / nsplit) / 4 * 4;
    const uint64_t drow = g * 4 + dgrp, crow = g * 4 + cgrp;
    const uint64_t dr = min(drow, a.br - 1);
#if RD_PREFETCH
    auto prefetch = [&](uint64_t t0, int buf) {
      const uint64_t idx = dr * a.bc + min(t0 + dcol, a.bc - 1);
      RecSlot& rs = R[warp][buf][lane];
      cpa(&rs.f, src.first + idx, 8);
      cpa(&rs.s, src.slope + idx, 8);
      const uint32_t* cw = reinterpret_cast<const uint32_t*>(src.coeffs + idx * KEPT);
#pragma unroll
      for (int w2 = 0; w2 < 7; ++w2) cpa(&rs.c[w2], cw + w2, 4);
      cpa(&rs.phiw, reinterpret_cast<const uint32_t*>(src.scale + (idx & ~3ull)), 4);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (c0 < c1) prefetch(c0, 0);
    int buf = 0;
#endif
    double acc = 0.0;
    if (q > 0) {  // wait for item (q-1, g), then continue its chains
      if (lane == 0) {
        while (*(volatile int*)(flags + g) < q) __nanosleep(200);
      }
      __syncwarp();
      __threadfence();
      acc = __ldcg(state + g * 32 + lane);
    }
    for (uint64_t t0 = c0; t0 < c1; t0 += 4) {
      {
        RBlock blk;
#if RD_PREFETCH
        if (t0 + 4 < c1) {
          prefetch(t0 + 4, buf ^ 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        {
          const RecSlot& rs = R[warp][buf][lane];
          const uint64_t idx = dr * a.bc + min(t0 + dcol, a.bc - 1);
          blk.f = rs.f;
          blk.s = rs.s;
          blk.phi = (rs.phiw >> (8 * (idx & 3))) & 0xffu;
#pragma unroll
          for (int w2 = 0; w2 < 7; ++w2) blk.c[w2] = rs.c[w2];
        }
        buf ^= 1;
#else
        const uint64_t t = min(t0 + dcol, a.bc - 1);
        const uint64_t idx = dr * a.bc + t;
        blk.f = src.first[idx];
        blk.s = src.slope[idx];
        blk.phi = src.scale[idx];
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(src.coeffs + idx * KEPT);
#pragma unroll
        for (int w2 = 0; w2 < 7; ++w2) blk.c[w2] = cw[w2];
#endif
        double* slot = S + lane * RD_SLOT;
        decompress_exact<SYM>(blk, B, [&](int u, const double (&row)[BD]) {
#pragma unroll
          for (int v = 0; v < BD; ++v) slot[u * 9 + v] = row[v];
        });
      }
      __syncwarp();
      if (crow < a.br) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t tk = t0 + k;
          if (tk < c1) {
            const uint64_t rem = a.cols - tk * BD;
            const int jlim = rem < BD ? (int)rem : BD;
            const double* sa = S + (cgrp * 4 + k) * RD_SLOT + u_own * 9;
            const double* sb = S + (16 + cgrp * 4 + k) * RD_SLOT + u_own * 9;
#pragma unroll
            for (int v = 0; v < BD; ++v)
              if (v < jlim) acc += sa[v] * sb[v];
          }
        }
      }
      __syncwarp();
    }
    if (q == nsplit - 1) {
      const uint64_t row = crow * BD + u_own;
      if (crow < a.br && row < a.rows) r[row] = acc;
      if (total) {  // publish the group's final row dots to the total warp
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(flags + g, nsplit);
      }
    } else {
      __stcg(state + g * 32 + lane, acc);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicExch(flags + g, q + 1);
    }
  }
}

uint64_t rowdot_scratch_bytes(const CMat& a) {
  const uint64_t groups = (a.br + 3) / 4;
  return 256 + groups * 4 + 256 + groups * 32 * sizeof(double);
}

// Ascending serial sum from +0.0 (the restated oracle's order; inherently one
// dependent DADD chain).  One warp: the lanes stage batches of 1,024 values in
// shared memory with cp.async (two buffers, the next batch in flight while the
// current one is added), lane 0 runs the chain out of shared memory, so the sum
// proceeds at the DADD latency.
__global__ void __launch_bounds__(32) k_sum(const double* __restrict__ v, uint64_t n, double* __restrict__ out) {
  __shared__ __align__(16) double buf[2][SUM_BATCH];
  const int lane = threadIdx.x & 31;
  const bool vec = (reinterpret_cast<uintptr_t>(v) & 15) == 0;
  const uint64_t nfull = vec ? n / SUM_BATCH : 0;  // whole batches
  auto stage = [&](uint64_t bidx, int slot) {
    const double* src = v + bidx * SUM_BATCH;
#pragma unroll
    for (int k = 0; k < SUM_BATCH / 64; ++k) {  // 16 x 16 bytes per lane
      const int e = 2 * (k * 32 + lane);
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[slot][e]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + e) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double s = 0.0;
  if (nfull) stage(0, 0);
  for (uint64_t bidx = 0; bidx < nfull; ++bidx) {
    const int slot = (int)(bidx & 1);
    if (bidx + 1 < nfull) {
      stage(bidx + 1, slot ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) {
      const double2* p = reinterpret_cast<const double2*>(buf[slot]);
#pragma unroll 16
      for (int k = 0; k < SUM_BATCH / 2; ++k) {
        const double2 x = p[k];
        s += x.x;
        s += x.y;
      }
    }
    __syncwarp();  // the slot is refilled two batches later
  }
  if (lane == 0) {
    for (uint64_t k = nfull * SUM_BATCH; k < n; ++k) s += v[k];
    *out = s;
  }
}

// A handful of queries on a wide inner dimension: one thread per (query, inner
// block t) decompresses row ri of A(bi, t) and column cj of B(t, bj) and stores the
// eight rounded products a(ri, k) b(k, cj); then one warp per query adds them in
// the reference's order (t ascending, k < klim) out of shared-memory batches.
template <bool SYM>
__global__ void __launch_bounds__(128) k_dot_products(const Basis B, CMat a, CMat b, const uint64_t* __restrict__ qi,
                                                      const uint64_t* __restrict__ qj, uint64_t n, uint64_t row0,
                                                      uint64_t rows_total, double* __restrict__ prod) {
  const uint64_t total = n * a.bc;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = x / a.bc, t = x % a.bc;
    const uint64_t ig = qi[q], j = qj[q];
    if (ig >= rows_total || j >= b.cols || ig < row0 || ig - row0 >= a.rows) continue;  // k_dot_sum decides
    const uint64_t i = ig - row0, bi = i / BD, bj = j / BD;
    const int ri = (int)(i % BD), cj = (int)(j % BD);
    double arow[BD], bcol[BD];
    decompress_exact<SYM>(load_block(a, bi * a.bc + t), B, [&](int u, const double (&row)[BD]) {
      if (u == ri) {
#pragma unroll
        for (int k = 0; k < BD; ++k) arow[k] = row[k];
      }
    });
    decompress_exact<SYM>(load_block(b, t * b.bc + bj), B, [&](int u, const double (&row)[BD]) {
      double v = row[0];
#pragma unroll
      for (int k = 1; k < BD; ++k) v = (cj == k) ? row[k] : v;
      bcol[u] = v;
    });
    double* pp = prod + x * BD;
#pragma unroll
    for (int k = 0; k < BD; ++k) pp[k] = arow[k] * bcol[k];
  }
}

constexpr int DOT_BATCH = 1024;  // products per shared-memory batch

__global__ void __launch_bounds__(32) k_dot_sum(CMat a, CMat b, const uint64_t* __restrict__ qi,
                                                const uint64_t* __restrict__ qj, uint64_t row0, uint64_t rows_total,
                                                const double* __restrict__ prod, double* __restrict__ out,
                                                unsigned long long* err) {
  __shared__ double buf[DOT_BATCH];
  const uint64_t q = blockIdx.x;
  const int lane = threadIdx.x;
  const uint64_t ig = qi[q], j = qj[q];
  if (ig >= rows_total || j >= b.cols) {
    if (lane == 0) {
      latch_error(err, q, DERR_DOT_RANGE);
      out[q] = 0.0;
    }
    return;
  }
  if (ig < row0 || ig - row0 >= a.rows) {  // another shard's row
    if (lane == 0) out[q] = 0.0;
    return;
  }
  const double* pp = prod + q * a.bc * BD;
  const uint64_t total = a.bc * BD;
  double r = 0.0;
  for (uint64_t base = 0; base < total; base += DOT_BATCH) {
    const int m = (int)(total - base < DOT_BATCH ? total - base : DOT_BATCH);
    for (int k = lane; k < m; k += 32) buf[k] = pp[base + k];
    __syncwarp();
    if (lane == 0) {
      const uint64_t t0 = base / BD;  // DOT_BATCH is a multiple of 8
      const int nt = m / BD;
      for (int tl = 0; tl < nt; ++tl) {
        const uint64_t rem = a.cols - (t0 + tl) * BD;
        const double* bp = buf + tl * BD;
        if (rem >= BD) {
#pragma unroll
          for (int k = 0; k < BD; ++k) r += bp[k];
        } else {
          for (int k = 0; k < (int)rem; ++k) r += bp[k];  // padding columns excluded (k < klim)
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) out[q] = r;
}

cudaError_t launch_dot_entries(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b,
                               const uint64_t* i, const uint64_t* j, uint64_t n, double* out, uint64_t row0,
                               uint64_t rows_total, double* prod) {
  if (n == 0) return cudaSuccess;
  const bool sym = c.basis_sym && !c.exact_only;
  if (prod && n <= kDotSplitMaxQueries && a.bc >= 32) {  // few queries, wide inner dimension
    const uint64_t total = n * a.bc;
    const unsigned g = (unsigned)((total + 127) / 128);
    if (sym)
      k_dot_products<true><<<g, 128, 0, c.stream>>>(B, a, b, i, j, n, row0, rows_total, prod);
    else
      k_dot_products<false><<<g, 128, 0, c.stream>>>(B, a, b, i, j, n, row0, rows_total, prod);
    k_dot_sum<<<(unsigned)n, 32, 0, c.stream>>>(a, b, i, j, row0, rows_total, prod, out, c.err);
    *c.launches += 2;
    return cudaGetLastError();
  }
  if (n <= (uint64_t)c.sm_count * 64) {  // few queries: a warp per query
    const unsigned gw = (unsigned)((n + 3) / 4);
    if (sym)
      k_dot_warp<true><<<gw, 128, 0, c.stream>>>(B, a, b, i, j, n, out, c.err, row0, rows_total);
    else
      k_dot_warp<false><<<gw, 128, 0, c.stream>>>(B, a, b, i, j, n, out, c.err, row0, rows_total);
    ++*c.launches;
    return cudaGetLastError();
  }
  const unsigned g = (unsigned)((n + 127) / 128 < (uint64_t)c.sm_count * 16 ? (n + 127) / 128
                                                                             : (uint64_t)c.sm_count * 16);
  if (c.basis_sym && !c.exact_only)
    k_dot_entries<true><<<g, 128, 0, c.stream>>>(B, a, b, i, j, n, out, c.err, row0, rows_total);
  else
    k_dot_entries<false><<<g, 128, 0, c.stream>>>(B, a, b, i, j, n, out, c.err, row0, rows_total);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_rowdot(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b, double* r,
                          void* scratch, double* total) {
  const uint64_t groups = (a.br + 3) / 4;
  const bool sym = c.basis_sym && !c.exact_only;
  // at least 8 chunks of 4 block-columns per range
  const int nsplit = (int)std::max<uint64_t>(1, std::min<uint64_t>(RD_SPLIT, a.bc / 32));
  if (scratch && nsplit > 1) {
    unsigned long long* counter = (unsigned long long*)scratch;
    int* flags = (int*)((char*)scratch + 256);
    double* state = (double*)((char*)scratch + 256 + ((groups * 4 + 255) / 256) * 256);
    cudaError_t e = cudaMemsetAsync(scratch, 0, 256 + groups * 4, c.stream);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = sym ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rowdot_split<true>, RD_WARPS * 32, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rowdot_split<false>, RD_WARPS * 32, 0);
    if (e != cudaSuccess) return e;
    const uint64_t want = (groups * nsplit + RD_WARPS - 1) / RD_WARPS;
    const uint64_t cap = (uint64_t)c.sm_count * (per_sm > 0 ? per_sm : 1);
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    // with a total, warp 0 of CTA 0 sums the finished row dots during the run
    if (sym)
      k_rowdot_split<true><<<g, RD_WARPS * 32, 0, c.stream>>>(B, a, b, r, counter, flags, state, nsplit, total);
    else
      k_rowdot_split<false><<<g, RD_WARPS * 32, 0, c.stream>>>(B, a, b, r, counter, flags, state, nsplit, total);
    ++*c.launches;
    return cudaGetLastError();
  }
  const uint64_t want = (groups + RD_WARPS - 1) / RD_WARPS;
  const uint64_t cap = (uint64_t)c.sm_count * 16;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  if (c.basis_sym && !c.exact_only)  // shared products of the repeated basis entries (blaz_device.cuh)
    k_rowdot<true><<<g, RD_WARPS * 32, 0, c.stream>>>(B, a, b, r);
  else
    k_rowdot<false><<<g, RD_WARPS * 32, 0, c.stream>>>(B, a, b, r);
  ++*c.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !total) return e;
  return launch_sum(c, r, a.rows, total);
}

cudaError_t launch_sum(const LaunchCtx& c, const double* v, uint64_t n, double* out) {
  k_sum<<<1, 32, 0, c.stream>>>(v, n, out);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
