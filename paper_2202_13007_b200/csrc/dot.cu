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

namespace blz {

__global__ void __launch_bounds__(128) k_dot_entries(const Basis B, CMat a, CMat b,
                                                     const uint64_t* __restrict__ qi,
                                                     const uint64_t* __restrict__ qj, uint64_t n,
                                                     double* __restrict__ out,
                                                     unsigned long long* err) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = qi[q], j = qj[q];
    if (i >= a.rows || j >= b.cols) {
      latch_error(err, q, DERR_DOT_RANGE);
      out[q] = 0.0;
      continue;
    }
    const uint64_t bi = i / BD, bj = j / BD;
    const int ri = (int)(i % BD), cj = (int)(j % BD);
    double r = 0.0;
    for (uint64_t t = 0; t < a.bc; ++t) {
      double arow[BD], bcol[BD];
      const RBlock ba = load_block(a, bi * a.bc + t);
      const RBlock bb = load_block(b, t * b.bc + bj);
      decompress_exact(ba, B, [&](int u, const double (&row)[BD]) {
        if (u == ri) {
#pragma unroll
          for (int k = 0; k < BD; ++k) arow[k] = row[k];
        }
      });
      decompress_exact(bb, B, [&](int u, const double (&row)[BD]) {
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

// One thread per block-row: 8 running row sums, blocks ascending.
__global__ void __launch_bounds__(128) k_rowdot(const Basis B, CMat a, CMat b, double* __restrict__ r) {
  for (uint64_t bi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; bi < a.br;
       bi += (uint64_t)gridDim.x * blockDim.x) {
    double acc[BD];
#pragma unroll
    for (int i = 0; i < BD; ++i) acc[i] = 0.0;
    for (uint64_t t = 0; t < a.bc; ++t) {
      double da[BC];
      decompress_exact_full(load_block(a, bi * a.bc + t), B, da);
      const RBlock bb = load_block(b, bi * b.bc + t);
      const uint64_t rem = a.cols - t * BD;
      const int jlim = rem < BD ? (int)rem : BD;
      decompress_exact(bb, B, [&](int u, const double (&row)[BD]) {
#pragma unroll
        for (int j = 0; j < BD; ++j)
          if (j < jlim) acc[u] += da[u * BD + j] * row[j];
      });
    }
#pragma unroll
    for (int i = 0; i < BD; ++i)
      if (bi * BD + i < a.rows) r[bi * BD + i] = acc[i];
  }
}

__global__ void k_sum(const double* __restrict__ v, uint64_t n, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (uint64_t k = 0; k < n; ++k) s += v[k];
    *out = s;
  }
}

cudaError_t launch_dot_entries(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b,
                               const uint64_t* i, const uint64_t* j, uint64_t n, double* out) {
  if (n == 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + 127) / 128 < (uint64_t)c.sm_count * 16 ? (n + 127) / 128
                                                                             : (uint64_t)c.sm_count * 16);
  k_dot_entries<<<g, 128, 0, c.stream>>>(B, a, b, i, j, n, out, c.err);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_rowdot(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b, double* r) {
  const unsigned g = (unsigned)((a.br + 127) / 128);
  k_rowdot<<<g ? g : 1, 128, 0, c.stream>>>(B, a, b, r);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_sum(const LaunchCtx& c, const double* v, uint64_t n, double* out) {
  k_sum<<<1, 32, 0, c.stream>>>(v, n, out);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
