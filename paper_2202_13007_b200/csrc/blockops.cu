// blockops.cu -- the block-level API on the device, batched:
// reconstruct_rows / reconstruct_cols / block_mul (H/block_ops.hpp:87-142) over
// n blocks (or block pairs) of SoA compressed matrices, one thread per block.
//
// * reconstruct_rows(b, k): rows 0..k of decompress_block(b), other rows +0.0
//   (partial_reconstruction.values); the materialised rows are bitwise a prefix
//   of the full decompression (the reference's own contract, :79-80), so the
//   kernel decompresses in reference order and masks.
// * reconstruct_cols(b, k): columns 0..k, other columns +0.0 -- likewise.
// * block_mul(b1, b2): out(i,j) = sum_k d1(i,k) d2(k,j), k ascending from +0.0,
//   DMUL then DADD (-fmad=false): d2 is staged in shared memory, d1 streams
//   row by row out of the decompression.
#include "blaz_device.cuh"
#include "launch.h"

namespace blz {

namespace {

// Warp-uniform loops (valid lanes predicated), as k_decompress: the basis
// operands then stay warp-uniform.
template <bool COLS, bool SYM>
__global__ void __launch_bounds__(128, 4) k_reconstruct(const Basis B, CMat in, int last, double* __restrict__ tiles) {
  const uint64_t nb = in.nb();
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp0 * 32; base < nb; base += nwarps * 32) {
    const uint64_t t = base + lane;
    const bool valid = t < nb;
    const RBlock rb = load_block(in, valid ? t : nb - 1);
    double2* dst = reinterpret_cast<double2*>(tiles + t * 64);
    decompress_exact<SYM>(rb, B, [&](int u, const double (&row)[BD]) {
      if (!valid) return;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double x = row[2 * q], y = row[2 * q + 1];
        if (COLS) {
          x = 2 * q <= last ? x : 0.0;
          y = 2 * q + 1 <= last ? y : 0.0;
        } else if (u > last) {
          x = y = 0.0;
        }
        dst[u * 4 + q] = make_double2(x, y);
      }
    });
  }
}

constexpr int BM_THREADS = 64;
constexpr int BM_STRIDE = 65;  // doubles per thread slot: conflict-free column reads

template <bool SYM>
__global__ void __launch_bounds__(BM_THREADS) k_block_mul(const Basis B, CMat a, CMat b, double* __restrict__ tiles,
                                                       int zero) {
  __shared__ double d2s[BM_THREADS * BM_STRIDE];
  double* d2 = d2s + threadIdx.x * BM_STRIDE;
  const uint64_t nb = a.nb();
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp0 * 32; base < nb; base += nwarps * 32) {
    const uint64_t t = base + lane;
    const bool valid = t < nb;
    const uint64_t tt = valid ? t : nb - 1;
    decompress_exact<SYM>(load_block(b, tt), B, [&](int u, const double (&row)[BD]) {
#pragma unroll
      for (int v = 0; v < BD; ++v) d2[u * BD + v] = row[v];
    });
    __syncwarp();  // orders the two decompressions (no interleaving: half the live registers)
    double2* dst = reinterpret_cast<double2*>(tiles + t * 64);
    decompress_exact<SYM>(load_block(a, tt), B, [&](int i, const double (&row)[BD]) {
      double o[BD];
#pragma unroll
      for (int j = 0; j < BD; ++j) {
        double r = 0.0;  // H/block_ops.hpp:137-139
#pragma unroll
        for (int k = 0; k < BD; ++k) r += row[k] * d2[k * BD + j + zero * i];  // reloaded per row (no hoisting)
        o[j] = r;
      }
      if (valid) {
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[i * 4 + q] = make_double2(o[2 * q], o[2 * q + 1]);
      }
    });
  }
}

unsigned grid_for(uint64_t n, unsigned threads, int sms, unsigned per_sm) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sms * per_sm;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_reconstruct(const LaunchCtx& c, const Basis& B, bool cols, const CMat& in, int last,
                               double* tiles) {
  const unsigned g = grid_for(in.nb(), 128, c.sm_count, 32);
  const bool sym = c.basis_sym && !c.exact_only;
  if (cols) {
    if (sym) k_reconstruct<true, true><<<g, 128, 0, c.stream>>>(B, in, last, tiles);
    else k_reconstruct<true, false><<<g, 128, 0, c.stream>>>(B, in, last, tiles);
  } else {
    if (sym) k_reconstruct<false, true><<<g, 128, 0, c.stream>>>(B, in, last, tiles);
    else k_reconstruct<false, false><<<g, 128, 0, c.stream>>>(B, in, last, tiles);
  }
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_block_mul(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b, double* tiles) {
  const unsigned g = grid_for(a.nb(), BM_THREADS, c.sm_count, 32);
  if (c.basis_sym && !c.exact_only)
    k_block_mul<true><<<g, BM_THREADS, 0, c.stream>>>(B, a, b, tiles, 0);
  else
    k_block_mul<false><<<g, BM_THREADS, 0, c.stream>>>(B, a, b, tiles, 0);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
