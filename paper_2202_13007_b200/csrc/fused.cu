// fused.cu -- SURVEY.md 8(f)2, fused op chains: add / sub / scale followed by the
// decompression of the result, in one pass.
//
// mat_add / mat_sub / mat_scale (H/matrix.hpp:128-151) and then decompress_matrix
// (:113-126) of the result.  Each thread combines (or scales) one block's record
// with exactly the arithmetic of addsub.cu / the scale kernel, stores the record
// (the compressed result is still produced), and decompresses it from registers
// with the same kernel body as k_decompress.  Relative to the two-kernel chain
// this saves the 45-byte re-read of every result record and a launch, and the
// FP64-bound decompress hides the combine's integer work.  Results are bitwise
// those of the unfused chain.
//
// s1 + s2 == 0 blocks (the dense fallback, H/block_ops.hpp:36-44) go to the
// worklist: k_addsub_fallback recomputes their records and k_decompress_list
// decompresses them afterwards.
#include "combine.cuh"
#include "launch.h"

namespace blz {

namespace {

template <bool SYM>
struct Emitter {
  double* dense;
  uint64_t ld, r0, c0, crop_rows, crop_cols;
  bool full, part, v4;
  __device__ __forceinline__ void operator()(int u, const double (&row)[BD]) const {
    if (full) {
      store_row8(dense + (r0 + u) * ld + c0, row, v4);
    } else if (part && r0 + u < crop_rows) {
#pragma unroll
      for (int j = 0; j < BD; ++j)
        if (c0 + j < crop_cols) dense[(r0 + u) * ld + c0 + j] = row[j];
    }
  }
};

// OP: 0 add, 1 sub, 2 scale
template <int OP, bool SYM>
__global__ void __launch_bounds__(128, 4)
    k_op_decompress(const Basis B, CMat a, CMat b, double k, CMat out, double* __restrict__ dense, uint64_t ld,
                    uint64_t crop_rows, uint64_t crop_cols, uint64_t* __restrict__ wl,
                    unsigned long long* __restrict__ wl_count) {
  const uint64_t nb = out.nb();
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool aligned = ((ld & 1) == 0) && (reinterpret_cast<uintptr_t>(dense) & 15) == 0;
  const bool v4 = rows_v4(dense, ld);
  for (uint64_t base = warp0 * 32; base < nb; base += nwarps * 32) {
    const uint64_t t = base + lane;
    const bool valid = t < nb;
    const uint64_t tt = valid ? t : nb - 1;
    const uint64_t bi = tt / out.bc, bj = tt % out.bc;
    const RBlock ra = load_block(a, tt);
    RBlock r;
    bool fb = false;
    if (OP == 2) {  // scale (H/block_ops.hpp:74-77)
      r = ra;
      r.f = ra.f * k;
      r.s = ra.s * k;
    } else {
      const RBlock rb = load_block(b, tt);
      const CombineOut o = combine_record<OP == 1>(ra.f, ra.s, ra.phi, ra.c, rb.f, rb.s, rb.phi, rb.c);
      r.f = o.f;
      r.s = o.s;
      r.phi = o.phi;
#pragma unroll
      for (int w = 0; w < 7; ++w) r.c[w] = o.c[w];
      fb = o.fallback;
      if (o.slow && valid && !fb) {  // huge weights: the reference rounding sequence
        const int8_t* b1 = reinterpret_cast<const int8_t*>(a.coeffs + t * KEPT);
        const int8_t* b2 = reinterpret_cast<const int8_t*>(b.coeffs + t * KEPT);
        int8_t* bo = reinterpret_cast<int8_t*>(out.coeffs + t * KEPT);
#pragma unroll 1
        for (int q = 0; q < KEPT; ++q) bo[q] = (int8_t)clamp_coeff(o.w1 * (double)b1[q] + o.w2 * (double)b2[q]);
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(out.coeffs + t * KEPT);
#pragma unroll
        for (int w = 0; w < 7; ++w) r.c[w] = cw[w];
      }
    }
    if (valid) {
      if (fb) wl[atomicAdd(wl_count, 1ull)] = t;
      else store_block(out, t, r);
    }
    const uint64_t r0 = bi * BD, c0 = bj * BD;
    Emitter<SYM> em{dense, ld, r0, c0, crop_rows, crop_cols, false, valid && !fb, v4};
    em.full = em.part && aligned && r0 + BD <= crop_rows && c0 + BD <= crop_cols;
    decompress_exact<SYM>(r, B, em);
  }
}

// Decompresses the blocks named by the worklist (after k_addsub_fallback wrote them).
__global__ void __launch_bounds__(128) k_decompress_list(const Basis B, CMat m, const uint64_t* __restrict__ wl,
                                                         const unsigned long long* __restrict__ wl_count,
                                                         double* __restrict__ dense, uint64_t ld, uint64_t crop_rows,
                                                         uint64_t crop_cols) {
  const uint64_t n = *wl_count;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = wl[q];
    const RBlock rb = load_block(m, t);
    const uint64_t r0 = (t / m.bc) * BD, c0 = (t % m.bc) * BD;
    Emitter<false> em{dense, ld, r0, c0, crop_rows, crop_cols, false, true, false};
    decompress_exact<false>(rb, B, em);
  }
}

}  // namespace

cudaError_t launch_op_decompress(const LaunchCtx& c, const Basis& B, int op, const CMat& a, const CMat& b, double k,
                                 const CMat& out, double* dense, uint64_t ld, uint64_t crop_rows, uint64_t crop_cols) {
  if (op != 2) {
    cudaError_t e = cudaMemsetAsync(c.wl_count, 0, sizeof(unsigned long long), c.stream);
    if (e != cudaSuccess) return e;
  }
  const uint64_t warps = (out.nb() + 31) / 32;
  const uint64_t want = (warps * 32 + 127) / 128;
  const uint64_t cap = (uint64_t)c.sm_count * 64;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  const bool sym = c.basis_sym && !c.exact_only;
#define BLZ_OPDEC(OPV, SYMV)                                                                                       \
  k_op_decompress<OPV, SYMV><<<g, 128, 0, c.stream>>>(B, a, b, k, out, dense, ld, crop_rows, crop_cols, c.wl, \
                                                      c.wl_count)
  if (op == 0) {
    if (sym) BLZ_OPDEC(0, true); else BLZ_OPDEC(0, false);
  } else if (op == 1) {
    if (sym) BLZ_OPDEC(1, true); else BLZ_OPDEC(1, false);
  } else {
    if (sym) BLZ_OPDEC(2, true); else BLZ_OPDEC(2, false);
  }
#undef BLZ_OPDEC
  ++*c.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || op == 2) return e;
  e = launch_addsub_fallback(c, B, op == 1, a, b, out);
  if (e != cudaSuccess) return e;
  k_decompress_list<<<(unsigned)c.sm_count, 128, 0, c.stream>>>(B, out, c.wl, c.wl_count, dense, ld, crop_rows,
                                                                 crop_cols);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
