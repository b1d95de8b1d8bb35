// io.cu -- device-side .blzc container I/O.
//
// write_compressed / read_compressed (H/io.hpp:93-134): a 13-byte header
// ("BLZC", version 1, rows and cols as little-endian u32) followed by one
// 45-byte record per block in row-major grid order: f and s as little-endian
// binary64, the scale byte, the 28 coefficients in keep-set order.  A warp
// owns 32 consecutive records (1,440 contiguous bytes): it assembles them in
// shared memory and moves them with coalesced byte accesses (the record
// stream is only byte-aligned: 13 + 45 t).  Validation follows the reference:
//   write: non-finite f or s -> "write_compressed: non-finite block field"
//   read : scale factor 0    -> "compressed matrix: zero scale factor in block t"
// (header and truncation checks are done on the host, capi.cu).
#include "blaz_device.cuh"
#include "launch.h"

namespace blz {

constexpr int REC = 45;

__device__ __forceinline__ void put_u64(uint8_t* p, unsigned long long v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ unsigned long long get_u64(const uint8_t* p) {
  unsigned long long v = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) v |= (unsigned long long)p[i] << (8 * i);
  return v;
}

__global__ void __launch_bounds__(128) k_pack_blzc(CMat in, uint8_t* __restrict__ out, unsigned long long* err) {
  __shared__ uint8_t stage[4][32 * REC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* S = stage[warp];
  const uint64_t nb = in.nb();
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // header (H/io.hpp:70-76)
    out[0] = 'B';
    out[1] = 'L';
    out[2] = 'Z';
    out[3] = 'C';
    out[4] = 1;
    const uint32_t r = (uint32_t)in.rows, c = (uint32_t)in.cols;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      out[5 + i] = (uint8_t)(r >> (8 * i));
      out[9 + i] = (uint8_t)(c >> (8 * i));
    }
  }
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t0 = gw * 32; t0 < nb; t0 += nw * 32) {
    const uint64_t t = t0 + lane;
    if (t < nb) {
      const RBlock b = load_block(in, t);
      if (!is_finite(b.f) || !is_finite(b.s)) latch_error(err, t, DERR_IO_NONFINITE_CODE);  // H/io.hpp:102-103
      uint8_t* r = S + lane * REC;
      put_u64(r, (unsigned long long)__double_as_longlong(b.f));
      put_u64(r + 8, (unsigned long long)__double_as_longlong(b.s));
      r[16] = (uint8_t)b.phi;
#pragma unroll
      for (int k = 0; k < KEPT; ++k) r[17 + k] = (uint8_t)(b.c[k >> 2] >> (8 * (k & 3)));
    }
    __syncwarp();
    const uint64_t n = min((uint64_t)32, nb - t0);
    uint8_t* dst = out + 13 + t0 * REC;
    for (int i = lane; i < (int)(n * REC); i += 32) dst[i] = S[i];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(128) k_unpack_blzc(const uint8_t* __restrict__ in, CMat out, uint64_t nlimit,
                                                     unsigned long long* err) {
  __shared__ uint8_t stage[4][32 * REC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* S = stage[warp];
  const uint64_t nb = min(out.nb(), nlimit);  // records present (truncated streams: a prefix)
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t0 = gw * 32; t0 < nb; t0 += nw * 32) {
    const uint64_t n = min((uint64_t)32, nb - t0);
    const uint8_t* src = in + 13 + t0 * REC;
    for (int i = lane; i < (int)(n * REC); i += 32) S[i] = src[i];
    __syncwarp();
    const uint64_t t = t0 + lane;
    if (t < nb) {
      const uint8_t* r = S + lane * REC;
      RBlock b;
      b.f = __longlong_as_double((long long)get_u64(r));
      b.s = __longlong_as_double((long long)get_u64(r + 8));
      b.phi = r[16];
      if (b.phi == 0) latch_error(err, t, DERR_IO_ZERO_PHI_CODE);  // H/io.hpp:129-130
#pragma unroll
      for (int w = 0; w < 7; ++w)
        b.c[w] = (uint32_t)r[17 + 4 * w] | ((uint32_t)r[18 + 4 * w] << 8) | ((uint32_t)r[19 + 4 * w] << 16) |
                 ((uint32_t)r[20 + 4 * w] << 24);
      store_block(out, t, b);
    }
    __syncwarp();
  }
}

static unsigned io_grid(uint64_t nb, int sms) {
  const uint64_t warps = (nb + 31) / 32;
  const uint64_t want = (warps + 3) / 4;
  const uint64_t cap = (uint64_t)sms * 16;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_pack_blzc(const LaunchCtx& c, const CMat& in, uint8_t* out) {
  k_pack_blzc<<<io_grid(in.nb(), c.sm_count), 128, 0, c.stream>>>(in, out, c.err);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_unpack_blzc(const LaunchCtx& c, const uint8_t* in, const CMat& out, uint64_t nlimit) {
  k_unpack_blzc<<<io_grid(out.nb(), c.sm_count), 128, 0, c.stream>>>(in, out, nlimit, c.err);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
