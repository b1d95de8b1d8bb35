// ops.cu -- K3 add/sub, K4 scale, K8 AoS<->SoA pack (exact mode).
//
// mat_add / mat_sub (H/matrix.hpp:128-144 -> H/block_ops.hpp:20-71) run in
// two kernels: the fast kernel handles every block except the rare
// s1 + s2 == 0 dense fallback (H/block_ops.hpp:36-44), whose block indices it
// appends to a device worklist; the fallback kernel then decompresses both
// operands, combines them densely and recompresses (same arithmetic as the
// reference).  mat_scale (H/matrix.hpp:146-151 -> H/block_ops.hpp:74-77)
// touches f and s and copies phi/C.
#include "blaz_device.cuh"
#include "launch.h"

namespace blz {

template <bool SUB>
__global__ void __launch_bounds__(256) k_addsub(CMat a, CMat b, CMat out, uint64_t* __restrict__ fb_list,
                                                unsigned long long* __restrict__ fb_count) {
  const uint64_t nb = out.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const RBlock b1 = load_block(a, t);
    const RBlock b2 = load_block(b, t);
    RBlock r;
    if (combine_fast<SUB>(b1, b2, r)) {
      store_block(out, t, r);
    } else {
      const unsigned long long slot = atomicAdd(fb_count, 1ull);
      fb_list[slot] = t;
    }
  }
}

// H/block_ops.hpp:36-44: decompress both, dense +/-, compress_block.
template <bool SUB>
__global__ void __launch_bounds__(128) k_addsub_fallback(const Basis B, CMat a, CMat b, CMat out,
                                                         const uint64_t* __restrict__ fb_list,
                                                         const unsigned long long* __restrict__ fb_count,
                                                         unsigned long long* err, unsigned long long* stats) {
  const uint64_t n = *fb_count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(stats, (unsigned long long)n);
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = fb_list[q];
    const RBlock b1 = load_block(a, t);
    const RBlock b2 = load_block(b, t);
    double d1[BC], d2[BC];
    decompress_exact_full(b1, B, d1);
    decompress_exact_full(b2, B, d2);
    const double rhs = SUB ? -1.0 : 1.0;
#pragma unroll
    for (int k = 0; k < BC; ++k) d1[k] = d1[k] + rhs * d2[k];
    RBlock r;
    const uint32_t e = compress_exact(d1, B, r);
    if (e != DERR_NONE) latch_error(err, t, e);
    store_block(out, t, r);
  }
}

__global__ void __launch_bounds__(256) k_scale(CMat a, double c, CMat out) {
  const uint64_t nb = out.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb;
       t += (uint64_t)gridDim.x * blockDim.x) {
    RBlock r = load_block(a, t);
    r.f = r.f * c;
    r.s = r.s * c;
    store_block(out, t, r);
  }
}

// 48-byte AoS record (blz_block / blaz::compressed_block) <-> SoA.
__device__ __forceinline__ void record_words(const RBlock& r, uint32_t (&w)[12]) {
  const unsigned long long fb = __double_as_longlong(r.f), sb = __double_as_longlong(r.s);
  w[0] = (uint32_t)fb;
  w[1] = (uint32_t)(fb >> 32);
  w[2] = (uint32_t)sb;
  w[3] = (uint32_t)(sb >> 32);
  // byte 16 = phi, bytes 17..44 = coeffs, 45..47 = pad (0)
  w[4] = r.phi & 0xff;
#pragma unroll
  for (int k = 5; k < 12; ++k) w[k] = 0;
#pragma unroll
  for (int k = 0; k < KEPT; ++k) {
    const uint32_t byte = (uint32_t)(get_coeff(r.c, k) & 0xff);
    const int pos = 17 + k;
    w[pos >> 2] |= byte << (8 * (pos & 3));
  }
}

__device__ __forceinline__ RBlock record_from_words(const uint32_t (&w)[12]) {
  RBlock r;
  r.f = __longlong_as_double(((long long)w[1] << 32) | w[0]);
  r.s = __longlong_as_double(((long long)w[3] << 32) | w[2]);
  r.phi = w[4] & 0xff;
#pragma unroll
  for (int q = 0; q < 7; ++q) r.c[q] = 0;
#pragma unroll
  for (int k = 0; k < KEPT; ++k) {
    const int pos = 17 + k;
    const int c = (int)(int8_t)(uint8_t)(w[pos >> 2] >> (8 * (pos & 3)));
    put_coeff(r.c, k, c);
  }
  return r;
}

// A warp moves its 32 records (1536 contiguous bytes) as 96 16-byte chunks,
// lane i taking chunks i, i + 32, i + 64: every store / load instruction covers
// 512 contiguous bytes.  That matters most when `aos` is page-locked host
// memory accessed zero-copy over PCIe (the host entry points), where 16-byte
// pieces 48 bytes apart would each become a separate PCIe transaction.
// Requires a 16-byte aligned `aos` (checked by the launchers); the partial
// last group of a grid goes record by record.
constexpr int AOS_THREADS = 256;

__global__ void __launch_bounds__(AOS_THREADS) k_pack_aos(CMat in, uint8_t* __restrict__ aos) {
  __shared__ __align__(16) uint4 stage[AOS_THREADS / 32][96];
  const uint64_t nb = in.nb();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint4* st = stage[warp];
  for (uint64_t t0 = gw * 32; t0 < nb; t0 += nw * 32) {
    const uint64_t t = t0 + lane;
    uint32_t w[12];
    if (t < nb) record_words(load_block(in, t), w);
    if (t0 + 32 <= nb) {
      st[3 * lane + 0] = make_uint4(w[0], w[1], w[2], w[3]);
      st[3 * lane + 1] = make_uint4(w[4], w[5], w[6], w[7]);
      st[3 * lane + 2] = make_uint4(w[8], w[9], w[10], w[11]);
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(aos + t0 * 48);
#pragma unroll
      for (int q = 0; q < 3; ++q) dst[lane + 32 * q] = st[lane + 32 * q];
      __syncwarp();
    } else if (t < nb) {
      uint4* dst = reinterpret_cast<uint4*>(aos + t * 48);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      dst[2] = make_uint4(w[8], w[9], w[10], w[11]);
    }
  }
}

__global__ void __launch_bounds__(AOS_THREADS) k_unpack_aos(const uint8_t* __restrict__ aos, CMat out) {
  __shared__ __align__(16) uint4 stage[AOS_THREADS / 32][96];
  const uint64_t nb = out.nb();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint4* st = stage[warp];
  for (uint64_t t0 = gw * 32; t0 < nb; t0 += nw * 32) {
    const uint64_t t = t0 + lane;
    uint4 q0, q1, q2;
    if (t0 + 32 <= nb) {
      const uint4* src = reinterpret_cast<const uint4*>(aos + t0 * 48);
#pragma unroll
      for (int q = 0; q < 3; ++q) st[lane + 32 * q] = src[lane + 32 * q];
      __syncwarp();
      q0 = st[3 * lane + 0];
      q1 = st[3 * lane + 1];
      q2 = st[3 * lane + 2];
      __syncwarp();
    } else if (t < nb) {
      const uint4* src = reinterpret_cast<const uint4*>(aos + t * 48);
      q0 = src[0];
      q1 = src[1];
      q2 = src[2];
    }
    if (t < nb) {
      const uint32_t w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
      store_block(out, t, record_from_words(w));
    }
  }
}

// Record-by-record variants for AoS buffers that are not 16-byte aligned.
__global__ void __launch_bounds__(256) k_pack_aos_u(CMat in, uint8_t* __restrict__ aos) {
  const uint64_t nb = in.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb; t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t w[12];
    record_words(load_block(in, t), w);
    uint2* dst = reinterpret_cast<uint2*>(aos + t * 48);  // blz_block is 8-byte aligned
#pragma unroll
    for (int k = 0; k < 6; ++k) dst[k] = make_uint2(w[2 * k], w[2 * k + 1]);
  }
}

__global__ void __launch_bounds__(256) k_unpack_aos_u(const uint8_t* __restrict__ aos, CMat out) {
  const uint64_t nb = out.nb();
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nb; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint2* src = reinterpret_cast<const uint2*>(aos + t * 48);
    uint32_t w[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const uint2 v = src[k];
      w[2 * k] = v.x;
      w[2 * k + 1] = v.y;
    }
    store_block(out, t, record_from_words(w));
  }
}

static unsigned grid_for(uint64_t n, unsigned threads, int sms) {
  const uint64_t want = (n + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sms * 32;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_addsub(const LaunchCtx& c, const Basis& B, bool sub, const CMat& a, const CMat& b,
                          const CMat& out) {
  cudaError_t e = cudaMemsetAsync(c.wl_count, 0, sizeof(unsigned long long), c.stream);
  if (e != cudaSuccess) return e;
  const unsigned g = grid_for(out.nb(), 256, c.sm_count);
  cudaError_t ev2 = cudaSuccess;
  if (launch_addsub_v2(c, sub, a, b, out, &ev2)) {
    if (ev2 != cudaSuccess) return ev2;
    --*c.launches;  // counted again below with the fallback kernel
  } else if (sub) {
    k_addsub<true><<<g, 256, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  } else {
    k_addsub<false><<<g, 256, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  }
  ++*c.launches;
  return launch_addsub_fallback(c, B, sub, a, b, out);
}

// Recomputes the worklisted s1 + s2 == 0 blocks (count read on the device).
cudaError_t launch_addsub_fallback(const LaunchCtx& c, const Basis& B, bool sub, const CMat& a, const CMat& b,
                                   const CMat& out) {
  const unsigned gf = (unsigned)c.sm_count;
  if (sub)
    k_addsub_fallback<true><<<gf, 128, 0, c.stream>>>(B, a, b, out, c.wl, c.wl_count, c.err, c.stats + 1);
  else
    k_addsub_fallback<false><<<gf, 128, 0, c.stream>>>(B, a, b, out, c.wl, c.wl_count, c.err, c.stats + 1);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_scale(const LaunchCtx& c, const CMat& a, double k, const CMat& out) {
  cudaError_t ev2 = cudaSuccess;
  if (launch_scale_v2(c, a, k, out, &ev2)) return ev2;
  k_scale<<<grid_for(out.nb(), 256, c.sm_count), 256, 0, c.stream>>>(a, k, out);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_pack_aos(const LaunchCtx& c, const CMat& in, void* aos) {
  const unsigned g = grid_for(in.nb(), AOS_THREADS, c.sm_count);
  if ((reinterpret_cast<uintptr_t>(aos) & 15) == 0)
    k_pack_aos<<<g, AOS_THREADS, 0, c.stream>>>(in, (uint8_t*)aos);
  else
    k_pack_aos_u<<<g, 256, 0, c.stream>>>(in, (uint8_t*)aos);
  ++*c.launches;
  return cudaGetLastError();
}

cudaError_t launch_unpack_aos(const LaunchCtx& c, const void* aos, const CMat& out) {
  const unsigned g = grid_for(out.nb(), AOS_THREADS, c.sm_count);
  if ((reinterpret_cast<uintptr_t>(aos) & 15) == 0)
    k_unpack_aos<<<g, AOS_THREADS, 0, c.stream>>>((const uint8_t*)aos, out);
  else
    k_unpack_aos_u<<<g, 256, 0, c.stream>>>((const uint8_t*)aos, out);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
