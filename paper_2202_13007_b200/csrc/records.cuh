// records.cuh -- warp-group staging of compressed records in shared memory.
//
// A warp owns 32 consecutive blocks of the SoA layout: their records (f, s: 8 B;
// C: 28 B; phi: 1 B) are 256 + 256 + 896 + 32 contiguous bytes, loaded with
// coalesced 16-byte cp.async copies (no registers held while in flight) into a
// WarpRecs slot, and stored back the same way.  Shared by add/sub (addsub.cu)
// and the staged decompress (codec.cu).
#pragma once
#include "blaz_device.cuh"

namespace blz {

struct __align__(16) WarpRecs {
  double f[32];
  double s[32];
  uint32_t c[32 * 7];
  uint8_t phi[32];
};

__device__ __forceinline__ double i8_to_double(int c) {
  return __hiloint2double(0x43300000, (int)((uint32_t)c ^ 0x80000000u)) - 4503601774854144.0;
}

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// predicated 16-byte copy (no branch around it)
__device__ __forceinline__ void cp16_if(bool pred, void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(sa),
               "l"(gmem), "r"((int)pred)
               : "memory");
}
__device__ __forceinline__ void st16_if(bool pred, void* gmem, uint4 v) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %5, 0; @p st.global.v4.b32 [%0], {%1, %2, %3, %4}; }" ::"l"(gmem),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"((int)pred)
               : "memory");
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Starts the (coalesced, asynchronous) load of the 32 records starting at
// block t0; the partial last group is loaded synchronously.
__device__ __forceinline__ void load_recs(const CMat& m, uint64_t t0, uint64_t nb, int lane, WarpRecs& r) {
  if (t0 + 32 <= nb) {
    // f and s are adjacent in WarpRecs: lanes 0-15 copy f, 16-31 copy s (selects, no branches)
    const double* fs = lane < 16 ? m.first + t0 + 2 * lane : m.slope + t0 + 2 * (lane - 16);
    cp16(&r.f[2 * lane], fs);
    cp16_if(lane < 2, &r.phi[16 * lane], m.scale + t0 + 16 * lane);  // idle lanes: no access
    const uint8_t* src = reinterpret_cast<const uint8_t*>(m.coeffs + t0 * 28);
    uint8_t* dst = reinterpret_cast<uint8_t*>(r.c);
    cp16(dst + 16 * lane, src + 16 * lane);
    cp16_if(lane < 24, dst + 16 * (32 + lane), src + 16 * (32 + lane));  // idle lanes: no access
  } else {
    const uint64_t t = t0 + lane;
    if (t < nb) {
      r.f[lane] = m.first[t];
      r.s[lane] = m.slope[t];
      r.phi[lane] = m.scale[t];
      const uint32_t* cw = reinterpret_cast<const uint32_t*>(m.coeffs + t * 28);
#pragma unroll
      for (int w = 0; w < 7; ++w) r.c[lane * 7 + w] = cw[w];
    }
  }
}

__device__ __forceinline__ void store_recs(const CMat& m, uint64_t t0, uint64_t nb, int lane, const WarpRecs& r) {
  __syncwarp();
  if (t0 + 32 <= nb) {
    double* fs = lane < 16 ? m.first + t0 + 2 * lane : m.slope + t0 + 2 * (lane - 16);
    *reinterpret_cast<double2*>(fs) = reinterpret_cast<const double2*>(r.f)[lane];
    m.scale[t0 + lane] = r.phi[lane];
    const uint4* src = reinterpret_cast<const uint4*>(r.c);
    uint4* dst = reinterpret_cast<uint4*>(m.coeffs + t0 * 28);
    dst[lane] = src[lane];
    const int l2 = lane < 24 ? 32 + lane : lane;  // in-bounds shared read for the idle lanes
    st16_if(lane < 24, dst + l2, src[l2]);
  } else {
    const uint64_t t = t0 + lane;
    if (t < nb) {
      m.first[t] = r.f[lane];
      m.slope[t] = r.s[lane];
      m.scale[t] = r.phi[lane];
      uint32_t* cw = reinterpret_cast<uint32_t*>(m.coeffs + t * 28);
#pragma unroll
      for (int w = 0; w < 7; ++w) cw[w] = r.c[lane * 7 + w];
    }
  }
}

}  // namespace blz
