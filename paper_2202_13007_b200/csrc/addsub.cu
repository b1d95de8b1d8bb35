// addsub.cu -- K3 add/sub and K4 scale over the SoA compressed layout.
//
// mat_add / mat_sub (H/matrix.hpp:128-144 -> H/block_ops.hpp:20-71).  A warp
// owns 32 consecutive blocks: their records (f, s: 8 B; phi: 1 B; C: 28 B) are
// loaded with coalesced 16-byte accesses into shared memory, combined per lane
// with exactly the reference's arithmetic, staged and stored coalesced.
//
// Exactness (combine.cuh):
//  * int8 -> double: I2F.F64.S8 on a byte lane (exact);
//  * the weight divisions s1 / s, s2 / s, a / p are correctly rounded quotients
//    from RN reciprocals plus one Markstein correction when the slopes lie in
//    [2^-400, 2^400]; otherwise IEEE divisions;
//  * round_half_away + clamp_coeff (H/block.hpp:61-81) for |v| < 2^30 as
//    sign(v) * min(trunc(RZ(|v| + 1/2)), 127), signs applied four bytes at a
//    time.  Larger |v| (s1 + s2 nearly cancelling) or NaN weights send the
//    block's 28 coefficients through the reference's own sequence (clamp_coeff).
// The s1 + s2 == 0 dense fallback (:36-44) is handed to k_addsub_fallback via
// the worklist.
#include "blaz_device.cuh"
#include "combine.cuh"
#include "fastpath.cuh"
#include "launch.h"
#include "records.cuh"

#ifndef ASB_GRID_PER_SM
#define ASB_GRID_PER_SM 96  // many short CTAs beat a resident grid (6/SM: 0.142 ms, 96: 0.126 ms)
#endif
#ifndef SCL_GRID_PER_SM
#define SCL_GRID_PER_SM 32
#endif

namespace blz {

// Requires 16-byte aligned SoA arrays whose block offset is a multiple of 4
// blocks (true for every blz_cmat_view-created matrix); the launcher checks.
// ALIAS: out is a or b (in-place use; the host compares the pointers).  The
// dense fallback (k_addsub_fallback) re-reads a[t] and b[t] afterwards, so a
// fallback lane must then leave the aliased input's record in place instead of
// storing its (meaningless) combined record.
template <bool SUB, bool ALIAS>
__global__ void __launch_bounds__(128) k_addsub_v2(CMat a, CMat b, CMat out, uint64_t* __restrict__ wl,
                                                   unsigned long long* __restrict__ wl_count) {
  __shared__ __align__(16) WarpRecs sa[2][4], sb[2][4], so[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t nb = out.nb();
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // out is disjoint from the inputs or identical to one of them (in place; host-checked)
  const int alias = out.first == a.first ? 1 : 2;  // used when ALIAS
  int buf = 0;
  uint64_t t0 = gw * 32;
  if (t0 < nb) {
    load_recs(a, t0, nb, lane, sa[0][warp]);
    load_recs(b, t0, nb, lane, sb[0][warp]);
  }
  cp_commit();
  for (; t0 < nb; t0 += nw * 32) {
    const uint64_t nx = t0 + nw * 32;
    if (nx < nb) {  // prefetch the next group while this one is combined
      load_recs(a, nx, nb, lane, sa[buf ^ 1][warp]);
      load_recs(b, nx, nb, lane, sb[buf ^ 1][warp]);
    }
    cp_commit();
    cp_wait1();
    __syncwarp();
    const WarpRecs& ra = sa[buf][warp];
    const WarpRecs& rb = sb[buf][warp];
    WarpRecs& ro = so[warp];
    const uint64_t t = t0 + lane;
    const double f1 = ra.f[lane], f2 = rb.f[lane], s1 = ra.s[lane], s2 = rb.s[lane];
    const uint32_t p1 = ra.phi[lane], p2 = rb.phi[lane];
    // the coefficient words straight from the staged records (each branch of the
    // combine loads what it uses; register copies between the branches cost 5 %)
    const CombineOut o = combine_record<SUB>(f1, s1, p1, SmemWords{&ra.c[lane * 7]}, f2, s2, p2,
                                             SmemWords{&rb.c[lane * 7]});
    const bool fallback = o.fallback, slow = o.slow;
    const double of = o.f, os = o.s, w1 = o.w1, w2 = o.w2;
    const uint32_t ophi = o.phi;
    uint32_t oc[7];
#pragma unroll
    for (int w = 0; w < 7; ++w) oc[w] = o.c[w];
    if (fallback && t < nb) wl[atomicAdd(wl_count, 1ull)] = t;
    if (ALIAS && fallback) {
      // k_addsub_fallback re-reads a[t] and b[t]: when out is one of the inputs
      // (in-place add/sub), that input's record must survive this store.
      const WarpRecs& keep = alias == 1 ? ra : rb;
      ro.f[lane] = keep.f[lane];
      ro.s[lane] = keep.s[lane];
      ro.phi[lane] = keep.phi[lane];
#pragma unroll
      for (int w = 0; w < 7; ++w) ro.c[lane * 7 + w] = keep.c[lane * 7 + w];
    } else {
      ro.f[lane] = of;
      ro.s[lane] = os;
      ro.phi[lane] = (uint8_t)ophi;
#pragma unroll
      for (int w = 0; w < 7; ++w) ro.c[lane * 7 + w] = oc[w];
    }
    if (slow && !(ALIAS && fallback)) {  // huge weights: the reference rounding sequence (blaz_device.cuh::clamp_coeff)
      const uint8_t* b1 = reinterpret_cast<const uint8_t*>(&ra.c[lane * 7]);
      const uint8_t* b2 = reinterpret_cast<const uint8_t*>(&rb.c[lane * 7]);
      uint8_t* bo = reinterpret_cast<uint8_t*>(&ro.c[lane * 7]);
#pragma unroll 1
      for (int k = 0; k < KEPT; ++k) {
        const double v = w1 * (double)(int8_t)b1[k] + w2 * (double)(int8_t)b2[k];
        bo[k] = (uint8_t)clamp_coeff(v);
      }
    }
    store_recs(out, t0, nb, lane, ro);
    __syncwarp();
    buf ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// mat_scale (H/block_ops.hpp:74-77): f*c, s*c; phi and C are copied, so the
// kernel is three flat streams with 16-byte accesses.
__global__ void __launch_bounds__(256) k_scale_v2(CMat a, double c, CMat out) {
  const uint64_t nb = out.nb();
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  // f and s, two blocks per 16-byte access
  const uint64_t n2 = nb / 2;
  for (uint64_t i = tid; i < n2; i += nth) {
    const double2 f = reinterpret_cast<const double2*>(a.first)[i];
    const double2 s = reinterpret_cast<const double2*>(a.slope)[i];
    reinterpret_cast<double2*>(out.first)[i] = make_double2(f.x * c, f.y * c);
    reinterpret_cast<double2*>(out.slope)[i] = make_double2(s.x * c, s.y * c);
  }
  if ((nb & 1) && tid == 0) {
    out.first[nb - 1] = a.first[nb - 1] * c;
    out.slope[nb - 1] = a.slope[nb - 1] * c;
  }
  // coefficients: nb*28 bytes = nb*7/4 16-byte chunks (+ tail words)
  const uint64_t cbytes = nb * 28;
  const uint64_t n16 = cbytes / 16;
  for (uint64_t i = tid; i < n16; i += nth)
    reinterpret_cast<uint4*>(out.coeffs)[i] = reinterpret_cast<const uint4*>(a.coeffs)[i];
  for (uint64_t i = n16 * 4 + tid; i < cbytes / 4; i += nth)
    reinterpret_cast<uint32_t*>(out.coeffs)[i] = reinterpret_cast<const uint32_t*>(a.coeffs)[i];
  // scale factors
  const uint64_t np = nb / 16;
  for (uint64_t i = tid; i < np; i += nth)
    reinterpret_cast<uint4*>(out.scale)[i] = reinterpret_cast<const uint4*>(a.scale)[i];
  for (uint64_t i = np * 16 + tid; i < nb; i += nth) out.scale[i] = a.scale[i];
}

// metadata-only mat_scale (H/block_ops.hpp:74-77 touches only f and s): two
// flat f64 streams, 16 B per block read and written (phi / C are aliased).
__global__ void __launch_bounds__(256) k_scale_fs(const double* __restrict__ f, const double* __restrict__ s, double c,
                                                  double* __restrict__ fo, double* __restrict__ so, uint64_t nb) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(fo) |
                     reinterpret_cast<uintptr_t>(so)) & 15) == 0;
  if (vec) {
    const uint64_t n2 = nb / 2;
    for (uint64_t i = tid; i < n2; i += nth) {
      const double2 a = reinterpret_cast<const double2*>(f)[i];
      const double2 b = reinterpret_cast<const double2*>(s)[i];
      reinterpret_cast<double2*>(fo)[i] = make_double2(a.x * c, a.y * c);
      reinterpret_cast<double2*>(so)[i] = make_double2(b.x * c, b.y * c);
    }
    if ((nb & 1) && tid == 0) {
      fo[nb - 1] = f[nb - 1] * c;
      so[nb - 1] = s[nb - 1] * c;
    }
  } else {
    for (uint64_t i = tid; i < nb; i += nth) {
      fo[i] = f[i] * c;
      so[i] = s[i] * c;
    }
  }
}

cudaError_t launch_scale_fs(const LaunchCtx& c, const double* f, const double* s, double k, double* fo, double* so,
                            uint64_t nb) {
  const uint64_t want = (nb / 2 + 255) / 256;
  const uint64_t cap = (uint64_t)c.sm_count * SCL_GRID_PER_SM;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  k_scale_fs<<<g, 256, 0, c.stream>>>(f, s, k, fo, so, nb);
  ++*c.launches;
  return cudaGetLastError();
}

static bool soa_aligned(const CMat& m) {
  return ((reinterpret_cast<uintptr_t>(m.first) | reinterpret_cast<uintptr_t>(m.slope) |
           reinterpret_cast<uintptr_t>(m.coeffs) | reinterpret_cast<uintptr_t>(m.scale)) & 15) == 0;
}

bool launch_addsub_v2(const LaunchCtx& c, bool sub, const CMat& a, const CMat& b, const CMat& out,
                      cudaError_t* err) {
  if (!soa_aligned(a) || !soa_aligned(b) || !soa_aligned(out)) return false;
  const uint64_t warps = (out.nb() + 31) / 32;
  const uint64_t want = (warps + 3) / 4;
  const uint64_t cap = (uint64_t)c.sm_count * ASB_GRID_PER_SM;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  const bool alias = out.first == a.first || out.first == b.first;
  if (sub && alias)
    k_addsub_v2<true, true><<<g, 128, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  else if (sub)
    k_addsub_v2<true, false><<<g, 128, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  else if (alias)
    k_addsub_v2<false, true><<<g, 128, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  else
    k_addsub_v2<false, false><<<g, 128, 0, c.stream>>>(a, b, out, c.wl, c.wl_count);
  ++*c.launches;
  *err = cudaGetLastError();
  return true;
}

bool launch_scale_v2(const LaunchCtx& c, const CMat& a, double k, const CMat& out, cudaError_t* err) {
  if (!soa_aligned(a) || !soa_aligned(out)) return false;
  const uint64_t n16 = out.nb() * 28 / 16;
  const uint64_t want = (n16 + 255) / 256;
  const uint64_t cap = (uint64_t)c.sm_count * SCL_GRID_PER_SM;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  k_scale_v2<<<g, 256, 0, c.stream>>>(a, k, out);
  ++*c.launches;
  *err = cudaGetLastError();
  return true;
}

}  // namespace blz
