// harness.cu -- GPU mean_relative_error of the evaluation harness.
//
// H/bench.hpp:67-84: mean of |(cand - ref) / ref| over the entries with
// |ref| >= 1e-12, summed serially in index order, divided by the kept count;
// excluded = n - kept.  The terms are formed by the whole CTA (IEEE division),
// the serial sum runs on one thread in the reference's order -- a running sum of
// non-negative terms that starts at +0.0 is never -0.0, so excluded entries add
// +0.0 (the identity) instead of being skipped.  Double-buffered chunks let the
// CTA form chunk c+1 while thread 0 sums chunk c.
#include "launch.h"

namespace blz {

namespace {

constexpr int MRE_THREADS = 256;
constexpr int MRE_CHUNK = 2048;

__global__ void __launch_bounds__(MRE_THREADS) k_mean_rel_error(const double* __restrict__ ref,
                                                                const double* __restrict__ cand, uint64_t n,
                                                                double* __restrict__ mean,
                                                                unsigned long long* __restrict__ excluded) {
  __shared__ double terms[2][MRE_CHUNK];
  __shared__ unsigned long long kept_total;
  if (threadIdx.x == 0) kept_total = 0;
  unsigned long long kept = 0;
  auto form = [&](uint64_t c, double* buf) {
    const uint64_t base = c * MRE_CHUNK;
    for (int k = threadIdx.x; k < MRE_CHUNK; k += MRE_THREADS) {
      const uint64_t q = base + k;
      double t = 0.0;
      if (q < n) {
        const double r = ref[q];
        if (!(fabs(r) < 1e-12)) {  // kept (NaN references are kept, as in the reference)
          t = fabs((cand[q] - r) / r);
          ++kept;
        }
      }
      buf[k] = t;
    }
  };
  const uint64_t chunks = (n + MRE_CHUNK - 1) / MRE_CHUNK;
  double sum = 0.0;
  if (chunks) form(0, terms[0]);
  __syncthreads();
  for (uint64_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) form(c + 1, terms[(c + 1) & 1]);
    if (threadIdx.x == 0) {
      const double* buf = terms[c & 1];
      const uint64_t left = n - c * MRE_CHUNK;
      const int m = left < (uint64_t)MRE_CHUNK ? (int)left : MRE_CHUNK;
      for (int k = 0; k < m; ++k) sum += buf[k];
    }
    __syncthreads();
  }
  atomicAdd(&kept_total, kept);
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long kt = kept_total;
    *mean = kt == 0 ? 0.0 : sum / (double)kt;
    *excluded = (unsigned long long)n - kt;
  }
}

}  // namespace

cudaError_t launch_mean_rel_error(const LaunchCtx& c, const double* ref, const double* cand, uint64_t n,
                                  double* mean, unsigned long long* excluded) {
  k_mean_rel_error<<<1, MRE_THREADS, 0, c.stream>>>(ref, cand, n, mean, excluded);
  ++*c.launches;
  return cudaGetLastError();
}

}  // namespace blz
