// launch.h -- host-side launchers implemented by the kernel translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "blaz_types.h"

namespace blz {

struct FastInfo {
  double ss00;     // RN(sigma_0^2) of the uploaded basis (extended-precision host sum)
  double bfly[8];  // 1/sqrt(8), cos(k pi/16)/2 for k = 1..7, correctly rounded
};

struct LaunchCtx {
  cudaStream_t stream;
  unsigned long long* err;       // device error latch (lowest block index wins)
  uint64_t* launches;            // host counter of kernel launches
  int sm_count;
  bool exact_only;               // BLZ_MODE_EXACT: reference-order kernels only
  const FastInfo* fast;          // null when the basis does not admit the verified path
  uint64_t* wl;                  // exact-path worklist (nb entries)
  unsigned long long* wl_count;  // worklist length
  unsigned long long* stats;     // [0] compress exact-path blocks, [1] add/sub dense-fallback blocks
  bool basis_sym;                // basis has the reference's repeated magnitudes (blaz_device.cuh, BasisSym)
  bool basis_bound;              // basis is the one bound to the device's c_basis_pairs (codec.cu)
};

// compress_pair.cu (verified fast path, two threads per block)
struct FastParams;
cudaError_t launch_compress_pair(const LaunchCtx& c, const FastParams& P, const double* dense, uint64_t rows,
                                 uint64_t cols, uint64_t ld, const CMat& out);
// compress_exact_warp.cu (exact compress of the worklist, one warp per block)
cudaError_t launch_compress_worklist_warp(const LaunchCtx& c, const Basis& B, const double* dense, uint64_t rows,
                                          uint64_t cols, uint64_t ld, const CMat& out);
// codec.cu
cudaError_t launch_compress(const LaunchCtx& c, const Basis& B, const double* dense, uint64_t rows,
                            uint64_t cols, uint64_t ld, const CMat& out);
cudaError_t launch_dequantize(const LaunchCtx& c, const Basis& B, const CMat& in, double* tiles);
// binds B to the current device's constant basis pairs (first basis per device wins)
cudaError_t bind_decompress_basis(const Basis& B, bool* bound);
cudaError_t launch_decompress(const LaunchCtx& c, const Basis& B, const CMat& in, double* dense,
                              uint64_t ld, uint64_t crop_rows, uint64_t crop_cols);
// A matrix held as consecutive block-row shards in separate SoA arrays (other
// ranks' shards through peer pointers): part[r] holds block-rows [lo[r], lo[r+1]).
struct ShardSet {
  static constexpr int kMax = 16;
  CMat part[kMax];
  uint64_t lo[kMax + 1];
  int n;
};
cudaError_t launch_decompress_gather(const LaunchCtx& c, const Basis& B, const ShardSet& S, uint64_t bc,
                                     double* dense, uint64_t ld, uint64_t crop_rows, uint64_t crop_cols);
// ops.cu
cudaError_t launch_addsub_fallback(const LaunchCtx& c, const Basis& B, bool sub, const CMat& a, const CMat& b,
                                   const CMat& out);
// fused.cu (op followed by decompress; op 0 add, 1 sub, 2 scale)
cudaError_t launch_op_decompress(const LaunchCtx& c, const Basis& B, int op, const CMat& a, const CMat& b, double k,
                                 const CMat& out, double* dense, uint64_t ld, uint64_t crop_rows, uint64_t crop_cols);
cudaError_t launch_addsub(const LaunchCtx& c, const Basis& B, bool sub, const CMat& a, const CMat& b,
                          const CMat& out);
cudaError_t launch_scale(const LaunchCtx& c, const CMat& a, double k, const CMat& out);
cudaError_t launch_pack_aos(const LaunchCtx& c, const CMat& in, void* aos);
cudaError_t launch_unpack_aos(const LaunchCtx& c, const void* aos, const CMat& out);
// addsub.cu (coalesced warp-staged variants; false if the SoA arrays are not 16-byte aligned)
bool launch_addsub_v2(const LaunchCtx& c, bool sub, const CMat& a, const CMat& b, const CMat& out, cudaError_t* err);
bool launch_scale_v2(const LaunchCtx& c, const CMat& a, double k, const CMat& out, cudaError_t* err);
// blockops.cu (batched block-level API)
cudaError_t launch_reconstruct(const LaunchCtx& c, const Basis& B, bool cols, const CMat& in, int last,
                               double* tiles);
cudaError_t launch_block_mul(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b, double* tiles);
// metadata-only scale: f and s (phi / C are shared with the input)
cudaError_t launch_scale_fs(const LaunchCtx& c, const double* f, const double* s, double k, double* fo, double* so,
                            uint64_t nb);
// io.cu (.blzc container)
cudaError_t launch_pack_blzc(const LaunchCtx& c, const CMat& in, uint8_t* out);
cudaError_t launch_unpack_blzc(const LaunchCtx& c, const uint8_t* in, const CMat& out, uint64_t nlimit);
// dot.cu
// prod (nullable): n * a.bc * 8 doubles of scratch; with it, up to
// kDotSplitMaxQueries queries spread each query's inner blocks over threads
constexpr uint64_t kDotSplitMaxQueries = 16;
cudaError_t launch_dot_entries(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b,
                               const uint64_t* i, const uint64_t* j, uint64_t n, double* out, uint64_t row0,
                               uint64_t rows_total, double* prod = nullptr);
// total != null: also the ascending total of r (inside the split kernel, or by
// k_sum after the unsplit one)
cudaError_t launch_rowdot(const LaunchCtx& c, const Basis& B, const CMat& a, const CMat& b, double* r,
                          void* scratch = nullptr, double* total = nullptr);
// scratch for the split persistent row-dot kernel (counter, flags, chain state)
uint64_t rowdot_scratch_bytes(const CMat& a);
cudaError_t launch_sum(const LaunchCtx& c, const double* v, uint64_t n, double* out);
// stages.cu (batched stage functions of the codec, one thread per block)
enum StageId { STAGE_NORMALIZE = 1, STAGE_DENORMALIZE, STAGE_MEAN_SLOPE, STAGE_PREDICT, STAGE_QUANTIZE, STAGE_DCT2,
               STAGE_IDCT2 };
cudaError_t launch_stage(const LaunchCtx& c, const Basis& B, int stage, const double* in0, const double* in1,
                         uint64_t n, double* out0, double* out1, double* out2, void* out3);
// harness.cu (evaluation-harness reduction)
cudaError_t launch_mean_rel_error(const LaunchCtx& c, const double* ref, const double* cand, uint64_t n,
                                  double* mean, unsigned long long* excluded);
// gemm.cu
cudaError_t launch_gemm(const LaunchCtx& c, int mode, const double* A, uint64_t lda, const double* Bm,
                        uint64_t ldb, double* Cm, uint64_t ldc, uint64_t M, uint64_t N, uint64_t K,
                        bool acc_c = false);

}  // namespace blz
