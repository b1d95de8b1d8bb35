// capi.cu -- the C ABI (include/blaz_cuda.h) over the sm_100a kernels.
//
// Mirrors the reference's matrix API (proj/include/blaz/matrix.hpp): argument
// checks, error categories and messages follow the reference line cited at
// each check.  There is no CPU fallback: every numeric result comes from a
// kernel launched here.
#include <cuda_runtime.h>

#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blaz_cuda.h"
#include "launch.h"

static_assert(sizeof(blz_block) == 48, "blz_block must match blaz::compressed_block (48 B)");

struct blz_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;  // created with the context (non-blocking); blz_ctx_set_stream may replace it
  blz::Basis basis{};
  std::string err;
  unsigned long long* d_err = nullptr;
  uint64_t launches = 0;
  int sm_count = 148;
  int mode = BLZ_MODE_DEFAULT;
  bool fast_ok = false;        // basis admits the verified fast path
  bool basis_sym = false;      // basis has the reference's repeated magnitudes (decompress sharing)
  bool basis_bound = false;    // basis is the device's constant basis of the decompress kernel
  blz::FastInfo fast{};
  unsigned long long* d_stats = nullptr;  // [0] compress exact-path blocks, [1] add/sub dense fallbacks
  uint64_t* d_wl = nullptr;               // exact-path worklist: 256 B counter + capacity entries
  uint64_t wl_cap = 0;
  // host-level pipelining: copy-in / copy-out streams and per-chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> events;
  // pageable host buffers: page-locked staging slots (two per direction, grow-only)
  struct Stage {
    void* p = nullptr;
    size_t bytes = 0, off = 0;
    cudaEvent_t ev = nullptr;
    bool busy = false;  // a copy from / into the slot is in flight (ev recorded)
    struct Drain {
      void* dst;
      const void* src;
      size_t n;
    };
    std::vector<Drain> drains;  // D2H: host copies still to make out of the slot
  };
  Stage st_in[2], st_out[2];
  int cur = 0;  // slot of the chunk being issued
  int stage_pieces = 1;  // H2D pieces per chunk (reservation hint)
  // grow-only device scratch slots (host-level calls, add fallback worklist)
  struct Slot {
    void* p = nullptr;
    size_t bytes = 0;
  };
  Slot slots[9];
};

namespace {

enum SlotId { S_ROWDOT = 0, S_IN0, S_IN1, S_OUT, S_CM0, S_CM1, S_CM2, S_AUX, S_DOT };

blz_status set_err(blz_ctx* c, blz_status st, const std::string& msg) {
  if (c) c->err = msg;
  return st;
}

blz_status cuda_err(blz_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return BLZ_OK;
  if (e == cudaErrorMemoryAllocation)
    return set_err(c, BLZ_OUT_OF_MEMORY, std::string(where) + ": " + cudaGetErrorString(e));
  return set_err(c, BLZ_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

#define BLZ_CUDA(ctx, expr, where)                      \
  do {                                                  \
    cudaError_t e__ = (expr);                           \
    if (e__ != cudaSuccess) return cuda_err(ctx, e__, where); \
  } while (0)

uint64_t nblk(uint64_t n) { return (n + 7) / 8; }

blz::CMat view(const blz_cmat* m) {
  return blz::CMat{m->rows, m->cols, m->block_rows, m->block_cols, m->first, m->slope, m->scale, m->coeffs};
}

blz::LaunchCtx lc(blz_ctx* c) {
  blz::LaunchCtx L{};
  L.stream = c->stream;
  L.err = c->d_err;
  L.launches = &c->launches;
  L.sm_count = c->sm_count;
  L.exact_only = (c->mode & BLZ_MODE_EXACT) != 0;
  L.fast = c->fast_ok ? &c->fast : nullptr;
  L.wl_count = (unsigned long long*)c->d_wl;
  L.wl = c->d_wl ? c->d_wl + 32 : nullptr;
  L.stats = c->d_stats;
  L.basis_sym = c->basis_sym;
  L.basis_bound = c->basis_bound;
  return L;
}

// Grows the exact-path worklist to nb entries (grow-only; first large call only).
blz_status ensure_worklist(blz_ctx* c, uint64_t nb) {
  if (c->wl_cap >= nb && c->d_wl) return BLZ_OK;
  if (c->d_wl) {
    cudaStreamSynchronize(c->stream);
    cudaFree(c->d_wl);
    c->d_wl = nullptr;
    c->wl_cap = 0;
  }
  const uint64_t cap = nb < 1024 ? 1024 : nb;
  cudaError_t e = cudaMalloc(&c->d_wl, (cap + 32) * sizeof(uint64_t));
  if (e != cudaSuccess) return cuda_err(c, e, "worklist allocation");
  c->wl_cap = cap;
  return BLZ_OK;
}

// The verified compress path relies on the basis being the orthonormal DCT-II
// up to rounding: row abs sums <= sqrt(8)(1+1e-12) and the
// off-DC entries of sigma sigma' tiny.  sigma_0^2 is summed in long double.
void analyse_basis(blz_ctx* c) {
  long double sig[8];
  double rowabs = 0;
  for (int i = 0; i < 8; ++i) {
    long double acc = 0;
    double ra = 0;
    for (int u = 0; u < 8; ++u) {
      acc += (long double)c->basis.t[i * 8 + u];
      ra += std::fabs(c->basis.t[i * 8 + u]);
    }
    sig[i] = acc;
    rowabs = ra > rowabs ? ra : rowabs;
  }
  long double off = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j)
      if (i || j) {
        long double v = sig[i] * sig[j];
        if (v < 0) v = -v;
        off = v > off ? v : off;
      }
  c->fast.ss00 = (double)(sig[0] * sig[0]);
  {
    const long double pi = 3.141592653589793238462643383279502884L;
    c->fast.bfly[0] = (double)(1.0L / std::sqrt(8.0L));
    for (int k = 1; k < 8; ++k) c->fast.bfly[k] = (double)(0.5L * std::cos((long double)k * pi / 16.0L));
  }
  // the dropped lo*sigma_i*sigma_j terms are budgeted at 64 u |lo| in E_d
  c->fast_ok = rowabs <= 2.8284271247461903 * (1.0 + 1e-12) && off <= 64.0 * 1.1102230246251565e-16 &&
               std::fabs(c->fast.ss00 - 8.0) < 1e-12;
  // bitwise repeats the decompress kernel shares products over (blaz_device.cuh, BasisSym)
  const double* t = c->basis.t;
  bool sym = t[1 * 8 + 7] == -t[1 * 8 + 0] && t[2 * 8 + 3] == -t[2 * 8 + 0] && t[3 * 8 + 5] == -t[3 * 8 + 2] &&
             t[4 * 8 + 4] == -t[4 * 8 + 2];
  for (int k = 1; k < 8; ++k) sym = sym && t[k] == t[0];
  c->basis_sym = sym;
}

void* slot(blz_ctx* c, int id, size_t bytes, cudaError_t* e) {
  auto& s = c->slots[id];
  *e = cudaSuccess;
  if (bytes == 0) bytes = 16;
  if (s.bytes < bytes) {
    if (s.p) {
      cudaStreamSynchronize(c->stream);
      cudaFree(s.p);
      s.p = nullptr;
      s.bytes = 0;
    }
    *e = cudaMalloc(&s.p, bytes);
    if (*e != cudaSuccess) return nullptr;
    s.bytes = bytes;
  }
  return s.p;
}

// H/dct.hpp:14-26, the same expression with the host libm.
void reference_basis(double* t) {
  const double pi = std::acos(-1.0);
  for (int i = 0; i < 8; ++i) {
    const double ai = (i == 0) ? std::sqrt(1.0 / 8.0) : std::sqrt(1.0 / 4.0);
    for (int u = 0; u < 8; ++u) t[i * 8 + u] = ai * std::cos((2 * u + 1) * i * pi / 16.0);
  }
}

blz_status check_cmat(blz_ctx* c, const blz_cmat* m, const char* what) {
  if (!m) return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": null matrix");
  if (m->block_rows != nblk(m->rows) || m->block_cols != nblk(m->cols))
    return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": inconsistent block grid");
  const uint64_t nb = m->block_rows * m->block_cols;
  if (nb && (!m->first || !m->slope || !m->scale || !m->coeffs))
    return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": null buffer");
  return BLZ_OK;
}

// out must be disjoint from `in` or be the very same matrix (in-place use): the
// kernels read and write each block's record in place, never another block's.
blz_status check_alias(blz_ctx* c, const blz_cmat* out, const blz_cmat* in, const char* what) {
  const uint64_t nb = in->block_rows * in->block_cols;
  if (nb == 0) return BLZ_OK;
  const bool same = out->first == in->first && out->slope == in->slope && out->scale == in->scale &&
                    out->coeffs == in->coeffs;
  if (same) return BLZ_OK;
  auto ov = [](const void* p, uint64_t np, const void* q, uint64_t nq) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p), b = reinterpret_cast<uintptr_t>(q);
    return a < b + nq && b < a + np;
  };
  const void* po[4] = {out->first, out->slope, out->scale, out->coeffs};
  const void* pi[4] = {in->first, in->slope, in->scale, in->coeffs};
  const uint64_t sz[4] = {8 * nb, 8 * nb, nb, 28 * nb};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      if (ov(po[i], sz[i], pi[j], sz[j]))
        return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": output partially overlaps an input");
  return BLZ_OK;
}

// H/matrix.hpp:86-93
blz_status same_dims(blz_ctx* c, uint64_t ar, uint64_t ac, uint64_t br, uint64_t bc, const char* what) {
  if (ar != br || ac != bc)
    return set_err(c, BLZ_INVALID_ARGUMENT,
                   std::string(what) + ": dimension mismatch (" + std::to_string(ar) + "x" +
                       std::to_string(ac) + " vs " + std::to_string(br) + "x" + std::to_string(bc) + ")");
  return BLZ_OK;
}

blz_status latch_status(blz_ctx* c) {
  unsigned long long v = ~0ull;
  BLZ_CUDA(c, cudaMemcpyAsync(&v, c->d_err, sizeof v, cudaMemcpyDeviceToHost, c->stream), "error latch");
  BLZ_CUDA(c, cudaStreamSynchronize(c->stream), "sync");
  if (v == ~0ull) return BLZ_OK;
  const unsigned long long reset = ~0ull;
  BLZ_CUDA(c, cudaMemcpyAsync(c->d_err, &reset, sizeof reset, cudaMemcpyHostToDevice, c->stream), "error latch reset");
  BLZ_CUDA(c, cudaStreamSynchronize(c->stream), "sync");
  switch ((uint32_t)(v & 0xff)) {
    case blz::DERR_NONFINITE_CODE:
      return set_err(c, BLZ_INVALID_ARGUMENT, "normalize: non-finite input");
    case blz::DERR_PREDICT_CODE:
      return set_err(c, BLZ_INVALID_ARGUMENT, "predict: mean slope must be positive");
    case blz::DERR_DOT_RANGE_CODE:
      return set_err(c, BLZ_OUT_OF_RANGE, "mat_dot: index out of range");
    case blz::DERR_IO_NONFINITE_CODE:
      return set_err(c, BLZ_IO_ERROR, "write_compressed: non-finite block field");
    case blz::DERR_IO_ZERO_PHI_CODE:
      return set_err(c, BLZ_IO_ERROR, "compressed matrix: zero scale factor in block " + std::to_string(v >> 8));
    default:
      return set_err(c, BLZ_CUDA_ERROR, "unknown device error");
  }
}

// Host-level helpers: a device SoA matrix laid over a scratch slot.
blz_status scratch_cmat(blz_ctx* c, int id, uint64_t rows, uint64_t cols, blz_cmat* m) {
  cudaError_t e;
  void* p = slot(c, id, blz_cmat_bytes(rows, cols), &e);
  if (!p) return cuda_err(c, e, "scratch allocation");
  return blz_cmat_view(rows, cols, p, m);
}

blz_status upload_blocks(blz_ctx* c, const blz_block* h, uint64_t rows, uint64_t cols, int id, blz_cmat* m) {
  blz_status st = scratch_cmat(c, id, rows, cols, m);
  if (st) return st;
  const uint64_t nb = m->block_rows * m->block_cols;
  cudaError_t e;
  void* aos = slot(c, S_AUX, nb * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  BLZ_CUDA(c, cudaMemcpyAsync(aos, h, nb * sizeof(blz_block), cudaMemcpyHostToDevice, c->stream), "H2D blocks");
  return blz_unpack_aos_dev(c, (const blz_block*)aos, m);
}

// One block-column (block index bj of a matrix with nbc block columns) as a
// rows x ncols matrix (ncols <= 8): a strided host read of one record per block-row.
blz_status upload_block_col(blz_ctx* c, const blz_block* h, uint64_t rows, uint64_t nbc, uint64_t bj,
                            uint64_t ncols, int id, blz_cmat* m) {
  blz_status st = scratch_cmat(c, id, rows, ncols, m);
  if (st) return st;
  const uint64_t nb = m->block_rows;
  cudaError_t e;
  void* aos = slot(c, S_AUX, nb * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  BLZ_CUDA(c, cudaMemcpy2DAsync(aos, sizeof(blz_block), h + bj, nbc * sizeof(blz_block), sizeof(blz_block), nb,
                                cudaMemcpyHostToDevice, c->stream), "H2D blocks");
  return blz_unpack_aos_dev(c, (const blz_block*)aos, m);
}

blz_status download_blocks(blz_ctx* c, const blz_cmat* m, blz_block* h) {
  const uint64_t nb = m->block_rows * m->block_cols;
  cudaError_t e;
  void* aos = slot(c, S_AUX, nb * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  blz_status st = blz_pack_aos_dev(c, m, (blz_block*)aos);
  if (st) return st;
  BLZ_CUDA(c, cudaMemcpyAsync(h, aos, nb * sizeof(blz_block), cudaMemcpyDeviceToHost, c->stream), "D2H blocks");
  return BLZ_OK;
}

}  // namespace

extern "C" {

int blz_abi_version(void) { return BLZ_ABI_VERSION; }

blz_status blz_ctx_create(int device, const double* basis, blz_ctx** out) {
  if (!out) return BLZ_INVALID_ARGUMENT;
  *out = nullptr;
  blz_ctx* c = new (std::nothrow) blz_ctx;
  if (!c) return BLZ_OUT_OF_MEMORY;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_err, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0xff, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_stats, 4 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->d_stats, 0, 4 * sizeof(unsigned long long));
  // a private non-blocking stream: contexts of different host threads (the drop-in
  // creates one per thread) never serialise on the legacy default stream
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) c->stream = c->own_stream;
  if (e != cudaSuccess) {
    delete c;
    return e == cudaErrorMemoryAllocation ? BLZ_OUT_OF_MEMORY : BLZ_CUDA_ERROR;
  }
  if (basis)
    std::memcpy(c->basis.t, basis, sizeof c->basis.t);
  else
    reference_basis(c->basis.t);
  analyse_basis(c);
  if (blz::bind_decompress_basis(c->basis, &c->basis_bound) != cudaSuccess) {
    blz_ctx_destroy(c);
    return BLZ_CUDA_ERROR;
  }
  *out = c;
  return BLZ_OK;
}

void blz_ctx_destroy(blz_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& s : c->slots)
    if (s.p) cudaFree(s.p);
  if (c->d_err) cudaFree(c->d_err);
  if (c->d_stats) cudaFree(c->d_stats);
  if (c->d_wl) cudaFree(c->d_wl);
  if (c->own_stream) {
    cudaStreamSynchronize(c->own_stream);
    cudaStreamDestroy(c->own_stream);
  }
  for (auto* g : {c->st_in, c->st_out})
    for (int k = 0; k < 2; ++k) {
      if (g[k].p) cudaFreeHost(g[k].p);
      if (g[k].ev) cudaEventDestroy(g[k].ev);
    }
  if (c->s_in) cudaStreamDestroy(c->s_in);
  if (c->s_out) cudaStreamDestroy(c->s_out);
  for (auto ev : c->events) cudaEventDestroy(ev);
  delete c;
}

blz_status blz_ctx_set_stream(blz_ctx* c, void* stream) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  c->stream = (cudaStream_t)stream;
  return BLZ_OK;
}

void* blz_ctx_get_stream(const blz_ctx* c) { return c ? (void*)c->stream : nullptr; }

const char* blz_last_error(const blz_ctx* c) { return c ? c->err.c_str() : "null context"; }

// for the other translation units of the library (sharded.cu); not exported
__attribute__((visibility("hidden"))) blz_status blz_internal_set_error(blz_ctx* c, blz_status st, const char* msg) {
  return set_err(c, st, msg);
}

blz_status blz_ctx_sync(blz_ctx* c) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  return latch_status(c);
}

blz_status blz_ctx_basis(const blz_ctx* c, double* out) {
  if (!c || !out) return BLZ_INVALID_ARGUMENT;
  std::memcpy(out, c->basis.t, sizeof c->basis.t);
  return BLZ_OK;
}

uint64_t blz_ctx_launches(const blz_ctx* c) { return c ? c->launches : 0; }

blz_status blz_ctx_set_mode(blz_ctx* c, int mode) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (mode & ~(BLZ_MODE_EXACT)) return set_err(c, BLZ_INVALID_ARGUMENT, "blz_ctx_set_mode: unknown mode bits");
  c->mode = mode;
  return BLZ_OK;
}

int blz_ctx_get_mode(const blz_ctx* c) { return c ? c->mode : -1; }

int blz_ctx_fast_path_available(const blz_ctx* c) { return c && c->fast_ok ? 1 : 0; }

blz_status blz_ctx_stats(blz_ctx* c, uint64_t* compress_exact_blocks, uint64_t* addsub_fallback_blocks) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  unsigned long long h[4] = {0, 0, 0, 0};
  BLZ_CUDA(c, cudaMemcpyAsync(h, c->d_stats, sizeof h, cudaMemcpyDeviceToHost, c->stream), "stats");
  BLZ_CUDA(c, cudaStreamSynchronize(c->stream), "stats sync");
  if (compress_exact_blocks) *compress_exact_blocks = h[0];
  if (addsub_fallback_blocks) *addsub_fallback_blocks = h[1];
  return BLZ_OK;
}

// ---- SoA matrices ----------------------------------------------------------
static uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }

uint64_t blz_cmat_bytes(uint64_t rows, uint64_t cols) {
  const uint64_t nb = nblk(rows) * nblk(cols);
  return align256(nb * 8) * 2 + align256(nb * 28) + align256(nb);
}

blz_status blz_cmat_view(uint64_t rows, uint64_t cols, void* mem, blz_cmat* m) {
  if (!m) return BLZ_INVALID_ARGUMENT;
  const uint64_t nb = nblk(rows) * nblk(cols);
  char* p = (char*)mem;
  m->rows = rows;
  m->cols = cols;
  m->block_rows = nblk(rows);
  m->block_cols = nblk(cols);
  m->first = (double*)p;
  p += align256(nb * 8);
  m->slope = (double*)p;
  p += align256(nb * 8);
  m->coeffs = (int8_t*)p;
  p += align256(nb * 28);
  m->scale = (uint8_t*)p;
  return BLZ_OK;
}

blz_status blz_cmat_alloc(blz_ctx* c, uint64_t rows, uint64_t cols, blz_cmat* m) {
  if (!c || !m) return BLZ_INVALID_ARGUMENT;
  void* p = nullptr;
  BLZ_CUDA(c, cudaMalloc(&p, blz_cmat_bytes(rows, cols)), "blz_cmat_alloc");
  return blz_cmat_view(rows, cols, p, m);
}

void blz_cmat_free(blz_ctx* c, blz_cmat* m) {
  (void)c;
  if (m && m->first) cudaFree(m->first);
  if (m) m->first = nullptr;
}

// ---- device-level operations -------------------------------------------------
blz_status blz_compress_dev(blz_ctx* c, const double* dense, uint64_t rows, uint64_t cols, uint64_t ld,
                            const blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (rows == 0 || cols == 0) return set_err(c, BLZ_INVALID_ARGUMENT, "compress_matrix: empty matrix");  // H/matrix.hpp:98
  if (blz_status st = check_cmat(c, out, "compress_matrix")) return st;
  if (out->rows != rows || out->cols != cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "compress_matrix: output dimension mismatch");
  if (ld < cols) return set_err(c, BLZ_INVALID_ARGUMENT, "compress_matrix: ld < cols");
  if (blz_status st = ensure_worklist(c, out->block_rows * out->block_cols)) return st;
  return cuda_err(c, blz::launch_compress(lc(c), c->basis, dense, rows, cols, ld, view(out)), "compress");
}

blz_status blz_decompress_dev(blz_ctx* c, const blz_cmat* in, double* dense, uint64_t ld) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, in, "decompress_matrix")) return st;
  if (ld < in->cols) return set_err(c, BLZ_INVALID_ARGUMENT, "decompress_matrix: ld < cols");
  if (in->block_rows * in->block_cols == 0) return BLZ_OK;
  return cuda_err(c, blz::launch_decompress(lc(c), c->basis, view(in), dense, ld, in->rows, in->cols),
                  "decompress");
}

static blz_status addsub_dev(blz_ctx* c, bool sub, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out) {
  const char* what = sub ? "mat_sub" : "mat_add";
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, what)) return st;
  if (blz_status st = check_cmat(c, b, what)) return st;
  if (blz_status st = check_cmat(c, out, what)) return st;
  if (blz_status st = same_dims(c, a->rows, a->cols, b->rows, b->cols, what)) return st;  // H/matrix.hpp:130
  if (out->rows != a->rows || out->cols != a->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": output dimension mismatch");
  if (blz_status st = check_alias(c, out, a, what)) return st;
  if (blz_status st = check_alias(c, out, b, what)) return st;
  const uint64_t nb = a->block_rows * a->block_cols;
  if (nb == 0) return BLZ_OK;
  if (blz_status st = ensure_worklist(c, nb)) return st;
  return cuda_err(c, blz::launch_addsub(lc(c), c->basis, sub, view(a), view(b), view(out)), what);
}

blz_status blz_add_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out) {
  return addsub_dev(c, false, a, b, out);
}
blz_status blz_sub_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out) {
  return addsub_dev(c, true, a, b, out);
}

blz_status blz_scale_dev(blz_ctx* c, const blz_cmat* a, double k, const blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_scale")) return st;
  if (blz_status st = check_cmat(c, out, "mat_scale")) return st;
  if (out->rows != a->rows || out->cols != a->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_scale: output dimension mismatch");
  const uint64_t nb = a->block_rows * a->block_cols;
  if (nb == 0) return BLZ_OK;  // the reference never calls scale() on an empty grid
  if (!std::isfinite(k)) return set_err(c, BLZ_INVALID_ARGUMENT, "scale: non-finite constant");  // H/block_ops.hpp:75
  return cuda_err(c, blz::launch_scale(lc(c), view(a), k, view(out)), "mat_scale");
}

blz_status blz_scale_meta_dev(blz_ctx* c, const blz_cmat* a, double k, blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_scale")) return st;
  if (!out) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_scale: null matrix");
  if (out->rows != a->rows || out->cols != a->cols || out->block_rows != a->block_rows ||
      out->block_cols != a->block_cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_scale: output dimension mismatch");
  const uint64_t nb = a->block_rows * a->block_cols;
  if (nb && (!out->first || !out->slope)) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_scale: null buffer");
  if (nb == 0) return BLZ_OK;
  if (!std::isfinite(k)) return set_err(c, BLZ_INVALID_ARGUMENT, "scale: non-finite constant");  // H/block_ops.hpp:75
  out->scale = a->scale;
  out->coeffs = a->coeffs;
  return cuda_err(c, blz::launch_scale_fs(lc(c), a->first, a->slope, k, out->first, out->slope, nb), "mat_scale");
}

// ---- device-batched block-level API (H/block_ops.hpp:87-142) ----------------
static blz_status reconstruct_dev(blz_ctx* c, bool cols, const blz_cmat* in, int last, double* tiles) {
  const char* what = cols ? "reconstruct_cols" : "reconstruct_rows";
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, in, what)) return st;
  if (last < 0 || last >= 8)  // H/block_ops.hpp:88-89, :101-102
    return set_err(c, BLZ_OUT_OF_RANGE,
                   std::string(what) + (cols ? ": column index out of range" : ": row index out of range"));
  const uint64_t nb = in->block_rows * in->block_cols;
  if (nb == 0) return BLZ_OK;
  if (!tiles) return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": null output");
  return cuda_err(c, blz::launch_reconstruct(lc(c), c->basis, cols, view(in), last, tiles), what);
}

blz_status blz_reconstruct_rows_dev(blz_ctx* c, const blz_cmat* in, int last_row, double* tiles) {
  return reconstruct_dev(c, false, in, last_row, tiles);
}
blz_status blz_reconstruct_cols_dev(blz_ctx* c, const blz_cmat* in, int last_col, double* tiles) {
  return reconstruct_dev(c, true, in, last_col, tiles);
}

blz_status blz_block_mul_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, double* tiles) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "block_mul")) return st;
  if (blz_status st = check_cmat(c, b, "block_mul")) return st;
  if (a->block_rows != b->block_rows || a->block_cols != b->block_cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "block_mul: block grids differ");
  const uint64_t nb = a->block_rows * a->block_cols;
  if (nb == 0) return BLZ_OK;
  if (!tiles) return set_err(c, BLZ_INVALID_ARGUMENT, "block_mul: null output");
  return cuda_err(c, blz::launch_block_mul(lc(c), c->basis, view(a), view(b), tiles), "block_mul");
}

// Fused op + decompress: out receives the compressed result
// (as blz_add_dev / blz_sub_dev / blz_scale_dev) and dense its decompression
// (as blz_decompress_dev), bitwise equal to the two-call chain.
static blz_status op_decompress_dev(blz_ctx* c, int op, const blz_cmat* a, const blz_cmat* b, double k,
                                    const blz_cmat* out, double* dense, uint64_t ld) {
  const char* what = op == 0 ? "mat_add" : (op == 1 ? "mat_sub" : "mat_scale");
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, what)) return st;
  if (op != 2) {
    if (blz_status st = check_cmat(c, b, what)) return st;
    if (blz_status st = same_dims(c, a->rows, a->cols, b->rows, b->cols, what)) return st;  // H/matrix.hpp:130
  }
  if (blz_status st = check_cmat(c, out, what)) return st;
  if (out->rows != a->rows || out->cols != a->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": output dimension mismatch");
  if (ld < a->cols) return set_err(c, BLZ_INVALID_ARGUMENT, "decompress_matrix: ld < cols");
  const uint64_t nb = a->block_rows * a->block_cols;
  if (nb == 0) return BLZ_OK;
  if (op == 2 && !std::isfinite(k)) return set_err(c, BLZ_INVALID_ARGUMENT, "scale: non-finite constant");
  // the two launches (op, then the decompress kernel) are faster than the fused kernel
  // since the round-2 add/sub kernels and k_decompress_ub (16384^2: add 0.105 + 0.442
  // against 0.628 ms, scale 0.067 + 0.442 against 0.533 ms), with the same bits; the
  // fused kernel remains for views whose arrays are not 16-byte aligned
  {
    const blz::CMat va = view(a), vb = op == 2 ? va : view(b), vo = view(out);
    uintptr_t bits = 0;
    for (const blz::CMat* m : {&va, &vb, &vo})
      bits |= reinterpret_cast<uintptr_t>(m->first) | reinterpret_cast<uintptr_t>(m->slope) |
              reinterpret_cast<uintptr_t>(m->scale) | reinterpret_cast<uintptr_t>(m->coeffs);
    if ((bits & 15) == 0) {
      blz_status st = op == 0 ? blz_add_dev(c, a, b, out) : op == 1 ? blz_sub_dev(c, a, b, out) : blz_scale_dev(c, a, k, out);
      if (st) return st;
      return blz_decompress_dev(c, out, dense, ld);
    }
  }
  if (op != 2)
    if (blz_status st = ensure_worklist(c, nb)) return st;
  const blz::CMat va = view(a);
  return cuda_err(c, blz::launch_op_decompress(lc(c), c->basis, op, va, op == 2 ? va : view(b), k, view(out), dense,
                                               ld, a->rows, a->cols),
                  what);
}

blz_status blz_add_decompress_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out,
                                  double* dense, uint64_t ld) {
  return op_decompress_dev(c, 0, a, b, 0.0, out, dense, ld);
}
blz_status blz_sub_decompress_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out,
                                  double* dense, uint64_t ld) {
  return op_decompress_dev(c, 1, a, b, 0.0, out, dense, ld);
}
blz_status blz_scale_decompress_dev(blz_ctx* c, const blz_cmat* a, double k, const blz_cmat* out, double* dense,
                                    uint64_t ld) {
  return op_decompress_dev(c, 2, a, nullptr, k, out, dense, ld);
}

blz_status blz_dot_entries_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, const uint64_t* i,
                               const uint64_t* j, uint64_t n, double* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_dot")) return st;
  if (blz_status st = check_cmat(c, b, "mat_dot")) return st;
  if (a->cols != b->rows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_dot: inner dimension mismatch");  // :159
  double* prod = nullptr;  // few queries: products spread over threads (context scratch)
  if (n && n <= blz::kDotSplitMaxQueries && a->block_cols >= 32) {
    cudaError_t e;
    prod = (double*)slot(c, S_DOT, n * a->block_cols * 8 * sizeof(double), &e);
    if (!prod) return cuda_err(c, e, "scratch allocation");
  }
  return cuda_err(c, blz::launch_dot_entries(lc(c), c->basis, view(a), view(b), i, j, n, out, 0, a->rows, prod),
                  "mat_dot");
}

blz_status blz_dot_entries_rows_dev(blz_ctx* c, const blz_cmat* a_rows, const blz_cmat* b, const uint64_t* i,
                                    const uint64_t* j, uint64_t n, uint64_t row0, uint64_t rows_total,
                                    double* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a_rows, "mat_dot")) return st;
  if (blz_status st = check_cmat(c, b, "mat_dot")) return st;
  if (a_rows->cols != b->rows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_dot: inner dimension mismatch");
  if (row0 % 8 != 0 || row0 > rows_total || a_rows->rows > rows_total - row0)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_dot: row shard outside the matrix");
  return cuda_err(c, blz::launch_dot_entries(lc(c), c->basis, view(a_rows), view(b), i, j, n, out, row0, rows_total),
                  "mat_dot");
}

blz_status blz_rowdot_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, double* r) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_rowdot")) return st;
  if (blz_status st = check_cmat(c, b, "mat_rowdot")) return st;
  if (blz_status st = same_dims(c, a->rows, a->cols, b->rows, b->cols, "mat_rowdot")) return st;
  if (a->block_rows * a->block_cols == 0) return BLZ_OK;
  cudaError_t e;
  void* scratch = slot(c, S_ROWDOT, blz::rowdot_scratch_bytes(view(a)), &e);  // grow-only context scratch
  if (!scratch) return cuda_err(c, e, "scratch allocation");
  return cuda_err(c, blz::launch_rowdot(lc(c), c->basis, view(a), view(b), r, scratch), "mat_rowdot");
}

// Row dots and their ascending total in one pass (the total follows the groups
// as they finish inside the split kernel; bitwise blz_rowdot_dev + blz_sum_dev).
blz_status blz_rowdot_frobenius_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, double* r, double* total) {
  if (!c || !total) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_rowdot")) return st;
  if (blz_status st = check_cmat(c, b, "mat_rowdot")) return st;
  if (blz_status st = same_dims(c, a->rows, a->cols, b->rows, b->cols, "mat_rowdot")) return st;
  if (a->block_rows * a->block_cols == 0) return blz_sum_dev(c, r, 0, total);
  cudaError_t e;
  void* scratch = slot(c, S_ROWDOT, blz::rowdot_scratch_bytes(view(a)), &e);
  if (!scratch) return cuda_err(c, e, "scratch allocation");
  return cuda_err(c, blz::launch_rowdot(lc(c), c->basis, view(a), view(b), r, scratch, total), "mat_rowdot");
}

blz_status blz_sum_dev(blz_ctx* c, const double* v, uint64_t n, double* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  return cuda_err(c, blz::launch_sum(lc(c), v, n, out), "sum");
}

uint64_t blz_matmul_scratch_bytes(const blz_cmat* a, const blz_cmat* b) {
  if (!a || !b) return 0;
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, kb = 8 * b->block_rows, nb = 8 * b->block_cols;
  return (ma * ka + kb * nb + ma * nb) * sizeof(double) + 256;
}

static blz_status matmul_common(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode, void* scratch,
                                double** dc) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_mul")) return st;
  if (blz_status st = check_cmat(c, b, "mat_mul")) return st;
  if (a->cols != b->rows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: inner dimension mismatch");  // :207
  if (mode < BLZ_GEMM_EXACT || mode > BLZ_GEMM_FUSED_DFMA) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: bad mode");
  if (!scratch) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: null scratch");
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, kb = 8 * b->block_rows, nn = 8 * b->block_cols;
  double* da = (double*)scratch;
  double* db = da + ma * ka;
  *dc = db + kb * nn;
  // decompress_tiles (H/matrix.hpp:178-183): full 8x8 tiles, padding included
  auto L = lc(c);
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(a), da, ka, ma, ka), "mat_mul decompress A");
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(b), db, nn, kb, nn), "mat_mul decompress B");
  BLZ_CUDA(c, blz::launch_gemm(L, mode, da, ka, db, nn, *dc, nn, ma, nn, a->cols), "mat_mul gemm");
  return BLZ_OK;
}

blz_status blz_matmul_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode, void* scratch,
                          const blz_cmat* out) {
  double* dc = nullptr;
  if (blz_status st = matmul_common(c, a, b, mode, scratch, &dc)) return st;
  if (blz_status st = check_cmat(c, out, "mat_mul")) return st;
  if (out->rows != a->rows || out->cols != b->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: output dimension mismatch");
  // each full accumulator tile compressed once (H/matrix.hpp:231-233)
  const uint64_t ma = 8 * a->block_rows, nn = 8 * b->block_cols;
  if (blz_status st = ensure_worklist(c, a->block_rows * b->block_cols)) return st;
  return cuda_err(c, blz::launch_compress(lc(c), c->basis, dc, ma, nn, nn, view(out)), "mat_mul compress");
}

// ---- fused all-gather + decompress over block-row shards (peer memory) --------
// shards[r] holds block-rows [lo_r, lo_r + shards[r].block_rows) of one matrix, in
// order; all but the last hold whole block-rows (rows a multiple of 8).
static blz_status shard_set(blz_ctx* c, const blz_cmat* shards, int n, blz::ShardSet* S, uint64_t* rows,
                            uint64_t* cols, const char* what) {
  if (!shards || n < 1 || n > blz::ShardSet::kMax)
    return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": 1 to 16 shards");
  S->n = n;
  S->lo[0] = 0;
  *rows = 0;
  *cols = shards[0].cols;
  for (int r = 0; r < n; ++r) {
    const blz_cmat& m = shards[r];
    if (m.block_rows) {
      if (blz_status st = check_cmat(c, &m, what)) return st;
    }
    if (m.cols != *cols || (r + 1 < n && m.rows % 8 != 0))
      return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": shards do not tile the block-rows");
    S->part[r] = view(&m);
    S->lo[r + 1] = S->lo[r] + m.block_rows;
    *rows += m.rows;
  }
  if (*rows == 0) return set_err(c, BLZ_INVALID_ARGUMENT, std::string(what) + ": empty matrix");
  return BLZ_OK;
}

blz_status blz_decompress_gather_dev(blz_ctx* c, const blz_cmat* shards, int nshards, double* dense, uint64_t ld) {
  if (!c || !dense) return BLZ_INVALID_ARGUMENT;
  blz::ShardSet S;
  uint64_t rows = 0, cols = 0;
  if (blz_status st = shard_set(c, shards, nshards, &S, &rows, &cols, "decompress_gather")) return st;
  if (ld < cols) return set_err(c, BLZ_INVALID_ARGUMENT, "decompress_gather: ld < cols");
  return cuda_err(c, blz::launch_decompress_gather(lc(c), c->basis, S, (cols + 7) / 8, dense, ld, rows, cols),
                  "decompress_gather");
}

blz_status blz_matmul_gather_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b_shards, int nshards, int mode,
                                 void* scratch, const blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  blz::ShardSet S;
  uint64_t brows = 0, bcols = 0;
  if (blz_status st = shard_set(c, b_shards, nshards, &S, &brows, &bcols, "mat_mul")) return st;
  if (blz_status st = check_cmat(c, a, "mat_mul")) return st;
  if (blz_status st = check_cmat(c, out, "mat_mul")) return st;
  if (a->cols != brows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: inner dimension mismatch");  // :207
  if (out->rows != a->rows || out->cols != bcols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: output dimension mismatch");
  if (mode < BLZ_GEMM_EXACT || mode > BLZ_GEMM_FUSED_DFMA) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: bad mode");
  if (!scratch) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: null scratch");
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, kb = 8 * S.lo[S.n], nn = 8 * ((bcols + 7) / 8);
  double* da = (double*)scratch;
  double* db = da + ma * ka;
  double* dc = db + kb * nn;
  auto L = lc(c);
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(a), da, ka, ma, ka), "mat_mul decompress A");
  // B straight from the shards (the ranks' arrays): no gathered compressed copy
  BLZ_CUDA(c, blz::launch_decompress_gather(L, c->basis, S, nn / 8, db, nn, kb, nn), "mat_mul decompress B");
  BLZ_CUDA(c, blz::launch_gemm(L, mode, da, ka, db, nn, dc, nn, ma, nn, a->cols), "mat_mul gemm");
  if (blz_status st = ensure_worklist(c, a->block_rows * (nn / 8))) return st;
  return cuda_err(c, blz::launch_compress(lc(c), c->basis, dc, ma, nn, nn, view(out)), "mat_mul compress");
}

blz_status blz_matmul_dense_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode, void* scratch,
                                double* out, uint64_t ld) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_mul")) return st;
  if (blz_status st = check_cmat(c, b, "mat_mul")) return st;
  if (a->cols != b->rows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: inner dimension mismatch");
  if (ld < b->cols) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul_dense: ld < cols");
  if (mode < BLZ_GEMM_EXACT || mode > BLZ_GEMM_FUSED_DFMA) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: bad mode");
  if (!scratch) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: null scratch");
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, kb = 8 * b->block_rows, nn = 8 * b->block_cols;
  double* da = (double*)scratch;
  double* db = da + ma * ka;
  auto L = lc(c);
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(a), da, ka, ma, ka), "mat_mul decompress A");
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(b), db, nn, kb, nn), "mat_mul decompress B");
  // crop (H/matrix.hpp:242-248): entries outside a.rows x b.cols are never formed
  BLZ_CUDA(c, blz::launch_gemm(L, mode, da, ka, db, nn, out, ld, a->rows, b->cols, a->cols), "mat_mul gemm");
  return BLZ_OK;
}

// ---- K-paneled compressed GEMM (decompression fed to the GEMM
// panel by panel, for HBM capacity) -------------------------------------------
// B is decompressed P block-rows at a time (a contiguous block-row range of its
// SoA arrays) and each panel's product is accumulated into C, the accumulators
// continuing from the previous panels' values: per output entry the operation
// sequence is exactly the single-pass one (H/matrix.hpp:188-202), so results are
// bitwise those of blz_matmul_dev.  Scratch: dense A + one B panel + dense C
// instead of dense A + dense B + dense C (8 GiB instead of 15 GiB per rank for
// config 4 on 8 GPUs, with 1/8 panels).
uint64_t blz_matmul_panel_scratch_bytes(const blz_cmat* a, const blz_cmat* b, uint64_t panel_block_rows) {
  if (!a || !b || panel_block_rows == 0) return 0;
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, nn = 8 * b->block_cols;
  const uint64_t pr = std::min<uint64_t>(panel_block_rows, b->block_rows);
  return (ma * ka + 8 * pr * nn + ma * nn) * sizeof(double) + 256;
}

}  // extern "C"
namespace {
blz_cmat sub_rows(const blz_cmat& m, uint64_t b0, uint64_t b1);
}
extern "C" {

static blz_status matmul_panel_common(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode,
                                      uint64_t panel_block_rows, void* scratch, double* dc, uint64_t ldc,
                                      uint64_t crop_m, uint64_t crop_n) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, a, "mat_mul")) return st;
  if (blz_status st = check_cmat(c, b, "mat_mul")) return st;
  if (a->cols != b->rows) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: inner dimension mismatch");  // :207
  if (mode < BLZ_GEMM_EXACT || mode > BLZ_GEMM_FUSED_DFMA) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: bad mode");
  if (!scratch) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: null scratch");
  if (panel_block_rows == 0 || panel_block_rows % 4)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: panel_block_rows must be a positive multiple of 4");
  const uint64_t ma = 8 * a->block_rows, ka = 8 * a->block_cols, nn = 8 * b->block_cols;
  double* da = (double*)scratch;
  double* db = da + ma * ka;
  if (!dc) dc = db + 8 * std::min<uint64_t>(panel_block_rows, b->block_rows) * nn;
  auto L = lc(c);
  BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(a), da, ka, ma, ka), "mat_mul decompress A");
  for (uint64_t p0 = 0; p0 < b->block_rows; p0 += panel_block_rows) {
    const uint64_t p1 = std::min(b->block_rows, p0 + panel_block_rows);
    const uint64_t k0 = 8 * p0, k1 = std::min<uint64_t>(8 * p1, a->cols);
    if (k1 <= k0) break;
    const blz_cmat bp = sub_rows(*b, p0, p1);
    BLZ_CUDA(c, blz::launch_decompress(L, c->basis, view(&bp), db, nn, 8 * (p1 - p0), nn), "mat_mul decompress B");
    BLZ_CUDA(c, blz::launch_gemm(L, mode, da + k0, ka, db, nn, dc, ldc, crop_m, crop_n, k1 - k0, p0 > 0),
             "mat_mul gemm");
  }
  return BLZ_OK;
}

blz_status blz_matmul_panel_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode, uint64_t panel_block_rows,
                                void* scratch, const blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, out, "mat_mul")) return st;
  if (out->rows != a->rows || out->cols != b->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: output dimension mismatch");
  const uint64_t ma = 8 * a->block_rows, nn = 8 * b->block_cols;
  double* dc = (double*)scratch + ma * 8 * a->block_cols +
               8 * std::min<uint64_t>(panel_block_rows ? panel_block_rows : 1, b->block_rows) * nn;
  // full accumulator tiles (padding included), each compressed once (H/matrix.hpp:231-233)
  if (blz_status st = matmul_panel_common(c, a, b, mode, panel_block_rows, scratch, dc, nn, ma, nn)) return st;
  if (blz_status st = ensure_worklist(c, a->block_rows * b->block_cols)) return st;
  return cuda_err(c, blz::launch_compress(lc(c), c->basis, dc, ma, nn, nn, view(out)), "mat_mul compress");
}

blz_status blz_matmul_dense_panel_dev(blz_ctx* c, const blz_cmat* a, const blz_cmat* b, int mode,
                                      uint64_t panel_block_rows, void* scratch, double* out, uint64_t ld) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (a && b && ld < b->cols) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul_dense: ld < cols");
  // crop (H/matrix.hpp:242-248): the panels accumulate straight into the caller's a.rows x b.cols
  return matmul_panel_common(c, a, b, mode, panel_block_rows, scratch, out, ld, a ? a->rows : 0, b ? b->cols : 0);
}

blz_status blz_pack_aos_dev(blz_ctx* c, const blz_cmat* in, blz_block* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, in, "pack")) return st;
  if (in->block_rows * in->block_cols == 0) return BLZ_OK;
  return cuda_err(c, blz::launch_pack_aos(lc(c), view(in), out), "pack_aos");
}

blz_status blz_unpack_aos_dev(blz_ctx* c, const blz_block* in, const blz_cmat* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, out, "unpack")) return st;
  if (out->block_rows * out->block_cols == 0) return BLZ_OK;
  return cuda_err(c, blz::launch_unpack_aos(lc(c), in, view(out)), "unpack_aos");
}

// ---- host-level drop-in entry points ------------------------------------------
// The big host-level calls are pipelined over block-row chunks: the upload of
// chunk i+1 (copy-in stream), the kernels of chunk i (context stream) and the
// download of chunk i-1 (copy-out stream) overlap, so a call costs about its
// larger PCIe direction instead of the sum of both plus the kernels.  Chunks
// start at multiples of 16 block-rows, which keeps every SoA sub-view 16-byte
// aligned for the vectorized kernels.

}  // extern "C"

namespace {

blz_cmat sub_rows(const blz_cmat& m, uint64_t b0, uint64_t b1) {
  blz_cmat v = m;
  const uint64_t off = b0 * m.block_cols;
  v.rows = std::min(m.rows, 8 * b1) - 8 * b0;
  v.block_rows = b1 - b0;
  v.first = m.first + off;
  v.slope = m.slope + off;
  v.coeffs = m.coeffs + 28 * off;
  v.scale = m.scale + off;
  return v;
}

blz_status ensure_pipe(blz_ctx* c, size_t nev) {
  if (!c->s_in) BLZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking), "stream");
  if (!c->s_out) BLZ_CUDA(c, cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking), "stream");
  while (c->events.size() < nev) {
    cudaEvent_t ev;
    BLZ_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    c->events.push_back(ev);
  }
  return BLZ_OK;
}

// ---- pageable host buffers ------------------------------------------------------
// cudaMemcpyAsync from / to pageable memory is staged by the driver at a fraction
// of the PCIe rate.  The host entry points stage pageable buffers themselves:
// a page-locked slot per chunk and direction (two slots, alternating), filled /
// emptied by a pool of host threads (parallel memcpy) while the copy engine
// moves the neighbouring chunk.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  // memcpy(dst, src, n) split over the pool and the calling thread
  void copy(void* dst, const void* src, size_t n) {
    // 4 MB pieces (1 / 2 MB: faster for 12 MB record chunks, slower for small
    // calls -- waking the pool costs more than it saves there)
    const size_t piece_min = size_t(4) << 20;
    const int parts = (int)std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, n / piece_min));
    if (parts <= 1) {
      std::memcpy(dst, src, n);
      return;
    }
    Batch b;
    b.left = parts - 1;
    const size_t per = (n + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int k = 1; k < parts; ++k) {
        const size_t o = k * per, m = std::min(per, n - o);
        jobs_.push_back({(char*)dst + o, (const char*)src + o, m, &b});
      }
    }
    cv_.notify_all();
    std::memcpy(dst, src, std::min(per, n));
    std::unique_lock<std::mutex> lk(b.mu);
    b.cv.wait(lk, [&] { return b.left == 0; });
  }

 private:
  struct Batch {
    std::mutex mu;
    std::condition_variable cv;
    int left = 0;
  };
  struct Job {
    char* d;
    const char* s;
    size_t n;
    Batch* b;
  };
  CopyPool() {
    cpu_set_t set;
    int n = (int)std::thread::hardware_concurrency();
    if (sched_getaffinity(0, sizeof set, &set) == 0) n = CPU_COUNT(&set);
    n = std::max(1, std::min(n, 16)) - 1;
    for (int k = 0; k < n; ++k) workers_.emplace_back([this] { run(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (stop_ && jobs_.empty()) return;
        j = jobs_.front();
        jobs_.pop_front();
      }
      std::memcpy(j.d, j.s, j.n);
      std::lock_guard<std::mutex> lk(j.b->mu);
      if (--j.b->left == 0) j.b->cv.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::deque<Job> jobs_;
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
};

const void* mapped_alias(const void* host);
bool page_locked(const void* host) { return mapped_alias(host) != nullptr; }

// Grows staging slot g to at least n bytes (waits for its in-flight copy first).
cudaError_t stage_reserve(blz_ctx::Stage& g, size_t n) {
  if (!g.ev) {
    cudaError_t e = cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  if (g.bytes >= n) return cudaSuccess;
  if (g.busy) {
    cudaError_t e = cudaEventSynchronize(g.ev);
    if (e != cudaSuccess) return e;
    g.busy = false;
  }
  if (g.p) cudaFreeHost(g.p);
  g.p = nullptr;
  g.bytes = 0;
  cudaError_t e = cudaHostAlloc(&g.p, n, cudaHostAllocDefault);
  if (e == cudaSuccess) g.bytes = n;
  return e;
}

// H2D of one piece of the current chunk: direct from page-locked memory, or
// through the chunk's staging slot (host copy now, DMA on s).
cudaError_t xfer_h2d(blz_ctx* c, void* dst, const void* src, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (page_locked(src)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s);
  blz_ctx::Stage& g = c->st_in[c->cur];
  if (g.busy) {  // the slot's previous chunk is still being uploaded
    cudaError_t e = cudaEventSynchronize(g.ev);
    if (e != cudaSuccess) return e;
    g.busy = false;
  }
  // the first piece of a chunk reserves room for all of the chunk's pieces (add /
  // sub upload two equal ones), also when the slot already holds enough for this
  // piece alone; a piece already in the slot is in flight, so the slot cannot grow
  // mid-chunk
  if (g.off == 0) {
    cudaError_t e = stage_reserve(g, (size_t)c->stage_pieces * n);
    if (e != cudaSuccess) return e;
  } else if (g.bytes < g.off + n) {
    return cudaErrorInvalidValue;
  }
  char* slotp = (char*)g.p + g.off;
  CopyPool::get().copy(slotp, src, n);
  g.off += n;
  return cudaMemcpyAsync(dst, slotp, n, cudaMemcpyHostToDevice, s);
}

// D2H of one piece of the current chunk: direct into page-locked memory, or
// into the chunk's staging slot, copied out by drain() once the DMA is done.
cudaError_t xfer_d2h(blz_ctx* c, void* dst, const void* src, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (page_locked(dst)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s);
  blz_ctx::Stage& g = c->st_out[c->cur];
  if (g.bytes < g.off + n) {
    if (g.off) return cudaErrorInvalidValue;  // one piece per chunk and direction for D2H
    cudaError_t e = stage_reserve(g, std::max(n, 2 * g.bytes));
    if (e != cudaSuccess) return e;
  }
  char* slotp = (char*)g.p + g.off;
  g.off += n;
  g.drains.push_back({dst, slotp, n});
  return cudaMemcpyAsync(slotp, src, n, cudaMemcpyDeviceToHost, s);
}

// Completes the host side of a staged D2H slot (waits for its DMA, copies out).
cudaError_t drain(blz_ctx::Stage& g) {
  if (g.drains.empty()) return cudaSuccess;
  cudaError_t e = cudaEventSynchronize(g.ev);
  for (auto& d : g.drains)
    if (e == cudaSuccess) CopyPool::get().copy(d.dst, d.src, d.n);
  g.drains.clear();
  g.busy = false;
  return e;
}

// Chunks: about 16 per call, each a multiple of 16 block-rows (16-byte aligned SoA
// sub-views) and moving at least kChunkMinBytes, so that small calls are not
// dominated by per-chunk synchronisation.
constexpr uint64_t kChunkMinBytes = uint64_t(8) << 20;

template <class H2D, class Compute, class D2H>
blz_status pipelined_body(blz_ctx* c, uint64_t block_rows, uint64_t bytes_per_block_row, H2D&& h2d, Compute&& compute,
                          D2H&& d2h) {
  uint64_t step = (block_rows + 15) / 16;
  step = (step + 15) / 16 * 16;
  if (step < 16) step = 16;
  if (bytes_per_block_row) {
    uint64_t min_step = (kChunkMinBytes + bytes_per_block_row - 1) / bytes_per_block_row;
    min_step = (min_step + 15) / 16 * 16;
    if (step < min_step) step = min_step;
  }
  const uint64_t nchunks = (block_rows + step - 1) / step;
  if (blz_status st = ensure_pipe(c, 2 * nchunks + 1)) return st;
  // uploads must not overtake earlier work queued on the context stream
  BLZ_CUDA(c, cudaEventRecord(c->events[2 * nchunks], c->stream), "event");
  BLZ_CUDA(c, cudaStreamWaitEvent(c->s_in, c->events[2 * nchunks], 0), "event");
  for (uint64_t i = 0; i < nchunks; ++i) {
    const uint64_t b0 = i * step, b1 = std::min(block_rows, b0 + step);
    cudaEvent_t in_done = c->events[2 * i], k_done = c->events[2 * i + 1];
    c->cur = (int)(i & 1);
    blz_ctx::Stage& gi = c->st_in[c->cur];
    blz_ctx::Stage& go = c->st_out[c->cur];
    gi.off = 0;
    go.off = 0;
    BLZ_CUDA(c, h2d(b0, b1, c->s_in), "H2D");
    if (gi.off) {
      BLZ_CUDA(c, cudaEventRecord(gi.ev, c->s_in), "event");
      gi.busy = true;
    }
    BLZ_CUDA(c, cudaEventRecord(in_done, c->s_in), "event");
    BLZ_CUDA(c, cudaStreamWaitEvent(c->stream, in_done, 0), "event");
    if (blz_status st = compute(b0, b1)) return st;
    BLZ_CUDA(c, cudaEventRecord(k_done, c->stream), "event");
    BLZ_CUDA(c, cudaStreamWaitEvent(c->s_out, k_done, 0), "event");
    BLZ_CUDA(c, d2h(b0, b1, c->s_out), "D2H");
    if (!go.drains.empty()) {
      BLZ_CUDA(c, cudaEventRecord(go.ev, c->s_out), "event");
      go.busy = true;
    }
    // the previous chunk's staged downloads complete while this chunk's move
    BLZ_CUDA(c, drain(c->st_out[c->cur ^ 1]), "D2H staging");
  }
  BLZ_CUDA(c, drain(c->st_out[c->cur]), "D2H staging");
  return BLZ_OK;
}

// Runs the chunk pipeline and always drains all three streams before returning,
// so no copy touches the caller's host buffers after the call (also on errors).
template <class H2D, class Compute, class D2H>
blz_status pipelined(blz_ctx* c, uint64_t block_rows, uint64_t bytes_per_block_row, H2D&& h2d, Compute&& compute,
                     D2H&& d2h) {
  const blz_status st = pipelined_body(c, block_rows, bytes_per_block_row, h2d, compute, d2h);
  c->stage_pieces = 1;
  const cudaError_t e1 = c->s_out ? cudaStreamSynchronize(c->s_out) : cudaSuccess;
  const cudaError_t e2 = c->s_in ? cudaStreamSynchronize(c->s_in) : cudaSuccess;
  const cudaError_t e3 = cudaStreamSynchronize(c->stream);
  for (auto* g : {c->st_in, c->st_out})  // error paths: nothing staged stays pending
    for (int k = 0; k < 2; ++k) {
      g[k].drains.clear();
      g[k].busy = false;
    }
  if (st != BLZ_OK) return st;
  if (e1 != cudaSuccess) return cuda_err(c, e1, "sync");
  if (e2 != cudaSuccess) return cuda_err(c, e2, "sync");
  return cuda_err(c, e3, "sync");
}

// device AoS staging for block-row range [b0, b1) of a (rows x cols) grid
blz_block* aos_at(void* base, uint64_t b0, uint64_t bc) { return (blz_block*)base + b0 * bc; }

// Device alias of a page-locked (pinned / registered, mapped) host buffer, or
// null for pageable memory.  The host entry points read their compressed-record
// inputs and write their compressed-record outputs through this alias: the
// unpack / pack kernels move those bytes over PCIe themselves (zero-copy), so
// the copy engines carry only the dense matrices, and the small transfers of
// one call never queue behind another call's large ones (calls from several
// host threads overlap their PCIe directions).
const void* mapped_alias(const void* host) {
  if (reinterpret_cast<uintptr_t>(host) & 7) return nullptr;  // records are read / written as 8-byte words
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

}  // namespace

extern "C" {

blz_status blz_compress_matrix(blz_ctx* c, const double* values, uint64_t rows, uint64_t cols, blz_block* out,
                               unsigned threads) {
  (void)threads;
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (rows == 0 || cols == 0) return set_err(c, BLZ_INVALID_ARGUMENT, "compress_matrix: empty matrix");
  cudaError_t e;
  double* d = (double*)slot(c, S_IN0, rows * cols * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  blz_cmat m;
  if (blz_status st = scratch_cmat(c, S_CM0, rows, cols, &m)) return st;
  const uint64_t bc = m.block_cols;
  void* aos = slot(c, S_AUX, m.block_rows * bc * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  if (blz_status st = ensure_worklist(c, m.block_rows * bc)) return st;
  blz_block* out_z = (blz_block*)mapped_alias(out);
  auto rows_of = [&](uint64_t b0, uint64_t b1) { return std::min(rows, 8 * b1) - 8 * b0; };
  blz_status st = pipelined(
      c, m.block_rows, 8 * cols * sizeof(double),
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        return xfer_h2d(c, d + 8 * b0 * cols, values + 8 * b0 * cols, rows_of(b0, b1) * cols * sizeof(double), s);
      },
      [&](uint64_t b0, uint64_t b1) {
        const blz_cmat v = sub_rows(m, b0, b1);
        if (blz_status st2 = blz_compress_dev(c, d + 8 * b0 * cols, v.rows, cols, cols, &v)) return st2;
        return blz_pack_aos_dev(c, &v, out_z ? out_z + b0 * bc : aos_at(aos, b0, bc));
      },
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        if (out_z) return cudaSuccess;  // written by the pack kernel
        return xfer_d2h(c, out + b0 * bc, aos_at(aos, b0, bc), (b1 - b0) * bc * sizeof(blz_block), s);
      });
  if (st) return st;
  return latch_status(c);
}

blz_status blz_decompress_matrix(blz_ctx* c, const blz_block* in, uint64_t rows, uint64_t cols, double* out,
                                 unsigned threads) {
  (void)threads;
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (rows == 0 || cols == 0) return BLZ_OK;
  blz_cmat m;
  if (blz_status st = scratch_cmat(c, S_CM0, rows, cols, &m)) return st;
  const uint64_t bc = m.block_cols;
  cudaError_t e;
  void* aos = slot(c, S_AUX, m.block_rows * bc * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  double* d = (double*)slot(c, S_OUT, rows * cols * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  const blz_block* in_z = (const blz_block*)mapped_alias(in);
  auto rows_of = [&](uint64_t b0, uint64_t b1) { return std::min(rows, 8 * b1) - 8 * b0; };
  blz_status st = pipelined(
      c, m.block_rows, 8 * cols * sizeof(double),
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        if (in_z) return cudaSuccess;  // read by the unpack kernel
        return xfer_h2d(c, aos_at(aos, b0, bc), in + b0 * bc, (b1 - b0) * bc * sizeof(blz_block), s);
      },
      [&](uint64_t b0, uint64_t b1) {
        const blz_cmat v = sub_rows(m, b0, b1);
        if (blz_status st2 = blz_unpack_aos_dev(c, in_z ? in_z + b0 * bc : aos_at(aos, b0, bc), &v)) return st2;
        return blz_decompress_dev(c, &v, d + 8 * b0 * cols, cols);
      },
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        return xfer_d2h(c, out + 8 * b0 * cols, d + 8 * b0 * cols, rows_of(b0, b1) * cols * sizeof(double), s);
      });
  if (st) return st;
  return latch_status(c);
}

// Shared body of mat_add / mat_sub / mat_scale on host records (k unused for add/sub).
static blz_status elementwise_host(blz_ctx* c, int op, const blz_block* a, const blz_block* b, uint64_t rows,
                                   uint64_t cols, double k, blz_block* out) {
  blz_cmat ma, mb, mo;
  if (blz_status st = scratch_cmat(c, S_CM0, rows, cols, &ma)) return st;
  if (op != 2)
    if (blz_status st = scratch_cmat(c, S_CM1, rows, cols, &mb)) return st;
  if (blz_status st = scratch_cmat(c, S_CM2, rows, cols, &mo)) return st;
  const uint64_t bc = ma.block_cols, nb = ma.block_rows * bc;
  cudaError_t e;
  // AoS staging: inputs a | b, output o (3 regions)
  blz_block* aos = (blz_block*)slot(c, S_AUX, 3 * nb * sizeof(blz_block), &e);
  if (!aos) return cuda_err(c, e, "scratch allocation");
  blz_block *sa = aos, *sb = aos + nb, *so = aos + 2 * nb;
  if (op != 2)
    if (blz_status st = ensure_worklist(c, nb)) return st;
  // the record streams of add / sub / scale go through the copy engines: both
  // directions are records here, and staged copies measured faster than
  // zero-copy kernel access for these calls (ZC_ELEMENTWISE=1 switches)
#ifndef ZC_ELEMENTWISE
#define ZC_ELEMENTWISE 0
#endif
  const blz_block* a_z = ZC_ELEMENTWISE ? (const blz_block*)mapped_alias(a) : nullptr;
  const blz_block* b_z = ZC_ELEMENTWISE && op != 2 ? (const blz_block*)mapped_alias(b) : nullptr;
  blz_block* o_z = ZC_ELEMENTWISE ? (blz_block*)mapped_alias(out) : nullptr;
  if (a_z) sa = (blz_block*)a_z;
  if (b_z) sb = (blz_block*)b_z;
  if (o_z) so = o_z;
  c->stage_pieces = op != 2 ? 2 : 1;
  return pipelined(
      c, ma.block_rows, bc * sizeof(blz_block) * (op != 2 ? 3 : 2),
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        const size_t n = (b1 - b0) * bc * sizeof(blz_block);
        cudaError_t e2 = cudaSuccess;
        if (!a_z) e2 = xfer_h2d(c, sa + b0 * bc, a + b0 * bc, n, s);
        if (e2 == cudaSuccess && op != 2 && !b_z) e2 = xfer_h2d(c, sb + b0 * bc, b + b0 * bc, n, s);
        return e2;
      },
      [&](uint64_t b0, uint64_t b1) {
        const blz_cmat va = sub_rows(ma, b0, b1), vo = sub_rows(mo, b0, b1);
        if (blz_status st2 = blz_unpack_aos_dev(c, sa + b0 * bc, &va)) return st2;
        if (op == 2) {
          if (blz_status st2 = blz_scale_dev(c, &va, k, &vo)) return st2;
        } else {
          const blz_cmat vb = sub_rows(mb, b0, b1);
          if (blz_status st2 = blz_unpack_aos_dev(c, sb + b0 * bc, &vb)) return st2;
          if (blz_status st2 = addsub_dev(c, op == 1, &va, &vb, &vo)) return st2;
        }
        return blz_pack_aos_dev(c, &vo, so + b0 * bc);
      },
      [&](uint64_t b0, uint64_t b1, cudaStream_t s) {
        if (o_z) return cudaSuccess;  // written by the pack kernel
        return xfer_d2h(c, out + b0 * bc, so + b0 * bc, (b1 - b0) * bc * sizeof(blz_block), s);
      });
}

static blz_status mat_addsub_host(blz_ctx* c, bool sub, const blz_block* a, uint64_t ar, uint64_t ac,
                                  const blz_block* b, uint64_t br, uint64_t bc, blz_block* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = same_dims(c, ar, ac, br, bc, sub ? "mat_sub" : "mat_add")) return st;
  if (ar == 0 || ac == 0) return BLZ_OK;
  if (blz_status st = elementwise_host(c, sub ? 1 : 0, a, b, ar, ac, 0.0, out)) return st;
  return latch_status(c);
}

blz_status blz_mat_add(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b, uint64_t br,
                       uint64_t bc, blz_block* out, unsigned threads) {
  (void)threads;
  return mat_addsub_host(c, false, a, ar, ac, b, br, bc, out);
}

blz_status blz_mat_sub(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b, uint64_t br,
                       uint64_t bc, blz_block* out, unsigned threads) {
  (void)threads;
  return mat_addsub_host(c, true, a, ar, ac, b, br, bc, out);
}

blz_status blz_mat_scale(blz_ctx* c, const blz_block* a, uint64_t rows, uint64_t cols, double k, blz_block* out,
                         unsigned threads) {
  (void)threads;
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (rows == 0 || cols == 0) return BLZ_OK;
  if (!std::isfinite(k)) return set_err(c, BLZ_INVALID_ARGUMENT, "scale: non-finite constant");
  if (blz_status st = elementwise_host(c, 2, a, nullptr, rows, cols, k, out)) return st;
  return latch_status(c);
}

blz_status blz_mat_dot(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b, uint64_t br,
                       uint64_t bc, uint64_t i, uint64_t j, double* out) {
  if (!c || !out) return BLZ_INVALID_ARGUMENT;
  if (ac != br) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_dot: inner dimension mismatch");  // H/matrix.hpp:159
  if (i >= ar || j >= bc) return set_err(c, BLZ_OUT_OF_RANGE, "mat_dot: index out of range");  // :160
  // entry (i, j) reads only block-row i / 8 of a and block-column j / 8 of b
  // (H/matrix.hpp:162-172): those are uploaded, as a (<= 8) x ac and a br x (<= 8)
  // matrix, and the entry is (i % 8, j % 8) of their product.
  const uint64_t bi = i / 8, bj = j / 8;
  blz_cmat ma, mb;
  if (blz_status st = upload_blocks(c, a + bi * ((ac + 7) / 8), std::min<uint64_t>(8, ar - 8 * bi), ac, S_CM0, &ma))
    return st;
  if (blz_status st = upload_block_col(c, b, br, (bc + 7) / 8, bj, std::min<uint64_t>(8, bc - 8 * bj), S_CM1, &mb))
    return st;
  cudaError_t e;
  uint64_t* q = (uint64_t*)slot(c, S_IN0, 4 * sizeof(uint64_t), &e);
  if (!q) return cuda_err(c, e, "scratch allocation");
  const uint64_t hq[2] = {i % 8, j % 8};
  BLZ_CUDA(c, cudaMemcpyAsync(q, hq, sizeof hq, cudaMemcpyHostToDevice, c->stream), "H2D query");
  double* d = (double*)(q + 2);
  if (blz_status st = blz_dot_entries_dev(c, &ma, &mb, q, q + 1, 1, d)) return st;
  BLZ_CUDA(c, cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}

// ---- stage functions (H/codec.hpp, H/dct.hpp), batched over n blocks ------------
// Host arrays in and out; staged through one scratch slot.  The kernels latch
// the reference's errors (normalize: non-finite input; predict: mean slope).
static blz_status stage_call(blz_ctx* c, int stage, const double* in0, uint64_t in0_per, const double* in1,
                             uint64_t in1_per, uint64_t n, double* out0, uint64_t out0_per, double* out1,
                             uint64_t out1_per, double* out2, uint64_t out2_per, void* out3, uint64_t out3_bytes) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (n == 0) return BLZ_OK;
  const uint64_t doubles = n * (in0_per + in1_per + out0_per + out1_per + out2_per) + (n * out3_bytes + 7) / 8;
  cudaError_t e;
  double* d = (double*)slot(c, S_IN0, doubles * sizeof(double) + 64, &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  double* d_in0 = d;
  double* d_in1 = d_in0 + n * in0_per;
  double* d_out0 = d_in1 + n * in1_per;
  double* d_out1 = d_out0 + n * out0_per;
  double* d_out2 = d_out1 + n * out1_per;
  void* d_out3 = d_out2 + n * out2_per;
  BLZ_CUDA(c, cudaMemcpyAsync(d_in0, in0, n * in0_per * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
  if (in1_per)
    BLZ_CUDA(c, cudaMemcpyAsync(d_in1, in1, n * in1_per * sizeof(double), cudaMemcpyHostToDevice, c->stream),
             "H2D");
  BLZ_CUDA(c, blz::launch_stage(lc(c), c->basis, stage, d_in0, d_in1, n, d_out0, d_out1, d_out2, d_out3), "stage");
  auto back = [&](void* h, const void* dv, uint64_t bytes) {
    return bytes ? cudaMemcpyAsync(h, dv, bytes, cudaMemcpyDeviceToHost, c->stream) : cudaSuccess;
  };
  BLZ_CUDA(c, back(out0, d_out0, n * out0_per * sizeof(double)), "D2H");
  BLZ_CUDA(c, back(out1, d_out1, n * out1_per * sizeof(double)), "D2H");
  BLZ_CUDA(c, back(out2, d_out2, n * out2_per * sizeof(double)), "D2H");
  BLZ_CUDA(c, back(out3, d_out3, n * out3_bytes), "D2H");
  return latch_status(c);
}

blz_status blz_normalize_blocks(blz_ctx* c, const double* m, uint64_t n, double* first, double* deltas) {
  return stage_call(c, blz::STAGE_NORMALIZE, m, 64, nullptr, 0, n, deltas, 64, first, 1, nullptr, 0, nullptr, 0);
}
blz_status blz_denormalize_blocks(blz_ctx* c, const double* first, const double* deltas, uint64_t n, double* m) {
  return stage_call(c, blz::STAGE_DENORMALIZE, deltas, 64, first, 1, n, m, 64, nullptr, 0, nullptr, 0, nullptr, 0);
}
blz_status blz_mean_slope_blocks(blz_ctx* c, const double* deltas, uint64_t n, double* s) {
  return stage_call(c, blz::STAGE_MEAN_SLOPE, deltas, 64, nullptr, 0, n, s, 1, nullptr, 0, nullptr, 0, nullptr, 0);
}
blz_status blz_predict_blocks(blz_ctx* c, const double* slopes, const double* slope_mean, uint64_t n,
                              uint8_t* indices, double* snapped, double* lo, double* step) {
  return stage_call(c, blz::STAGE_PREDICT, slopes, 64, slope_mean, 1, n, snapped, 64, lo, 1, step, 1, indices, 64);
}
blz_status blz_quantize_coeffs_blocks(blz_ctx* c, const double* d, uint64_t n, uint8_t* scale, int8_t* coeffs) {
  // coeffs (n x 28 bytes) travel in the out1 slot, scale bytes in out3
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (n == 0) return BLZ_OK;
  cudaError_t e;
  const uint64_t cd = (n * 28 + 7) / 8;
  double* s = (double*)slot(c, S_IN0, (n * 64 + cd) * sizeof(double) + n + 64, &e);
  if (!s) return cuda_err(c, e, "scratch allocation");
  double* d_in = s;
  double* d_c = d_in + n * 64;
  uint8_t* d_scale = reinterpret_cast<uint8_t*>(d_c + cd);
  BLZ_CUDA(c, cudaMemcpyAsync(d_in, d, n * 64 * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
  BLZ_CUDA(c, blz::launch_stage(lc(c), c->basis, blz::STAGE_QUANTIZE, d_in, nullptr, n, nullptr, d_c, nullptr, d_scale),
           "quantize_coeffs");
  BLZ_CUDA(c, cudaMemcpyAsync(coeffs, d_c, n * 28, cudaMemcpyDeviceToHost, c->stream), "D2H");
  BLZ_CUDA(c, cudaMemcpyAsync(scale, d_scale, n, cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}
blz_status blz_dct2_blocks(blz_ctx* c, const double* x, uint64_t n, double* d) {
  return stage_call(c, blz::STAGE_DCT2, x, 64, nullptr, 0, n, d, 64, nullptr, 0, nullptr, 0, nullptr, 0);
}
blz_status blz_idct2_blocks(blz_ctx* c, const double* d, uint64_t n, double* x) {
  return stage_call(c, blz::STAGE_IDCT2, d, 64, nullptr, 0, n, x, 64, nullptr, 0, nullptr, 0, nullptr, 0);
}

// ---- evaluation harness (H/bench.hpp:67-84) ------------------------------------
blz_status blz_mean_relative_error_dev(blz_ctx* c, const double* ref, const double* cand, uint64_t n, double* mean,
                                       uint64_t* excluded) {
  if (!c || !mean || !excluded) return BLZ_INVALID_ARGUMENT;
  return cuda_err(c, blz::launch_mean_rel_error(lc(c), ref, cand, n, mean, (unsigned long long*)excluded),
                  "mean_relative_error");
}

blz_status blz_mean_relative_error(blz_ctx* c, const double* ref, uint64_t rr, uint64_t rc, const double* cand,
                                   uint64_t cr, uint64_t cc, double* mean, uint64_t* excluded) {
  if (!c || !mean || !excluded) return BLZ_INVALID_ARGUMENT;
  if (rr != cr || rc != cc) return set_err(c, BLZ_INVALID_ARGUMENT, "mean_relative_error: dimension mismatch");
  const uint64_t n = rr * rc;
  cudaError_t e;
  double* d = (double*)slot(c, S_IN0, (2 * n + 2) * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  if (n) {
    BLZ_CUDA(c, cudaMemcpyAsync(d, ref, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
    BLZ_CUDA(c, cudaMemcpyAsync(d + n, cand, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
  }
  double* res = d + 2 * n;
  if (blz_status st = blz_mean_relative_error_dev(c, d, d + n, n, res, (uint64_t*)(res + 1))) return st;
  BLZ_CUDA(c, cudaMemcpyAsync(mean, res, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  BLZ_CUDA(c, cudaMemcpyAsync(excluded, res + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}

static blz_status mat_mul_host(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b,
                               uint64_t br, uint64_t bc, blz_block* out_c, double* out_d) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (ac != br) return set_err(c, BLZ_INVALID_ARGUMENT, "mat_mul: inner dimension mismatch");  // H/matrix.hpp:207
  blz_cmat ma, mb;
  if (blz_status st = upload_blocks(c, a, ar, ac, S_CM0, &ma)) return st;
  if (blz_status st = upload_blocks(c, b, br, bc, S_CM1, &mb)) return st;
  cudaError_t e;
  void* scratch = slot(c, S_IN1, blz_matmul_scratch_bytes(&ma, &mb), &e);
  if (!scratch) return cuda_err(c, e, "scratch allocation");
  if (out_c) {
    blz_cmat mo;
    if (blz_status st = scratch_cmat(c, S_CM2, ar, bc, &mo)) return st;
    if (blz_status st = blz_matmul_dev(c, &ma, &mb, BLZ_GEMM_EXACT, scratch, &mo)) return st;
    if (blz_status st = download_blocks(c, &mo, out_c)) return st;
  } else {
    double* d = (double*)slot(c, S_OUT, ar * bc * sizeof(double), &e);
    if (!d) return cuda_err(c, e, "scratch allocation");
    if (blz_status st = blz_matmul_dense_dev(c, &ma, &mb, BLZ_GEMM_EXACT, scratch, d, bc)) return st;
    BLZ_CUDA(c, cudaMemcpyAsync(out_d, d, ar * bc * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  }
  return latch_status(c);
}

blz_status blz_mat_mul(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b, uint64_t br,
                       uint64_t bc, blz_block* out, unsigned threads) {
  (void)threads;
  return mat_mul_host(c, a, ar, ac, b, br, bc, out, nullptr);
}

blz_status blz_mat_mul_dense(blz_ctx* c, const blz_block* a, uint64_t ar, uint64_t ac, const blz_block* b,
                             uint64_t br, uint64_t bc, double* out, unsigned threads) {
  (void)threads;
  return mat_mul_host(c, a, ar, ac, b, br, bc, nullptr, out);
}

blz_status blz_mat_rowdot(blz_ctx* c, const blz_block* a, const blz_block* b, uint64_t rows, uint64_t cols,
                          double* r, double* frob) {
  if (!c || !r) return BLZ_INVALID_ARGUMENT;
  if (rows == 0 || cols == 0) return BLZ_OK;
  blz_cmat ma, mb;
  if (blz_status st = upload_blocks(c, a, rows, cols, S_CM0, &ma)) return st;
  if (blz_status st = upload_blocks(c, b, rows, cols, S_CM1, &mb)) return st;
  cudaError_t e;
  double* d = (double*)slot(c, S_OUT, (rows + 1) * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  if (frob) {
    if (blz_status st = blz_rowdot_frobenius_dev(c, &ma, &mb, d, d + rows)) return st;
  } else if (blz_status st = blz_rowdot_dev(c, &ma, &mb, d)) {
    return st;
  }
  BLZ_CUDA(c, cudaMemcpyAsync(r, d, rows * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  if (frob) BLZ_CUDA(c, cudaMemcpyAsync(frob, d + rows, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}

blz_status blz_compress_blocks(blz_ctx* c, const double* tiles, uint64_t n, blz_block* out) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (n == 0) return BLZ_OK;
  // n tiles side by side form an 8 x 8n dense matrix with ld = 64 ... stored
  // tile-major; view them as an (8n x 8) matrix: tile t = rows 8t..8t+7.
  cudaError_t e;
  double* d = (double*)slot(c, S_IN0, n * 64 * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  BLZ_CUDA(c, cudaMemcpyAsync(d, tiles, n * 64 * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
  blz_cmat m;
  if (blz_status st = scratch_cmat(c, S_CM0, 8 * n, 8, &m)) return st;
  if (blz_status st = blz_compress_dev(c, d, 8 * n, 8, 8, &m)) return st;
  if (blz_status st = download_blocks(c, &m, out)) return st;
  return latch_status(c);
}

blz_status blz_decompress_blocks(blz_ctx* c, const blz_block* in, uint64_t n, double* tiles) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (n == 0) return BLZ_OK;
  blz_cmat m;
  if (blz_status st = upload_blocks(c, in, 8 * n, 8, S_CM0, &m)) return st;
  cudaError_t e;
  double* d = (double*)slot(c, S_OUT, n * 64 * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  if (blz_status st = blz_decompress_dev(c, &m, d, 8)) return st;
  BLZ_CUDA(c, cudaMemcpyAsync(tiles, d, n * 64 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}

blz_status blz_dequantize_blocks(blz_ctx* c, const blz_block* in, uint64_t n, double* tiles) {
  if (!c) return BLZ_INVALID_ARGUMENT;
  if (n == 0) return BLZ_OK;
  blz_cmat m;
  if (blz_status st = upload_blocks(c, in, 8 * n, 8, S_CM0, &m)) return st;
  cudaError_t e;
  double* d = (double*)slot(c, S_OUT, n * 64 * sizeof(double), &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  BLZ_CUDA(c, blz::launch_dequantize(lc(c), c->basis, view(&m), d), "dequantize");
  BLZ_CUDA(c, cudaMemcpyAsync(tiles, d, n * 64 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  return latch_status(c);
}

// ---- .blzc container (H/io.hpp:93-134) ---------------------------------------------
uint64_t blz_blzc_bytes(uint64_t rows, uint64_t cols) { return 13 + 45 * nblk(rows) * nblk(cols); }

blz_status blz_pack_blzc_dev(blz_ctx* c, const blz_cmat* in, uint8_t* out) {
  if (!c || !out) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, in, "write_compressed")) return st;
  return cuda_err(c, blz::launch_pack_blzc(lc(c), view(in), out), "write_compressed");
}

// Header checks of read_header (H/io.hpp:78-89) on the 13 host bytes.
static blz_status parse_header(blz_ctx* c, const uint8_t* h, uint64_t nbytes, uint64_t* rows, uint64_t* cols) {
  const std::string kind = "compressed matrix";
  if (nbytes < 13) return set_err(c, BLZ_IO_ERROR, kind + ": truncated header");
  if (std::memcmp(h, "BLZC", 4) != 0)
    return set_err(c, BLZ_IO_ERROR, kind + ": magic mismatch (not a " + kind + " file)");
  if (h[4] != 1) return set_err(c, BLZ_IO_ERROR, kind + ": unsupported version " + std::to_string(h[4]));
  auto u32 = [](const uint8_t* p) {
    return (uint64_t)p[0] | (uint64_t)p[1] << 8 | (uint64_t)p[2] << 16 | (uint64_t)p[3] << 24;
  };
  *rows = u32(h + 5);
  *cols = u32(h + 9);
  if (*rows == 0 || *cols == 0) return set_err(c, BLZ_IO_ERROR, kind + ": zero dimension in header");
  return BLZ_OK;
}

// Unpacks a device byte stream into `out` (dims must match the header).  A
// zero scale factor in an earlier block is reported before a truncation, as
// the reference's sequential reader does (H/io.hpp:121-132).
static blz_status unpack_stream(blz_ctx* c, const uint8_t* dev_bytes, uint64_t nbytes, const blz_cmat* out) {
  const uint64_t nb = out->block_rows * out->block_cols;
  const uint64_t avail = (nbytes - 13) / 45;
  BLZ_CUDA(c, blz::launch_unpack_blzc(lc(c), dev_bytes, view(out), avail), "read_compressed");
  if (blz_status st = latch_status(c)) return st;
  if (avail < nb)
    return set_err(c, BLZ_IO_ERROR, "compressed matrix: truncated at block " + std::to_string(avail));
  return BLZ_OK;
}

blz_status blz_unpack_blzc_dev(blz_ctx* c, const uint8_t* in, uint64_t nbytes, const blz_cmat* out) {
  if (!c || !in) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = check_cmat(c, out, "read_compressed")) return st;
  uint8_t h[13] = {0};
  if (nbytes >= 13)
    BLZ_CUDA(c, cudaMemcpyAsync(h, in, 13, cudaMemcpyDeviceToHost, c->stream), "read_compressed header");
  BLZ_CUDA(c, cudaStreamSynchronize(c->stream), "sync");
  uint64_t rows = 0, cols = 0;
  if (blz_status st = parse_header(c, h, nbytes, &rows, &cols)) return st;
  if (rows != out->rows || cols != out->cols)
    return set_err(c, BLZ_INVALID_ARGUMENT, "read_compressed: output dimension mismatch");
  return unpack_stream(c, in, nbytes, out);
}

blz_status blz_write_compressed(blz_ctx* c, const blz_block* blocks, uint64_t rows, uint64_t cols, uint8_t* out,
                                uint64_t capacity, uint64_t* written) {
  if (!c || !out) return BLZ_INVALID_ARGUMENT;
  const uint64_t need = blz_blzc_bytes(rows, cols);
  if (capacity < need) return set_err(c, BLZ_INVALID_ARGUMENT, "write_compressed: output buffer too small");
  blz_cmat m;
  if (blz_status st = upload_blocks(c, blocks, rows, cols, S_CM0, &m)) return st;
  cudaError_t e;
  uint8_t* d = (uint8_t*)slot(c, S_OUT, need, &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  if (blz_status st = blz_pack_blzc_dev(c, &m, d)) return st;
  if (blz_status st = latch_status(c)) return st;
  BLZ_CUDA(c, cudaMemcpyAsync(out, d, need, cudaMemcpyDeviceToHost, c->stream), "D2H");
  BLZ_CUDA(c, cudaStreamSynchronize(c->stream), "sync");
  if (written) *written = need;
  return BLZ_OK;
}

blz_status blz_read_compressed(blz_ctx* c, const uint8_t* bytes, uint64_t nbytes, uint64_t* rows, uint64_t* cols,
                               blz_block* out, uint64_t out_capacity) {
  if (!c || !bytes || !rows || !cols) return BLZ_INVALID_ARGUMENT;
  if (blz_status st = parse_header(c, bytes, nbytes, rows, cols)) return st;
  if (!out) return BLZ_OK;  // dimension query
  const uint64_t nb = nblk(*rows) * nblk(*cols);
  if (out_capacity < nb) return set_err(c, BLZ_INVALID_ARGUMENT, "read_compressed: output buffer too small");
  cudaError_t e;
  const uint64_t take = nbytes < blz_blzc_bytes(*rows, *cols) ? nbytes : blz_blzc_bytes(*rows, *cols);
  uint8_t* d = (uint8_t*)slot(c, S_IN0, take, &e);
  if (!d) return cuda_err(c, e, "scratch allocation");
  BLZ_CUDA(c, cudaMemcpyAsync(d, bytes, take, cudaMemcpyHostToDevice, c->stream), "H2D");
  blz_cmat m;
  if (blz_status st = scratch_cmat(c, S_CM0, *rows, *cols, &m)) return st;
  if (blz_status st = unpack_stream(c, d, take, &m)) return st;
  if (blz_status st = download_blocks(c, &m, out)) return st;
  return latch_status(c);
}

}  // extern "C"
