// sharded.cu -- block-row sharded operations over NCCL, as C-ABI entry points
// (SURVEY.md 8(b) "sharded variants taking an ncclComm_t and row range", 8(e)).
//
// Rank r of G owns block-rows [BR*r/G, BR*(r+1)/G) of every operand and result
// (the convention of paper_2202_13007_b200/shard.py).  Shard sizes differ by up
// to one block-row, so the gathers are G broadcasts in one NCCL group (exact
// sizes, no padding).  NCCL is opened at run time (dlopen libnccl.so.2): the
// library itself has no NCCL link dependency, and these calls return
// BLZ_NOT_SUPPORTED where NCCL is absent.
//
//   blz_allgather_cmat_nccl     full compressed matrix from the row shards
//                               (45 B per block over NVLink instead of 512 B)
//   blz_rowdot_frobenius_nccl   config 2: local row dots, all ranks' r_i gathered
//                               in row order, ascending total -- bit-identical to
//                               the single-GPU result for every world size
//   blz_frobenius_allreduce_nccl  per-rank ascending partials + one allreduce
//                               (tolerance variant)
//   blz_matmul_nccl             config 4: A row-sharded, compressed B gathered,
//                               local C rows
//   blz_dot_entries_nccl        batched mat_dot: B gathered, each query evaluated
//                               by the rank owning its row, combined by an
//                               integer-sum allreduce of the 64-bit patterns
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "../../include/blaz_cuda.h"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*user_rank)(const ncclComm_t, int*) = nullptr;
  const char* (*errstr)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // BLZ_NCCL_LIB names another NCCL-compatible library (the tests' in-process
    // multi-rank mock, tests/mock_nccl); otherwise the system / torch NCCL
    const char* alt = getenv("BLZ_NCCL_LIB");
    void* h = alt && *alt ? dlopen(alt, RTLD_NOW | RTLD_GLOBAL) : nullptr;
    if (alt && *alt && !h) return a;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.bcast = reinterpret_cast<decltype(a.bcast)>(dlsym(h, "ncclBroadcast"));
    a.allreduce = reinterpret_cast<decltype(a.allreduce)>(dlsym(h, "ncclAllReduce"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.count = reinterpret_cast<decltype(a.count)>(dlsym(h, "ncclCommCount"));
    a.user_rank = reinterpret_cast<decltype(a.user_rank)>(dlsym(h, "ncclCommUserRank"));
    a.errstr = reinterpret_cast<decltype(a.errstr)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.bcast && a.allreduce && a.group_start && a.group_end && a.count && a.user_rank && a.errstr;
    return a;
  }();
  return api;
}

uint64_t shard_lo(uint64_t br, int r, int g) { return br * (uint64_t)r / (uint64_t)g; }

}  // namespace

extern "C" {

// helper from capi.cu (not exported)
__attribute__((visibility("hidden"))) blz_status blz_internal_set_error(blz_ctx* ctx, blz_status st,
                                                                         const char* msg);

static blz_status nccl_status(blz_ctx* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return BLZ_OK;
  const std::string m = std::string(what) + ": " + nccl().errstr(r);
  return blz_internal_set_error(c, BLZ_CUDA_ERROR, m.c_str());
}

static blz_status comm_info(blz_ctx* c, void* comm, int* rank, int* world) {
  if (!nccl().ok) return blz_internal_set_error(c, BLZ_NOT_SUPPORTED, "NCCL (libnccl.so.2) is not available");
  if (!comm) return blz_internal_set_error(c, BLZ_INVALID_ARGUMENT, "null NCCL communicator");
  if (blz_status st = nccl_status(c, nccl().count((ncclComm_t)comm, world), "ncclCommCount")) return st;
  return nccl_status(c, nccl().user_rank((ncclComm_t)comm, rank), "ncclCommUserRank");
}

// Gathers the row shards (block_rows_local x bc blocks each, in rank order) of a
// compressed matrix into `full` (rows x cols of the whole matrix).
blz_status blz_allgather_cmat_nccl(blz_ctx* c, void* comm, const blz_cmat* local, const blz_cmat* full) {
  if (!c || !local || !full) return BLZ_INVALID_ARGUMENT;
  int rank = 0, world = 1;
  if (blz_status st = comm_info(c, comm, &rank, &world)) return st;
  const uint64_t br = full->block_rows, bc = full->block_cols;
  if (local->block_cols != bc || local->block_rows != shard_lo(br, rank + 1, world) - shard_lo(br, rank, world))
    return blz_internal_set_error(c, BLZ_INVALID_ARGUMENT, "allgather: local shard does not match the row range");
  cudaStream_t s = (cudaStream_t)blz_ctx_get_stream(c);
  const NcclApi& n = nccl();
  if (blz_status st = nccl_status(c, n.group_start(), "ncclGroupStart")) return st;
  // every call inside the group is checked; the group is always closed, and the
  // first failing call's code is reported
  ncclResult_t first = ncclSuccess;
  const char* what = "allgather";
  auto keep = [&](ncclResult_t r, const char* w) {
    if (first == ncclSuccess && r != ncclSuccess) {
      first = r;
      what = w;
    }
  };
  for (int r = 0; r < world; ++r) {
    const uint64_t b0 = shard_lo(br, r, world) * bc, nb = shard_lo(br, r + 1, world) * bc - b0;
    if (nb == 0) continue;
    const bool me = r == rank;
    keep(n.bcast(me ? (const void*)local->first : nullptr, full->first + b0, nb, ncclFloat64, r, (ncclComm_t)comm, s),
         "ncclBroadcast(first)");
    keep(n.bcast(me ? (const void*)local->slope : nullptr, full->slope + b0, nb, ncclFloat64, r, (ncclComm_t)comm, s),
         "ncclBroadcast(slope)");
    keep(n.bcast(me ? (const void*)local->coeffs : nullptr, full->coeffs + 28 * b0, 28 * nb, ncclInt8, r,
                 (ncclComm_t)comm, s),
         "ncclBroadcast(coeffs)");
    keep(n.bcast(me ? (const void*)local->scale : nullptr, full->scale + b0, nb, ncclUint8, r, (ncclComm_t)comm, s),
         "ncclBroadcast(scale)");
  }
  const ncclResult_t end = n.group_end();
  if (first != ncclSuccess) return nccl_status(c, first, what);
  return nccl_status(c, end, "allgather");
}

// r_all: device array of the global row count; rank r's rows land at their
// global offset, every rank ends with all rows and the ascending total.
blz_status blz_rowdot_frobenius_nccl(blz_ctx* c, void* comm, const blz_cmat* a_local, const blz_cmat* b_local,
                                     uint64_t rows_total, double* r_all, double* total) {
  if (!c || !a_local || !b_local || !r_all || !total) return BLZ_INVALID_ARGUMENT;
  int rank = 0, world = 1;
  if (blz_status st = comm_info(c, comm, &rank, &world)) return st;
  const uint64_t br = (rows_total + 7) / 8;
  const uint64_t row0 = 8 * shard_lo(br, rank, world);
  if (blz_status st = blz_rowdot_dev(c, a_local, b_local, r_all + row0)) return st;
  cudaStream_t s = (cudaStream_t)blz_ctx_get_stream(c);
  const NcclApi& n = nccl();
  if (blz_status st = nccl_status(c, n.group_start(), "ncclGroupStart")) return st;
  ncclResult_t first = ncclSuccess;
  for (int r = 0; r < world; ++r) {
    const uint64_t lo = 8 * shard_lo(br, r, world);
    const uint64_t hi = 8 * shard_lo(br, r + 1, world) < rows_total ? 8 * shard_lo(br, r + 1, world) : rows_total;
    if (hi <= lo) continue;
    const ncclResult_t res = n.bcast(r == rank ? (const void*)(r_all + lo) : nullptr, r_all + lo, hi - lo,
                                     ncclFloat64, r, (ncclComm_t)comm, s);
    if (first == ncclSuccess) first = res;
  }
  const ncclResult_t end = n.group_end();
  if (first != ncclSuccess) return nccl_status(c, first, "ncclBroadcast(row dots)");
  if (blz_status st = nccl_status(c, end, "allgather of row dots")) return st;
  return blz_sum_dev(c, r_all, rows_total, total);
}

// total: device scalar = sum over ranks of each rank's ascending partial.
blz_status blz_frobenius_allreduce_nccl(blz_ctx* c, void* comm, const blz_cmat* a_local, const blz_cmat* b_local,
                                        double* r_local, double* total) {
  if (!c || !a_local || !b_local || !r_local || !total) return BLZ_INVALID_ARGUMENT;
  int rank = 0, world = 1;
  if (blz_status st = comm_info(c, comm, &rank, &world)) return st;
  if (blz_status st = blz_rowdot_dev(c, a_local, b_local, r_local)) return st;
  if (blz_status st = blz_sum_dev(c, r_local, a_local->rows, total)) return st;
  cudaStream_t s = (cudaStream_t)blz_ctx_get_stream(c);
  return nccl_status(c, nccl().allreduce(total, total, 1, ncclFloat64, ncclSum, (ncclComm_t)comm, s),
                     "allreduce");
}

// C rows of this rank = (A rows of this rank) x (the whole B, gathered from the
// ranks' row shards into b_full).  scratch: blz_matmul_scratch_bytes(a_local, b_full).
blz_status blz_matmul_nccl(blz_ctx* c, void* comm, const blz_cmat* a_local, const blz_cmat* b_local,
                           const blz_cmat* b_full, int mode, void* scratch, const blz_cmat* c_local) {
  if (blz_status st = blz_allgather_cmat_nccl(c, comm, b_local, b_full)) return st;
  return blz_matmul_dev(c, a_local, b_full, mode, scratch, c_local);
}

// Every rank: out[q] = (A x B)(i[q], j[q]) for all n queries.  Each rank
// evaluates the queries on its own rows (others get +0.0, all bits zero), so an
// allreduce of the 64-bit patterns with an integer sum delivers each entry
// exactly as its owner computed it.
blz_status blz_dot_entries_nccl(blz_ctx* c, void* comm, const blz_cmat* a_local, const blz_cmat* b_local,
                                const blz_cmat* b_full, uint64_t rows_total, const uint64_t* i, const uint64_t* j,
                                uint64_t n, double* out) {
  if (!c || !a_local || !b_local || !b_full || (n && (!i || !j || !out))) return BLZ_INVALID_ARGUMENT;
  int rank = 0, world = 1;
  if (blz_status st = comm_info(c, comm, &rank, &world)) return st;
  if (blz_status st = blz_allgather_cmat_nccl(c, comm, b_local, b_full)) return st;
  const uint64_t br = (rows_total + 7) / 8;
  const uint64_t row0 = 8 * shard_lo(br, rank, world);
  if (n == 0) return BLZ_OK;
  if (blz_status st = blz_dot_entries_rows_dev(c, a_local, b_full, i, j, n, row0, rows_total, out)) return st;
  cudaStream_t s = (cudaStream_t)blz_ctx_get_stream(c);
  return nccl_status(c, nccl().allreduce(out, out, n, ncclUint64, ncclSum, (ncclComm_t)comm, s),
                     "allreduce(dot entries)");
}

}  // extern "C"
