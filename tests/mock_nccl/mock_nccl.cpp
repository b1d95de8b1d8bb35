// mock_nccl.cpp -- an in-process, multi-rank stand-in for libnccl, for testing
// the library's NCCL C-ABI entry points (paper_2202_13007_b200/csrc/sharded.cu)
// with G > 1 ranks on ONE GPU.  Test infrastructure only.
//
// Each rank is a host thread with its own blz context and stream; the ranks of
// a world share this library's state.  Implemented: ncclBroadcast,
// ncclAllReduce (sum, in rank order), ncclGroupStart/End (calls inside a group
// are queued per thread and run in order at ncclGroupEnd), ncclCommCount,
// ncclCommUserRank, ncclGetErrorString.  Every collective is a rendezvous of
// all ranks: each rank synchronises its stream (its inputs are ready), posts its
// arguments, waits for the others, performs its own part with synchronous
// cudaMemcpy (device to device, or through the host for the reduction), and
// waits again so no rank reuses a buffer another rank still reads.
//
// Select it with BLZ_NCCL_LIB=/path/libmock_nccl.so before the first NCCL call
// of the process; create communicators with mockNcclWorldCreate / mockNcclComm.
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

namespace {

struct Op {
  enum Kind { BCAST, ALLREDUCE } kind;
  const void* send;
  void* recv;
  size_t count;
  ncclDataType_t dtype;
  int root;
  ncclRedOp_t red;
  cudaStream_t stream;
};

struct World {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long gen = 0;
  std::vector<Op> posted;
  explicit World(int n_) : n(n_), posted(n_) {}

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct Comm {
  World* w;
  int rank;
};

thread_local int group_depth = 0;
thread_local std::vector<std::pair<Comm*, Op>> queued;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    case ncclFloat16: return 2;
    default: return 0;
  }
}

ncclResult_t run(Comm* c, const Op& op) {
  World& w = *c->w;
  if (cudaStreamSynchronize(op.stream) != cudaSuccess) return ncclUnhandledCudaError;
  w.posted[c->rank] = op;
  w.barrier();
  // all ranks must agree on the collective (same kind / count / root)
  for (int r = 0; r < w.n; ++r) {
    const Op& o = w.posted[r];
    if (o.kind != op.kind || o.count != op.count || o.dtype != op.dtype || (op.kind == Op::BCAST && o.root != op.root)) {
      w.barrier();
      return ncclInvalidUsage;
    }
  }
  const size_t bytes = op.count * type_size(op.dtype);
  ncclResult_t res = ncclSuccess;
  if (op.kind == Op::BCAST) {
    const void* src = w.posted[op.root].send;
    if (bytes && src != op.recv && cudaMemcpy(op.recv, src, bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
      res = ncclUnhandledCudaError;
  } else if (bytes) {  // sum in rank order (what the library reduces: float64, and 64-bit integers)
    const bool f64 = op.dtype == ncclFloat64;
    const bool i64 = op.dtype == ncclUint64 || op.dtype == ncclInt64;
    if (!(f64 || i64) || op.red != ncclSum) {
      res = ncclInvalidArgument;
    } else {
      std::vector<double> acc(op.count, 0.0), part(op.count);
      std::vector<uint64_t> iacc(op.count, 0), ipart(op.count);
      for (int r = 0; r < w.n && res == ncclSuccess; ++r) {
        if (cudaMemcpy(f64 ? (void*)part.data() : (void*)ipart.data(), w.posted[r].send, bytes,
                       cudaMemcpyDeviceToHost) != cudaSuccess)
          res = ncclUnhandledCudaError;
        for (size_t i = 0; i < op.count; ++i) {
          if (f64) acc[i] = r == 0 ? part[i] : acc[i] + part[i];
          else iacc[i] += ipart[i];  // two's complement: the same bits for signed and unsigned
        }
      }
      w.barrier();  // every rank has read every send buffer before any recv (maybe == send) changes
      if (res == ncclSuccess && cudaMemcpy(op.recv, f64 ? (const void*)acc.data() : (const void*)iacc.data(), bytes,
                                           cudaMemcpyHostToDevice) != cudaSuccess)
        res = ncclUnhandledCudaError;
    }
  }
  w.barrier();
  return res;
}

ncclResult_t submit(Comm* c, const Op& op) {
  if (!c || !c->w) return ncclInvalidArgument;
  if (type_size(op.dtype) == 0) return ncclInvalidArgument;
  if (op.kind == Op::BCAST && (op.root < 0 || op.root >= c->w->n)) return ncclInvalidArgument;
  if (group_depth > 0) {
    queued.emplace_back(c, op);
    return ncclSuccess;
  }
  return run(c, op);
}

}  // namespace

extern "C" {

// ---- mock-only API ------------------------------------------------------------
void* mockNcclWorldCreate(int n) { return n > 0 ? new World(n) : nullptr; }
void mockNcclWorldDestroy(void* w) { delete static_cast<World*>(w); }
void* mockNcclComm(void* w, int rank) {
  World* wd = static_cast<World*>(w);
  if (!wd || rank < 0 || rank >= wd->n) return nullptr;
  return new Comm{wd, rank};
}
void mockNcclCommFree(void* c) { delete static_cast<Comm*>(c); }

// ---- the NCCL entry points the library binds (sharded.cu) ------------------------
ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t dtype, int root,
                           ncclComm_t comm, cudaStream_t stream) {
  return submit(reinterpret_cast<Comm*>(comm), Op{Op::BCAST, send, recv, count, dtype, root, ncclSum, stream});
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dtype, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
  return submit(reinterpret_cast<Comm*>(comm), Op{Op::ALLREDUCE, send, recv, count, dtype, 0, op, stream});
}

ncclResult_t ncclGroupStart() {
  ++group_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (group_depth == 0) return ncclInvalidUsage;
  if (--group_depth > 0) return ncclSuccess;
  std::vector<std::pair<Comm*, Op>> ops;
  ops.swap(queued);
  ncclResult_t first = ncclSuccess;
  for (auto& [c, op] : ops) {
    const ncclResult_t r = run(c, op);
    if (first == ncclSuccess) first = r;
  }
  return first;
}

ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  const Comm* c = reinterpret_cast<const Comm*>(comm);
  if (!c || !count) return ncclInvalidArgument;
  *count = c->w->n;
  return ncclSuccess;
}

ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  const Comm* c = reinterpret_cast<const Comm*>(comm);
  if (!c || !rank) return ncclInvalidArgument;
  *rank = c->rank;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "unhandled cuda error (mock)";
    case ncclInvalidArgument: return "invalid argument (mock)";
    case ncclInvalidUsage: return "invalid usage (mock)";
    default: return "error (mock)";
  }
}

}  // extern "C"
