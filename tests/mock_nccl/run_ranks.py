"""G ranks as threads on one GPU over the mock NCCL (tests/mock_nccl): runs the
library's NCCL C-ABI entry points (csrc/sharded.cu) and compares every rank's
results with the single-GPU operations, bitwise.  Prints one JSON line.

    BLZ_NCCL_LIB=tests/mock_nccl/libmock_nccl.so python tests/mock_nccl/run_ranks.py G
"""
import ctypes as C
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import shard as S  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

G = int(sys.argv[1])
mock = C.CDLL(os.environ["BLZ_NCCL_LIB"])
mock.mockNcclWorldCreate.restype = C.c_void_p
mock.mockNcclWorldCreate.argtypes = [C.c_int]
mock.mockNcclComm.restype = C.c_void_p
mock.mockNcclComm.argtypes = [C.c_void_p, C.c_int]

FIELDS = ("first", "slope", "scale", "coeffs")
rows, cols, inner = 8 * 37 + 5, 200, 8 * 19 + 3  # ragged: 38 block-rows, partial last block-row
A = dev.compress(W.smooth_field(rows, cols, seed=81, device="cuda"))
Bm = dev.compress(W.rough_uniform(rows, cols, seed=82, device="cuda"))
Ak = dev.compress(W.smooth_field(rows, inner, seed=83, device="cuda"))   # matmul: (rows x inner) x (inner x cols)
Bk = dev.compress(W.quadratic_blocks(inner, cols, seed=84, device="cuda"))
r_ref, t_ref = dev.frobenius(A, Bm)
c_ref = dev.matmul(Ak, Bk, mode=blz.GEMM_EXACT)
# batched mat_dot queries over every shard (first / last rows and columns included)
_g = torch.Generator().manual_seed(85)
q_i = [0, rows - 1, rows - 1, 0] + torch.randint(0, rows, (60,), generator=_g).tolist()
q_j = [0, cols - 1, 0, cols - 1] + torch.randint(0, cols, (60,), generator=_g).tolist()
d_ref = dev.dot_entries(Ak, Bk, torch.tensor(q_i), torch.tensor(q_j))
dev.sync()


def shard_of(cm, rank):
    """Rank's block-row shard of a compressed matrix (copied SoA slices)."""
    lo, hi = S.block_row_range(cm.block_rows, rank, G)
    r0, nr = 8 * lo, max(0, min(cm.rows, 8 * hi) - 8 * lo)
    sh = dev.DeviceCMat(nr, cm.cols)
    b0, b1 = lo * cm.block_cols, hi * cm.block_cols
    for f in FIELDS:
        getattr(sh, f).copy_(getattr(cm, f)[b0:b1])
    return sh, r0, nr


world = mock.mockNcclWorldCreate(G)
results = [None] * G


def rank_main(rank):
    try:
        torch.cuda.set_device(0)
        ctx = blz.Context(0)
        lib, h = ctx.lib, ctx.handle
        comm = C.c_void_p(mock.mockNcclComm(world, rank))
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        out = {}
        a_l, r0, nr = shard_of(A, rank)
        b_l, _, _ = shard_of(Bm, rank)
        torch.cuda.synchronize()
        # all-gather of a compressed matrix from the row shards
        full = dev.DeviceCMat(rows, cols)
        ctx.check(lib.blz_allgather_cmat_nccl(h, comm, a_l.ref(), full.ref()))
        ctx.sync()
        out["allgather"] = all(torch.equal(getattr(full, f), getattr(A, f)) for f in FIELDS)
        # config 2: row dots gathered in row order + ascending total (bit-exact for every G)
        r_all = torch.zeros(rows, dtype=torch.float64, device="cuda")
        tot = torch.zeros(1, dtype=torch.float64, device="cuda")
        ctx.check(lib.blz_rowdot_frobenius_nccl(h, comm, a_l.ref(), b_l.ref(), rows, P(r_all), P(tot)))
        ctx.sync()
        out["rowdot"] = bool(torch.equal(r_all.view(torch.int64), r_ref.view(torch.int64)))
        out["frobenius"] = bool(torch.equal(tot.view(torch.int64), t_ref.view(torch.int64)))
        # tolerance variant: per-rank ascending partials + one allreduce
        r_loc = torch.zeros(max(nr, 1), dtype=torch.float64, device="cuda")
        tot2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        ctx.check(lib.blz_frobenius_allreduce_nccl(h, comm, a_l.ref(), b_l.ref(), P(r_loc), P(tot2)))
        ctx.sync()
        out["allreduce_rel"] = abs(float(tot2.item()) - float(t_ref.item())) / max(abs(float(t_ref.item())), 1e-300)
        # config 4: A row-sharded, compressed B gathered, local C rows
        ak_l, _, _ = shard_of(Ak, rank)
        bk_l, _, _ = shard_of(Bk, rank)
        b_full = dev.DeviceCMat(inner, cols)
        scratch = dev.matmul_scratch(ak_l, b_full)
        c_l = dev.DeviceCMat(ak_l.rows, cols)
        ctx.check(lib.blz_matmul_nccl(h, comm, ak_l.ref(), bk_l.ref(), b_full.ref(), blz.GEMM_EXACT, P(scratch),
                                      c_l.ref()))
        ctx.sync()
        want, _, _ = shard_of(c_ref, rank)
        out["matmul"] = all(torch.equal(getattr(c_l, f), getattr(want, f)) for f in FIELDS)
        # batched mat_dot: B gathered, each rank's rows, integer-sum combine
        qi = torch.tensor(q_i, dtype=torch.int64, device="cuda")
        qj = torch.tensor(q_j, dtype=torch.int64, device="cuda")
        dots = torch.empty(len(q_i), dtype=torch.float64, device="cuda")
        b_full2 = dev.DeviceCMat(inner, cols)
        ctx.check(lib.blz_dot_entries_nccl(h, comm, ak_l.ref(), bk_l.ref(), b_full2.ref(), rows, P(qi), P(qj),
                                           len(q_i), P(dots)))
        ctx.sync()
        out["dot_entries"] = bool(torch.equal(dots.view(torch.int64), d_ref.view(torch.int64)))
        out["rows"] = [r0, nr]
        results[rank] = out
    except Exception as e:  # reported, the test fails on it
        results[rank] = {"error": repr(e)}


threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
for t in threads:
    t.start()
for t in threads:
    t.join(timeout=300)
print(json.dumps({"G": G, "ranks": results}))
