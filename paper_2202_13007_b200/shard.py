"""Block-row sharding of the hot path over ranks (one process per GPU).

Blocks are independent (H/matrix.hpp:105-109), so rank r of G
owns block-rows [r*BR//G, (r+1)*BR//G) of every operand and result:

* compress / decompress / add / sub / scale: purely local, no collective;
* row dots (config 2): local r_i, then an all-gather of the r_i in rank
  (= row) order and one ascending total -- bit-identical to the single-device
  restatement r_i = sum_j A(i,j)B(i,j), frob = sum_i r_i;
  `frobenius_allreduce` is the cheaper tolerance variant (one allreduce);
* matmul (config 4): A row-sharded; compressed B is all-gathered in SoA form
  (45 B per block instead of 512 B of fp64, ~11.4x fewer NVLink bytes) and
  each rank multiplies its A rows by the whole B.

The collective helpers take plain torch tensors (NCCL on GPUs, gloo in the
CPU tests); the per-rank arithmetic is the CUDA library (`device.py`).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def block_row_range(block_rows: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) block-rows owned by `rank` (contiguous, sizes differ by <= 1)."""
    return block_rows * rank // world, block_rows * (rank + 1) // world


def local_rows(rows: int, rank: int, world: int) -> tuple[int, int]:
    """(first element row, number of element rows) of `rank`'s shard."""
    br = (rows + 7) // 8
    lo, hi = block_row_range(br, rank, world)
    r0 = 8 * lo
    r1 = min(rows, 8 * hi)
    return r0, max(0, r1 - r0)


def gather_uneven(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather along dim 0 with per-rank sizes that may differ; rank order.

    NCCL gathers device tensors directly; other backends (gloo: CPU tests, the
    single-GPU multi-rank dry run) go through host memory.  Without a process
    group (one process) the local tensor is the whole result."""
    if not (dist.is_available() and dist.is_initialized()):
        return t
    if t.is_cuda and dist.get_backend(group) != "nccl":
        return gather_uneven(t.cpu(), group).to(t.device)
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def gather_soa(first: torch.Tensor, slope: torch.Tensor, coeffs: torch.Tensor, scale: torch.Tensor,
               group=None):
    """All-gather a row-sharded compressed matrix (SoA arrays of the local
    block-rows) into the full arrays, in block-row order."""
    return (gather_uneven(first, group), gather_uneven(slope, group),
            gather_uneven(coeffs.reshape(-1, 28), group), gather_uneven(scale, group))


def ascending_total_reference(r: torch.Tensor) -> float:
    """The serial ascending sum used as the cross-check in tests (host)."""
    s = 0.0
    for v in r.tolist():
        s = s + v
    return s


# ---- device-level sharded operations (CUDA library + NCCL) -----------------------
def rowdot_frobenius(a_local, b_local, group=None):
    """Row dots of the local shard, gathered in row order, and their ascending
    total (bit-exact and deterministic for every world size)."""
    from . import device as dev
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dev.frobenius(a_local, b_local)  # one pass: the total follows the row dots
    r_local = dev.rowdot(a_local, b_local)
    r_all = gather_uneven(r_local, group)
    return r_all, dev.sum_ascending(r_all)


def frobenius_allreduce(a_local, b_local, group=None):
    """Per-rank ascending partial totals, summed by one allreduce (tolerance parity)."""
    from . import device as dev
    part = dev.sum_ascending(dev.rowdot(a_local, b_local))
    if not (dist.is_available() and dist.is_initialized()):
        return part
    if part.is_cuda and dist.get_backend(group) != "nccl":
        host = part.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        return host.to(part.device)
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part


def allgather_cmat(local, rows: int, cols: int, group=None, out=None):
    """Full compressed matrix (DeviceCMat) from the row shards of all ranks
    (written into `out` when given)."""
    from . import device as dev
    first, slope, coeffs, scale = gather_soa(local.first, local.slope, local.coeffs, local.scale, group)
    full = out if out is not None else dev.DeviceCMat(rows, cols, device=local.buf.device)
    full.first.copy_(first)
    full.slope.copy_(slope)
    full.coeffs.copy_(coeffs)
    full.scale.copy_(scale)
    return full


def matmul(a_local, b_local, b_rows: int, b_cols: int, mode: int = 0, group=None, b_full=None, out=None,
           scratch=None):
    """C rows of this rank = (A rows of this rank) x (all-gathered compressed B).
    `b_full`, `out` and `scratch` are reused when given (steady-state loops)."""
    from . import device as dev
    b_full = allgather_cmat(b_local, b_rows, b_cols, group, out=b_full)
    return dev.matmul(a_local, b_full, mode=mode, out=out, scratch=scratch)


def combine_shard_entries(part: torch.Tensor, group=None) -> torch.Tensor:
    """Entries computed on one shard (+0.0 where another shard owns the query)
    combined over the ranks: an integer sum of the 64-bit patterns, so every entry
    arrives exactly as its owner computed it (-0.0 and NaN payloads included)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return part
    bits = part.view(torch.int64)
    if bits.is_cuda and dist.get_backend(group) != "nccl":
        host = bits.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        return host.to(part.device).view(torch.float64)
    dist.all_reduce(bits, op=dist.ReduceOp.SUM, group=group)
    return bits.view(torch.float64)


def dot_entries(a_local, b_local, rows_total: int, b_rows: int, b_cols: int, qi, qj, group=None, b_full=None):
    """Batched mat_dot (H/matrix.hpp:157-173) over row shards: the
    compressed B is all-gathered, each rank evaluates the queries on its own rows
    of A, and the entries are combined exactly (combine_shard_entries).  qi are
    global row indices, the same on every rank; every rank returns all entries,
    bit-identical to the one-GPU dot_entries."""
    from . import device as dev
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    b_all = allgather_cmat(b_local, b_rows, b_cols, group, out=b_full) if world > 1 else b_local
    r0, _ = local_rows(rows_total, rank, world)
    part = dev.dot_entries_rows(a_local, b_all, qi, qj, r0, rows_total)
    return combine_shard_entries(part, group)


def peer_shards(local, rows: int, cols: int, group=None):
    """Every rank's block-row shard of a compressed matrix as DeviceCMat views --
    the other ranks' arrays opened through CUDA IPC, so kernels read them as peer
    memory over NVLink (or plain device memory when ranks share a GPU).  A
    collective, done once per buffer like communicator setup: the views alias
    the ranks' live buffers, which must stay allocated while they are used."""
    from torch.multiprocessing.reductions import reduce_tensor

    from . import device as dev
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    handles = [None] * world
    dist.all_gather_object(handles, reduce_tensor(local.buf), group=group)
    views = []
    for r, (rebuild, args) in enumerate(handles):
        buf = local.buf if r == rank else rebuild(*args)
        _, nr = local_rows(rows, r, world)
        views.append(local if r == rank else dev.DeviceCMat(nr, cols, buf=buf))
    return views


def matmul_peer(a_local, b_views, mode: int = 0, group=None, out=None, scratch=None):
    """Config 4 without a gather: this rank's C rows = its A rows x B, where B is
    decompressed straight from all ranks' shards (peer_shards) by one kernel --
    the all-gather fused into the decompression (blz_matmul_gather_dev), bitwise
    the result of matmul().  The shards must be complete on every rank first (a
    device sync and a barrier here), and no rank may overwrite its shard before
    the others' products are done (the caller's barrier)."""
    from . import device as dev
    torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.barrier(group)
    return dev.matmul_gather(a_local, b_views, mode, out=out, scratch=scratch)

