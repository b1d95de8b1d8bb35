"""Fused all-gather + decompress over block-row shards (needs a B200).

* one process: a compressed matrix split into separate shard arrays is
  decompressed by one gather kernel bitwise like the whole matrix, and
  mat_mul with B given as shards equals mat_mul on the whole B;
* two processes sharing the GPU (gloo for the handshake): each compresses its
  own block-rows, opens the other's shard through CUDA IPC (shard.peer_shards --
  the same mechanism that gives peer access over NVLink on a multi-GPU box) and
  runs the fused path; every rank's C rows equal the single-process product.
"""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU boxes deselect -m gpu
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import shard as S  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

FIELDS = ("first", "slope", "scale", "coeffs")


def _equal(x, y):
    return all(torch.equal(getattr(x, f), getattr(y, f)) for f in FIELDS)


def _shard(cm, r, world):
    lo, hi = S.block_row_range(cm.block_rows, r, world)
    nr = max(0, min(cm.rows, 8 * hi) - 8 * lo)
    sh = dev.DeviceCMat(nr, cm.cols)
    for f in FIELDS:
        getattr(sh, f).copy_(getattr(cm, f)[lo * cm.block_cols:hi * cm.block_cols])
    return sh


@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_gather_decompress_and_matmul_from_shards(world):
    m, k, n = 8 * 13 + 5, 8 * 17 + 3, 8 * 9 + 6
    A = dev.compress(W.rough_uniform(m, k, seed=101, device="cuda"))
    B = dev.compress(W.smooth_field(k, n, seed=102, device="cuda"))
    shards = [_shard(B, r, world) for r in range(world)]
    got = dev.decompress_gather(shards)
    want = dev.decompress(B)
    assert torch.equal(got.view(torch.int64), want.view(torch.int64))
    for mode in (blz.GEMM_EXACT, blz.GEMM_FUSED):
        assert _equal(dev.matmul_gather(A, shards, mode), dev.matmul(A, B, mode))
    with pytest.raises(blz.InvalidArgument, match="shards do not tile"):
        bad = dev.DeviceCMat(8 * 3 + 1, n)  # a non-final shard with a partial block-row
        dev.decompress_gather([bad, shards[-1]])
    with pytest.raises(blz.InvalidArgument, match="shards do not tile"):
        dev.decompress_gather([shards[0], dev.DeviceCMat(8, n + 8)])  # column counts differ
    with pytest.raises(blz.InvalidArgument, match="mat_mul: inner dimension mismatch"):
        dev.matmul_gather(A, shards[:-1] if world > 1 else [dev.DeviceCMat(8, n)])
    with pytest.raises(blz.InvalidArgument, match="1 to 16 shards"):
        dev.decompress_gather([shards[0]] * 17)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _peer_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m, k, n = 8 * 20 + 3, 8 * 22, 8 * 15 + 2
        a = W.rough_uniform(m, k, seed=111, device="cuda")
        b = W.smooth_field(k, n, seed=112, device="cuda")
        # this rank's block-rows of A and of B, compressed locally
        r0a, nra = S.local_rows(m, rank, world)
        r0b, nrb = S.local_rows(k, rank, world)
        a_l = dev.compress(a[r0a:r0a + nra].contiguous())
        b_l = dev.compress(b[r0b:r0b + nrb].contiguous())
        views = S.peer_shards(b_l, k, n)
        c_l = S.matmul_peer(a_l, views, blz.GEMM_EXACT)
        dense_b = dev.decompress_gather(views)
        torch.cuda.synchronize()
        dist.barrier()  # nobody frees its shard while another rank still reads it
        # single-process reference: the whole matrices
        A, B = dev.compress(a), dev.compress(b)
        C = dev.matmul(A, B, blz.GEMM_EXACT)
        lo, hi = S.block_row_range(A.block_rows, rank, world)
        ok_c = all(torch.equal(getattr(c_l, f), getattr(C, f)[lo * C.block_cols:hi * C.block_cols]) for f in FIELDS)
        ok_b = torch.equal(dense_b.view(torch.int64), dev.decompress(B).view(torch.int64))
        q.put((rank, bool(ok_c), bool(ok_b)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_shards_over_ipc_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == [(0, True, True), (1, True, True)]
