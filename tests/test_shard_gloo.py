"""World-size-2 gloo tests of the block-row sharding logic (CPU).

Each rank owns its block-row shard (shard.block_row_range); the per-rank
arithmetic is stood in for by the oracle port (the CUDA kernels need a GPU),
and the collectives + reassembly of shard.py must reproduce the single-device
results bit for bit: gathered compressed matrices, gathered row dots and the
ascending Frobenius total.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows, cols, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_2202_13007_b200 import shard
        from paper_2202_13007_b200 import workloads as W

        port_ = O.port()
        a = W.smooth_field(rows, cols, seed=5).numpy()
        b = W.smooth_field(rows, cols, seed=6).numpy()
        r0, nr = shard.local_rows(rows, rank, world)
        # per-rank compression of the own rows (stand-in for dev.compress)
        ca = port_.compress_matrix(a[r0:r0 + nr]).reshape(-1)
        cb = port_.compress_matrix(b[r0:r0 + nr]).reshape(-1)
        first = torch.from_numpy(ca["first"].copy())
        slope = torch.from_numpy(ca["slope"].copy())
        coeffs = torch.from_numpy(ca["coeffs"].copy())
        scale = torch.from_numpy(ca["scale_factor"].copy())
        f, s, c, p = shard.gather_soa(first, slope, coeffs, scale)
        # per-rank row dots (stand-in for dev.rowdot) gathered in row order
        r_local = torch.from_numpy(port_.rowdot(ca, cb, nr, cols))
        r_all = shard.gather_uneven(r_local)
        if rank == 0:
            out_q.put({"first": f.numpy(), "slope": s.numpy(), "coeffs": c.numpy(), "scale": p.numpy(),
                       "r": r_all.numpy(), "total": shard.ascending_total_reference(r_all)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols,world", [(64, 48, 2), (75, 40, 2), (40, 24, 3)])
def test_sharded_gather_matches_single_device(rows, cols, world):
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    port_ = O.port()
    from paper_2202_13007_b200 import workloads as W
    a = W.smooth_field(rows, cols, seed=5).numpy()
    b = W.smooth_field(rows, cols, seed=6).numpy()
    full_a = port_.compress_matrix(a).reshape(-1)
    full_b = port_.compress_matrix(b).reshape(-1)
    assert np.array_equal(res["first"].view(np.uint64), full_a["first"].view(np.uint64))
    assert np.array_equal(res["slope"].view(np.uint64), full_a["slope"].view(np.uint64))
    assert np.array_equal(res["coeffs"], full_a["coeffs"])
    assert np.array_equal(res["scale"], full_a["scale_factor"])
    r = port_.rowdot(full_a, full_b, rows, cols)
    assert np.array_equal(res["r"].view(np.uint64), r.view(np.uint64))
    assert np.float64(res["total"]).view(np.uint64) == np.float64(port_.sum_ascending(r)).view(np.uint64)


def test_block_row_ranges_partition():
    from paper_2202_13007_b200 import shard
    for br in (1, 7, 8, 2048, 8191):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.block_row_range(br, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == br
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def _dot_worker(rank, world, port, ar, ac, bc, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_2202_13007_b200 import shard
        from paper_2202_13007_b200 import workloads as W

        port_ = O.port()
        a = W.rough_uniform(ar, ac, seed=91).numpy()
        b = W.smooth_field(ac, bc, seed=92).numpy()
        ca, cb = port_.compress_matrix(a), port_.compress_matrix(b)
        rng = np.random.default_rng(93)
        qi = [0, ar - 1] + rng.integers(0, ar, 30).tolist()
        qj = [bc - 1, 0] + rng.integers(0, bc, 30).tolist()
        r0, nr = shard.local_rows(ar, rank, world)
        # per-rank entries of the own rows (stand-in for dev.dot_entries_rows): +0.0 elsewhere
        part = np.zeros(len(qi), np.float64)
        for k, (i, j) in enumerate(zip(qi, qj)):
            if r0 <= i < r0 + nr:
                part[k] = port_.mat_dot(ca, ar, ac, cb, ac, bc, i, j)
        got = shard.combine_shard_entries(torch.from_numpy(part))
        # signed zeros and NaN payloads survive the combine bit for bit
        special = np.array([-0.0, np.nan, 1e-310, -np.inf], np.float64)
        special.view(np.uint64)[1] |= 0x5A5A
        sp = np.zeros(len(special) * world, np.float64)
        sp[rank::world] = special
        sp_got = shard.combine_shard_entries(torch.from_numpy(sp))
        if rank == 0:
            want = [port_.mat_dot(ca, ar, ac, cb, ac, bc, i, j) for i, j in zip(qi, qj)]
            out_q.put({"got": got.numpy(), "want": np.array(want), "sp": sp_got.numpy(),
                       "sp_want": np.tile(special, 1)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_dot_entries_combine_exactly(world):
    """Batched mat_dot over row shards: each rank's own-row entries, combined by the
    integer sum of the 64-bit patterns, equal the single-device entries bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dot_worker, args=(r, world, port, 45, 37, 29, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res["got"].view(np.uint64), res["want"].view(np.uint64))
    sp = res["sp"].view(np.uint64).reshape(-1, world)
    want = res["sp_want"].view(np.uint64)
    for r in range(world):  # rank r owned entries r, r + world, ...
        assert np.array_equal(sp[:, r], want)
