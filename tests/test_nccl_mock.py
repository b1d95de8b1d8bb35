"""The NCCL C-ABI entry points (csrc/sharded.cu) with G = 2, 3 and 8 ranks.

One GPU per call is available here, so the ranks are threads of one process,
each with its own library context and stream, joined by an in-process NCCL
stand-in (tests/mock_nccl, selected through BLZ_NCCL_LIB).  Every rank's
gathered matrix, row dots, Frobenius total and matmul rows must equal the
single-GPU results bitwise (the allreduce variant within a stated tolerance).
This covers the row-range arithmetic (shard_lo) and every ncclResult_t path
of the sharded functions for G > 1.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

MOCK = os.path.join(ROOT, "tests", "mock_nccl", "libmock_nccl.so")


@pytest.mark.parametrize("G", [2, 3, 8])
def test_sharded_nccl_entry_points_multi_rank(G):
    if not os.path.exists(MOCK):
        pytest.fail("tests/mock_nccl/libmock_nccl.so not built (run __graft_entry__.build())")
    env = dict(os.environ, BLZ_NCCL_LIB=MOCK)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "mock_nccl", "run_ranks.py"), str(G)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["G"] == G
    rows_seen = 0
    for rank, out in enumerate(res["ranks"]):
        assert out is not None and "error" not in out, (rank, out)
        assert out["allgather"] and out["rowdot"] and out["frobenius"] and out["matmul"], (rank, out)
        assert out["dot_entries"], (rank, out)
        assert out["allreduce_rel"] <= 1e-13, (rank, out)  # per-rank partials summed in rank order
        assert out["rows"][0] == rows_seen  # contiguous block-row shards in rank order
        rows_seen += out["rows"][1]
    assert rows_seen == 8 * 37 + 5
