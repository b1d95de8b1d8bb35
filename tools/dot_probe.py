"""Latency of a single mat_dot query and of a batch (blz_dot_entries_dev) on 16384^2 operands."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

n = 16384
A = dev.compress(W.make("smooth", n, n, seed=1, device="cuda"))
B = dev.compress(W.make("smooth", n, n, seed=2, device="cuda"))
for q in (1, 64, 100000):
    i = torch.randint(0, n, (q,), device="cuda")
    j = torch.randint(0, n, (q,), device="cuda")
    dev.dot_entries(A, B, i, j)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = dev.dot_entries(A, B, i, j)
    torch.cuda.synchronize()
    print(f"{q} queries: {1e3 * (time.perf_counter() - t0):.2f} ms")
