"""Runs the compressed matmul once in each mode (for ncu captures of k_gemm_exact / k_gemm_dmma).

    python tools/profile_gemm.py [--n 4096]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
a = ap.parse_args()
A = dev.compress(W.make("smooth", a.n, a.n, seed=1, device="cuda"))
B = dev.compress(W.make("smooth", a.n, a.n, seed=2, device="cuda"))
scratch = dev.matmul_scratch(A, B)
for mode in (0, 1):
    dev.matmul(A, B, mode=mode, scratch=scratch)
dev.sync()
torch.cuda.synchronize()
print("ok")
