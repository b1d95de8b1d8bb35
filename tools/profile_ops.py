"""Runs each hot-path kernel a few times on cfg1-sized data (for ncu captures).

    python tools/profile_ops.py [--ops compress,decompress,add,scale] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ops", default="compress,decompress,add,sub,scale_meta")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--gen", default="quadratic")
args = ap.parse_args()
rows = cols = args.rows
A = W.make(args.gen, rows, cols, seed=1, device="cuda")
B = W.make(args.gen, rows, cols, seed=2, device="cuda")
cA, cB, cS = dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols)
cK = dev.ScaledCMat(cA)
out = torch.empty_like(A)
dev.compress(A, cA)
dev.compress(B, cB)
ops = args.ops.split(",")
for _ in range(args.reps):
    if "compress" in ops:
        dev.compress(A, cA)
    if "add" in ops:
        dev.add(cA, cB, cS)
    if "sub" in ops:
        dev.sub(cA, cB, cS)
    if "scale_meta" in ops:
        dev.scale_meta(cA, 3.5, cK)
    if "scale" in ops:
        dev.scale(cA, 3.5, cS)
    if "decompress" in ops:
        dev.decompress(cA, out)
dev.sync()
print("ok")
