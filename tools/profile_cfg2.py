"""Builds config-2 operands (two 65536^2 smooth fields, compressed chunk by chunk)
and runs the row dots + Frobenius once (for an ncu capture of k_rowdot / k_sum).

    python tools/profile_cfg2.py [--n 65536]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
args = ap.parse_args()
A, _ = bench._shard_compress("smooth", 0, args.n, args.n, 11)
B, _ = bench._shard_compress("smooth", 0, args.n, args.n, 12)
dev.sync()
dev.frobenius(A, B)
dev.sync()
print("ok")
