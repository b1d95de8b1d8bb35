"""Times dev.frobenius (row dots + ascending total) on config-2-sized inputs (A/B helper).

    BLZ_LIB_PATH=... python tools/time_rowdot.py [--n 65536] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
A, _ = bench._shard_compress("smooth", 0, args.n, args.n, 11)
B, _ = bench._shard_compress("smooth", 0, args.n, args.n, 12)
ms = bench._time_dist(lambda: dev.frobenius(A, B), args.reps, 1)
print(json.dumps({"lib": os.environ.get("BLZ_LIB_PATH", "in-tree"), "n": args.n, "frobenius_ms": round(ms, 3)}))
