"""Times each hot-path op on cfg1-sized data with CUDA events (A/B helper).

    BLZ_LIB_PATH=... python tools/time_ops.py [--reps 20] [--rows 16384]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--rows", type=int, default=16384)
ap.add_argument("--gen", default="quadratic")
ap.add_argument("--ops", default="compress,decompress,add,sub,scale")
args = ap.parse_args()
rows = cols = args.rows
A = W.make(args.gen, rows, cols, seed=1, device="cuda")
B = W.make(args.gen, rows, cols, seed=2, device="cuda")
cA, cB, cS = dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols)
out = torch.empty_like(A)
dev.compress(A, cA)
dev.compress(B, cB)
fns = {"compress": lambda: dev.compress(A, cA), "decompress": lambda: dev.decompress(cA, out),
       "add": lambda: dev.add(cA, cB, cS), "sub": lambda: dev.sub(cA, cB, cS), "scale": lambda: dev.scale(cA, 3.5, cS),
       "rowdot": lambda: dev.rowdot(cA, cB), "frobenius": lambda: dev.frobenius(cA, cB),
       "add_dec": lambda: dev.add_decompress(cA, cB, cS, out), "sub_dec": lambda: dev.sub_decompress(cA, cB, cS, out),
       "scale_dec": lambda: dev.scale_decompress(cA, 3.5, cS, out)}
if any(o.startswith("matmul") for o in args.ops.split(",")):
    scratch = dev.matmul_scratch(cA, cB)
    fns["matmul_exact"] = lambda: dev.matmul(cA, cB, mode=0, out=cS, scratch=scratch)
    fns["matmul_fused"] = lambda: dev.matmul(cA, cB, mode=1, out=cS, scratch=scratch)
res = {}
flops = {"matmul_exact": 2.0 * rows ** 3, "matmul_fused": 2.0 * rows ** 3}
for name in args.ops.split(","):
    f = fns[name]
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) / args.reps, 4)
    if name in flops:
        res[name + "_tflops"] = round(flops[name] / (res[name] * 1e-3) / 1e12, 2)
dev.sync()
print(json.dumps({"lib": os.environ.get("BLZ_LIB_PATH", "in-tree"), "ms": res}))
