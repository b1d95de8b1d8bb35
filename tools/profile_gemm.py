"""Runs the compressed matmul in each GEMM mode (ncu captures of k_gemm_simt / k_gemm_dmma2),
and with --time prints CUDA-event ms and TFLOP/s per mode.

    python tools/profile_gemm.py [--n 4096] [--time] [--reps 3]
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
ap.add_argument("--time", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--modes", default="0,2,3")
a = ap.parse_args()
A = dev.compress(W.make("smooth", a.n, a.n, seed=1, device="cuda"))
B = dev.compress(W.make("smooth", a.n, a.n, seed=2, device="cuda"))
scratch = dev.matmul_scratch(A, B)
C = dev.DeviceCMat(a.n, a.n)
names = {0: "exact (DMUL+DADD)", 1: "fused (default)", 2: "fused DMMA", 3: "fused DFMA"}
for mode in (int(m) for m in a.modes.split(",")):
    D = dev.matmul_dense(A, B, mode=mode, scratch=scratch)  # the GEMM alone (dense out)
    if a.time:
        dev.sync()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(a.reps):
            dev.matmul_dense(A, B, mode=mode, out=D, scratch=scratch)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.reps
        print(f"{names[mode]}: matmul_dense {a.n}^3 {ms:.3f} ms {2 * a.n ** 3 / ms / 1e9:.2f} TFLOP/s", flush=True)
    dev.matmul(A, B, mode=mode, out=C, scratch=scratch)
dev.sync()
torch.cuda.synchronize()
print("ok")

# K-paneled variant (B decompressed panel by panel) against the one-pass call
if a.time:
    for panel in (a.n // 8 // 8, a.n // 8 // 2):
        scr = dev.matmul_panel_scratch(A, B, panel)
        dev.matmul_panel(A, B, panel, mode=1, out=C, scratch=scr)
        dev.sync()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(a.reps):
            dev.matmul_panel(A, B, panel, mode=1, out=C, scratch=scr)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.reps
        print(f"fused, B in panels of {panel} block-rows: matmul {a.n}^3 {ms:.3f} ms, scratch {scr.numel() / 2**30:.2f} GiB "
              f"(one pass: {scratch.numel() / 2**30:.2f} GiB)", flush=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        dev.matmul(A, B, mode=1, out=C, scratch=scratch)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"fused, one pass: matmul {a.n}^3 {ev[0].elapsed_time(ev[1]) / a.reps:.3f} ms", flush=True)
