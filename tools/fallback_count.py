import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2202_13007_b200 import device as dev
from paper_2202_13007_b200 import workloads as W
ctx = dev.context()
for gen, seed in [("quadratic", 1), ("quadratic", 2), ("smooth", 1), ("rough", 1)]:
    A = W.make(gen, 16384, 16384, seed=seed, device="cuda")
    before = ctx.stats()["compress_exact_blocks"]
    c = dev.compress(A)
    dev.sync()
    n = ctx.stats()["compress_exact_blocks"] - before
    print(gen, seed, "exact-path blocks:", n, "of", c.nblocks)
    del A, c
