"""Co-scheduling probe: compress(B) and decompress(K) alone and launched
concurrently on two streams (config-1 data), to see whether the FP64-latency-bound
decompress and the load-latency-bound compress fill each other's stalls.

    BLZ_LIB_PATH=... python tools/cosched_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

n = 16384
A = W.make("quadratic", n, n, seed=1, device="cuda")
B = W.make("quadratic", n, n, seed=2, device="cuda")
cA, cB = dev.DeviceCMat(n, n), dev.DeviceCMat(n, n)
dev.compress(A, cA)
out = torch.empty_like(A)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def comp():
    dev.compress(B, cB)


def dec():
    dev.decompress(cA, out)


def both():
    e = torch.cuda.Event()
    e.record(main)
    with torch.cuda.stream(s1):
        s1.wait_event(e)
        comp()
    with torch.cuda.stream(s2):
        s2.wait_event(e)
        dec()
    for s in (s1, s2):
        f = torch.cuda.Event()
        f.record(s)
        main.wait_event(f)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


r = {"compress": t(comp), "decompress": t(dec), "both": t(both)}
r["sum"] = r["compress"] + r["decompress"]
print(json.dumps({"lib": os.environ.get("BLZ_LIB_PATH", "in-tree"), **{k: round(v, 4) for k, v in r.items()}}))
