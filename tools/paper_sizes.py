"""The paper's own published operations (PAPER.md:320-324, 2000 x 2000 on a
4-core i7-1165G7: add 0.15 ms, scale 0.14 ms, one entry of A.B 0.12 ms) timed
here at the same size: device-resident API (CUDA events, inputs in HBM) and
through the host C ABI (host buffers, copies included).

    python tools/paper_sizes.py [--n 2000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402


def dev_ms(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def host_ms(fn, reps=20):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2000)
n = ap.parse_args().n
a = W.smooth_field(n, n, seed=1, device="cuda")
b = W.smooth_field(n, n, seed=2, device="cuda")
A, B = dev.compress(a), dev.compress(b)
out = dev.DeviceCMat(n, n)
qi = torch.tensor([n // 2], dtype=torch.int64, device="cuda")
qj = torch.tensor([n // 3], dtype=torch.int64, device="cuda")
res = {"n": n, "device_ms": {
    "add": dev_ms(lambda: dev.add(A, B, out)),
    "scale": dev_ms(lambda: dev.scale(A, 3.5, out)),
    "dot_one_entry": dev_ms(lambda: dev.dot_entries(A, B, qi, qj)),
    "compress": dev_ms(lambda: dev.compress(a, out)),
    "decompress": dev_ms(lambda: dev.decompress(A)),
}}
ha, hb = a.cpu().numpy(), b.cpu().numpy()
HA, HB = blz.compress_matrix(ha), blz.compress_matrix(hb)
res["host_api_ms"] = {
    "add": host_ms(lambda: blz.mat_add(HA, HB)),
    "scale": host_ms(lambda: blz.mat_scale(HA, 3.5)),
    "dot_one_entry": host_ms(lambda: blz.mat_dot(HA, HB, n // 2, n // 3)),
    "compress": host_ms(lambda: blz.compress_matrix(ha)),
    "decompress": host_ms(lambda: blz.decompress_matrix(HA)),
}
res["paper_i7_ms"] = {"add": 0.15, "scale": 0.14, "dot_one_entry": 0.12}
print(json.dumps({k: ({kk: round(vv, 4) for kk, vv in v.items()} if isinstance(v, dict) else v) for k, v in res.items()}))
