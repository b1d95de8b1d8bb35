"""Per-call times of the host-buffer (e2e) step against their PCIe bytes.

    python tools/e2e_probe.py [--rows 16384]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16384)
args = ap.parse_args()
rows = cols = args.rows
nb = (rows // 8) * (cols // 8)
ctx = blz.Context(0)
lib, h = ctx.lib, ctx.handle
hA = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
hB = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
hA.copy_(W.make("quadratic", rows, cols, seed=1, device="cuda"))
hB.copy_(W.make("quadratic", rows, cols, seed=2, device="cuda"))


def blocks():
    t = torch.empty(nb * 48, dtype=torch.uint8, pin_memory=True)
    return t.numpy().view(blz.BLOCK_DTYPE).reshape(rows // 8, cols // 8)


cA, cB, cS = blocks(), blocks(), blocks()
dS = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True).numpy()
P = lambda a: a.ctypes.data  # noqa: E731
npA, npB = hA.numpy(), hB.numpy()
calls = {
    "compress": (lambda: lib.blz_compress_matrix(h, P(npA), rows, cols, P(cA), 0), rows * cols * 8, nb * 48),
    "add": (lambda: lib.blz_mat_add(h, P(cA), rows, cols, P(cB), rows, cols, P(cS), 0), 2 * nb * 48, nb * 48),
    "scale": (lambda: lib.blz_mat_scale(h, P(cA), rows, cols, 3.5, P(cS), 0), nb * 48, nb * 48),
    "decompress": (lambda: lib.blz_decompress_matrix(h, P(cS), rows, cols, P(dS), 0), nb * 48, rows * cols * 8),
}
lib.blz_compress_matrix(h, P(npB), rows, cols, P(cB), 0)
for name, (f, hin, hout) in calls.items():
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        ctx.check(f())
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(f"{name:10s} {ms:7.2f} ms   H2D {hin / 1e9:.3f} GB  D2H {hout / 1e9:.3f} GB   "
          f"{(hin + hout) / ms / 1e6:.1f} GB/s total, {max(hin, hout) / ms / 1e6:.1f} GB/s on the busier direction")
ctx.close()
