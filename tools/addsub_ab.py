"""A/B helper for the add / sub kernel: hashes the outputs of add and sub on
config-1 data and on random records (every phi, slope magnitudes over the
whole exponent range, near-cancelling slope pairs, zero slopes), and times
add / sub at 16384^2.  Run once per library build and compare the hashes:

    BLZ_LIB_PATH=lib/variants/X.so python tools/addsub_ab.py
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402


def digest(m, h):
    for f in ("first", "slope", "scale", "coeffs"):
        h.update(getattr(m, f).cpu().numpy().tobytes())


def random_records(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    m = dev.DeviceCMat(8, 8 * n)
    nb = m.scale.numel()
    m.first.copy_(torch.randn(nb, device="cuda", dtype=torch.float64, generator=g))
    mag = torch.randint(-1000, 1000, (nb,), device="cuda", generator=g).to(torch.float64)
    s = torch.randn(nb, device="cuda", dtype=torch.float64, generator=g) * torch.exp2(mag * (torch.rand(nb, device="cuda", generator=g, dtype=torch.float64) < 0.1))
    s[torch.rand(nb, device="cuda", generator=g) < 0.02] = 0.0
    m.slope.copy_(s)
    m.scale.copy_(torch.randint(1, 256, (nb,), device="cuda", generator=g).to(torch.uint8))
    m.coeffs.copy_(torch.randint(-128, 128, m.coeffs.shape, device="cuda", generator=g).to(torch.int8))
    return m


def main():
    h = hashlib.sha256()
    rows = 16384
    A = dev.compress(W.make("quadratic", rows, rows, seed=1, device="cuda"))
    B = dev.compress(W.make("quadratic", rows, rows, seed=2, device="cuda"))
    out = dev.DeviceCMat(rows, rows)
    for op in (dev.add, dev.sub):
        op(A, B, out)
        dev.sync()
        digest(out, h)
    for seed in (5, 6, 7):
        a, b = random_records(1 << 18, seed), random_records(1 << 18, seed + 100)
        # near-cancelling and exactly cancelling slope pairs
        k = a.slope.numel() // 8
        b.slope[:k] = -a.slope[:k] * (1 + 2.0 ** -40)
        b.slope[k:2 * k] = -a.slope[k:2 * k]
        for op in (dev.add, dev.sub):
            digest(op(a, b), h)
    dev.sync()
    res = {}
    for name, op in (("add", dev.add), ("sub", dev.sub)):
        for _ in range(5):
            op(A, B, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            op(A, B, out)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 50, 4)
    print(json.dumps({"lib": os.environ.get("BLZ_LIB_PATH", "in-tree"), "hash": h.hexdigest()[:16], "ms": res}))


if __name__ == "__main__":
    main()
