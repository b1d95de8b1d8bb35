"""Pinned host <-> device copy bandwidth (the bound of the host-API e2e path)."""
import time

import torch

n = 2 ** 28  # 2 GiB of float64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
h.fill_(1.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = n * 8 / 1e9
th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


tb = t(both)
print(f"H2D {gb / th:.1f} GB/s  D2H {gb / td:.1f} GB/s  both directions at once {2 * gb / tb:.1f} GB/s total")


def d2h_split(k):
    ss = [torch.cuda.Stream() for _ in range(k)]
    step = n // k

    def f():
        for i, s_ in enumerate(ss):
            with torch.cuda.stream(s_):
                h2[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
    return f


def d2h_chunks(chunk):
    def f():
        for i in range(0, n, chunk):
            h2[i:i + chunk].copy_(d[i:i + chunk], non_blocking=True)
    return f


for k in (2, 4):
    print(f"D2H over {k} streams: {gb / t(d2h_split(k)):.1f} GB/s")
for c in (2 ** 20, 2 ** 23):
    print(f"D2H in {c * 8 >> 20} MiB chunks: {gb / t(d2h_chunks(c)):.1f} GB/s")
