"""HBM write-only / read-only / copy bandwidth on this GPU (torch kernels), for the
decompress (write-dominated) and compress (read-dominated) rooflines."""
import torch

n = 2 ** 28  # 2 GiB of float64
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
x.fill_(1.0)
y.fill_(2.0)


def t(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


gb = n * 8 / 1e9
tw = t(lambda: x.fill_(3.0))
tc = t(lambda: y.copy_(x))
tr = t(lambda: x.sum())
print(f"write-only {gb / tw:.0f} GB/s  copy {2 * gb / tc:.0f} GB/s  read(sum) {gb / tr:.0f} GB/s")
