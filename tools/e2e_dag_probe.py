"""Host-buffer call overlap probe: compress_matrix(B) (H2D-heavy) and
decompress_matrix(K) (D2H-heavy) alone and concurrently from two host threads
(one context each), on 16384^2 config-1 data from pinned buffers.

    python tools/e2e_dag_probe.py
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

n = 16384
nb = (n // 8) ** 2
A = W.make("quadratic", n, n, seed=1, device="cuda")
hA = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
hA.copy_(A)
del A
cb = torch.empty(nb * 48, dtype=torch.uint8, pin_memory=True).numpy().view(blz.BLOCK_DTYPE)
ck = torch.empty(nb * 48, dtype=torch.uint8, pin_memory=True).numpy().view(blz.BLOCK_DTYPE)
dk = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
c1, c2 = blz.Context(0), blz.Context(0)
lib = c1.lib
P = lambda a: a.ctypes.data  # noqa: E731
npA = hA.numpy()
c1.check(lib.blz_compress_matrix(c1.handle, P(npA), n, n, P(ck), 0))


def comp(c):
    c.check(lib.blz_compress_matrix(c.handle, P(npA), n, n, P(cb), 0))


def dec(c):
    c.check(lib.blz_decompress_matrix(c.handle, P(ck), n, n, P(dk), 0))


def t(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


def both():
    th = threading.Thread(target=comp, args=(c2,))
    th.start()
    dec(c1)
    th.join()


res = {"compress_ms": t(lambda: comp(c2)), "decompress_ms": t(lambda: dec(c1)), "both_threads_ms": t(both)}
res["sum_ms"] = res["compress_ms"] + res["decompress_ms"]
print(json.dumps({k: round(v, 2) for k, v in res.items()}))

# --- diagnostics: is the GIL released during the call, and does a library call
# overlap a plain torch copy in the other direction?
counter = [0]
stop = threading.Event()


def spin():
    while not stop.is_set():
        counter[0] += 1


th = threading.Thread(target=spin)
th.start()
t0 = time.perf_counter()
comp(c2)
dt = time.perf_counter() - t0
stop.set()
th.join()
d2 = torch.empty((n, n), dtype=torch.float64, device="cuda")
hd = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
s2 = torch.cuda.Stream()


def torch_d2h():
    with torch.cuda.stream(s2):
        hd.copy_(d2, non_blocking=True)
    s2.synchronize()


def comp_and_torch():
    th2 = threading.Thread(target=torch_d2h)
    th2.start()
    comp(c2)
    th2.join()


print(json.dumps({"python_iters_during_compress": counter[0], "compress_ms": round(dt * 1e3, 2),
                  "torch_d2h_ms": round(t(torch_d2h), 2), "compress_with_torch_d2h_ms": round(t(comp_and_torch), 2)}))
