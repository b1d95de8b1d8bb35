"""Cost of page-locking a pageable host buffer in place (cudaHostRegister /
cudaHostUnregister) against copying it through a pinned buffer.

    python tools/host_register_probe.py

Measured on the B200 box: 2 GiB registers in 61 ms and unregisters in 56 ms; a
one-thread copy into a pinned buffer takes 145 ms.  The host entry points stage
pageable buffers through page-locked slots with a pool of copy threads instead
(DESIGN.md section 5).
"""
import ctypes as C
import json
import time

import numpy as np
import torch

torch.cuda.init()
cudart = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = C.CDLL(name)
        break
    except OSError:
        pass
res = {}
for gib in (0.25, 2.0):
    n = int(gib * (1 << 30))
    a = np.ones(n // 8)
    p = a.ctypes.data
    t0 = time.perf_counter()
    st = cudart.cudaHostRegister(C.c_void_p(p), C.c_size_t(n), 0)
    t1 = time.perf_counter()
    st2 = cudart.cudaHostUnregister(C.c_void_p(p))
    t2 = time.perf_counter()
    pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
    t3 = time.perf_counter()
    np.copyto(pinned.view(np.float64), a)
    t4 = time.perf_counter()
    res[f"{gib}GiB"] = {"register_ms": round((t1 - t0) * 1e3, 2), "unregister_ms": round((t2 - t1) * 1e3, 2),
                        "status": [st, st2], "numpy_copy_to_pinned_ms": round((t4 - t3) * 1e3, 2)}
print(json.dumps(res))
