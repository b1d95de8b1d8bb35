"""cuBLAS DGEMM (torch.matmul, float64) at 8192^3 and 4096^3 as a reference point
for the hand-written fused GEMM kernels (k_gemm_dmma2 / k_gemm_simt).

    python tools/dgemm_probe.py
"""
import json

import torch

res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[n] = {"ms": round(ms, 3), "tflops": round(2 * n ** 3 / ms / 1e9, 2)}
print(json.dumps(res))
