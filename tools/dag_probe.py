"""Sequential vs multi-stream (DAG) cfg1 step on one GPU (timing probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402

rows = cols = 16384
A = W.make("quadratic", rows, cols, seed=1, device="cuda")
B = W.make("quadratic", rows, cols, seed=2, device="cuda")
cA, cB, cS, cD, cK = (dev.DeviceCMat(rows, cols) for _ in range(5))
oS, oD, oK = (torch.empty((rows, cols), dtype=torch.float64, device="cuda") for _ in range(3))
main = torch.cuda.current_stream()
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    dev.compress(A, cA); dev.compress(B, cB)
    dev.add(cA, cB, cS); dev.sub(cA, cB, cD); dev.scale(cA, 3.5, cK)
    dev.decompress(cS, oS); dev.decompress(cD, oD); dev.decompress(cK, oK)


def dag(fused=False):
    dev.compress(A, cA)
    ea = torch.cuda.Event(); ea.record(main)
    with torch.cuda.stream(s3):
        s3.wait_event(ea)
        if fused:
            dev.scale_decompress(cA, 3.5, cK, oK)
        else:
            dev.scale(cA, 3.5, cK); dev.decompress(cK, oK)
    dev.compress(B, cB)
    eb = torch.cuda.Event(); eb.record(main)
    with torch.cuda.stream(s1):
        s1.wait_event(eb)
        dev.add(cA, cB, cS); dev.decompress(cS, oS)
    with torch.cuda.stream(s2):
        s2.wait_event(eb)
        dev.sub(cA, cB, cD); dev.decompress(cD, oD)
    for s in (s1, s2, s3):
        e = torch.cuda.Event(); e.record(s); main.wait_event(e)


def timeit(f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(n):
        f()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("seq ms", round(timeit(seq), 4))
print("dag ms", round(timeit(dag), 4))
print("dag+fused-scale ms", round(timeit(lambda: dag(True)), 4))
# outputs identical?
seq(); torch.cuda.synchronize()
ref = [oS.clone(), oD.clone(), oK.clone()]
dag(True); torch.cuda.synchronize()
print("identical", all(torch.equal(x.view(torch.int64), y.view(torch.int64)) for x, y in zip(ref, [oS, oD, oK])))
