import hashlib, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2202_13007_b200 import device as dev
from paper_2202_13007_b200 import workloads as W
h = hashlib.sha256()
def dig(c):
    for f in ("first", "slope", "scale", "coeffs"):
        h.update(getattr(c, f).cpu().numpy().tobytes())
A = W.make("quadratic", 16384, 16384, seed=1, device="cuda")
cA = dev.DeviceCMat(16384, 16384)
dev.compress(A, cA); dig(cA)
for gen, r, c in (("rough", 1000, 1024), ("smooth", 2048, 2056), ("smooth", 1024, 1024)):
    dig(dev.compress(W.make(gen, r, c, seed=3, device="cuda")))
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        dev.compress(A, cA)
    e1.record(); torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1) / 30, 4))
print(json.dumps({"lib": os.environ.get("BLZ_LIB_PATH", "").split("/")[-1], "hash": h.hexdigest()[:16], "ms": res}))
