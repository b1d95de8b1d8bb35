import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2202_13007_b200 import device as dev, workloads as W
for gen in ("quadratic", "smooth", "rough"):
    rows = cols = 4096
    A = W.make(gen, rows, cols, seed=1, device="cuda"); B = W.make(gen, rows, cols, seed=2, device="cuda")
    cA, cB = dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols)
    dev.compress(A, cA); dev.compress(B, cB); dev.sync()
    f = lambda m, n: getattr(m, n).cpu().numpy()
    s1, s2 = f(cA, "slope").astype(np.float64), f(cB, "slope").astype(np.float64)
    p1, p2 = f(cA, "scale").astype(np.int64), f(cB, "scale").astype(np.int64)
    c1 = f(cA, "coeffs").view(np.int8).reshape(-1, 28).astype(np.float64)
    c2 = f(cB, "coeffs").view(np.int8).reshape(-1, 28).astype(np.float64)
    os_ = s1 + s2
    phi = np.clip((p1 * p2) // np.maximum(p1 + p2, 1), 1, 255).astype(np.float64)
    with np.errstate(all="ignore"):
        a1 = s1 / os_; a2 = s2 / os_
        w1 = a1 / p1 * phi; w2 = a2 / p2 * phi
        v = w1[:, None] * c1 + w2[:, None] * c2
        k = np.round(v)  # half-even
        fr = v - k
    tie = (np.abs(fr) == 0.5)
    big = ~(np.abs(v) < 2**30)
    gen_mask = (s1 != 0) & (s2 != 0)
    print(gen, "blocks", len(s1), "tie-blocks", int((tie.any(1) & gen_mask).sum()), "big-blocks", int((big.any(1) & gen_mask).sum()),
          "w1 sample", w1[:3], "p", p1[:5], p2[:5])
