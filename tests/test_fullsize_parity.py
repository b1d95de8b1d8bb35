"""Parity at the full BASELINE sizes of configs 2, 3 and 4 (needs a B200).

The oracle cannot run these sizes in seconds, so each config is checked the
way SURVEY.md 8(c) prescribes: blocks are independent, so sampled block-rows
are compared with the reference itself (oracle/_ref, the reference headers
compiled unmodified; the C restatement where it is absent), and every block
is checked through size-independent properties:

* cfg2 (two 65536^2 smooth fields, 67 M blocks each): the default (verified
  fast) compress equals the reference-order exact compress on EVERY block;
  the row dots of the first, middle and last block-rows equal the oracle
  bitwise, and the total is the ascending sum of all row dots.
* cfg3 (8192^3 smooth) and cfg4 (32768^3 rough U[-1,1]), exact GEMM mode:
  the first, middle and last block-rows of C equal the reference's mat_mul;
  the GEMM epilogue's compress is the fast path, so on EVERY output block it
  must equal the exact compress of the same dense product
  (H/matrix.hpp:223-235), and the compressed output must equal the compress
  of mat_mul_dense.
* fused GEMM mode (FP64 FMA chains; tolerance parity, north_star): phi / C
  flips are counted, f and s are compared normwise, and the dense product
  normwise, against the stated tolerances `compare.FUSED_TOL`.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU boxes deselect -m gpu
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import compare as CMP  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _equal(x, y):
    return all(torch.equal(getattr(x, f), getattr(y, f)) for f in ("first", "slope", "scale", "coeffs"))


def _same_blocks(x, y):
    return all(np.array_equal(np.ascontiguousarray(x[f]).view(np.uint8), np.ascontiguousarray(y[f]).view(np.uint8))
               for f in ("first", "slope", "scale_factor", "coeffs"))


def _gen(gen, rows, cols, seed, row0):
    if gen == "smooth":
        return W.smooth_field(rows, cols, seed, device="cuda", row0=row0)
    return W.make(gen, rows, cols, seed + row0, device="cuda")


def _compress_checked(gen, n, seed, chunk_rows):
    """n x n matrix compressed chunk by chunk; every chunk is also compressed in
    exact mode and compared block for block.  Returns (DeviceCMat, mismatches)."""
    full = dev.DeviceCMat(n, n)
    bc = (n + 7) // 8
    ctx = dev.context()
    bad = 0
    for r0 in range(0, n, chunk_rows):
        d = _gen(gen, min(chunk_rows, n - r0), n, seed, r0)
        fast = dev.compress(d)
        ctx.set_mode(blz.MODE_EXACT)
        try:
            exact = dev.compress(d)
            dev.sync()
        finally:
            ctx.set_mode(blz.MODE_DEFAULT)
        bad += 0 if _equal(fast, exact) else 1
        b0 = (r0 // 8) * bc
        b1 = b0 + fast.nblocks
        full.first[b0:b1].copy_(fast.first)
        full.slope[b0:b1].copy_(fast.slope)
        full.coeffs[b0:b1].copy_(fast.coeffs)
        full.scale[b0:b1].copy_(fast.scale)
        del d, fast, exact
    torch.cuda.synchronize()
    return full, bad


def _block_rows(cm, brs):
    """Host AoS blocks of the listed block-rows (packed on the device)."""
    bc = cm.block_cols
    sub = dev.DeviceCMat(8 * len(brs), cm.cols)
    for k, br in enumerate(brs):
        lo, hi = br * bc, (br + 1) * bc
        sub.first[k * bc:(k + 1) * bc].copy_(cm.first[lo:hi])
        sub.slope[k * bc:(k + 1) * bc].copy_(cm.slope[lo:hi])
        sub.coeffs[k * bc:(k + 1) * bc].copy_(cm.coeffs[lo:hi])
        sub.scale[k * bc:(k + 1) * bc].copy_(cm.scale[lo:hi])
    return sub.to_host().blocks


def _host_threads():
    import os
    return len(os.sched_getaffinity(0))


def test_cfg2_full_size_compress_and_rowdots(port):
    n = 65536
    A, bad_a = _compress_checked("smooth", n, 11, 4096)
    B, bad_b = _compress_checked("smooth", n, 12, 4096)
    assert bad_a == 0 and bad_b == 0, "fast compress differs from the exact kernel"
    r, total = dev.frobenius(A, B)
    dev.sync()
    nbr = A.block_rows
    for br in (0, nbr // 2, nbr - 1):
        want = port.rowdot(_block_rows(A, [br]), _block_rows(B, [br]), 8, n)
        got = r[8 * br: 8 * br + 8].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), f"row dots of block-row {br}"
    # the total is the ascending sum of the row dots (SURVEY.md 8(c) restated oracle)
    acc = 0.0
    for v in r.cpu().numpy().tolist():
        acc = acc + v
    assert np.float64(acc).view(np.uint64) == np.float64(float(total.item())).view(np.uint64)


@pytest.mark.parametrize("cfg,gen,n,seeds", [("cfg3", "smooth", 8192, (21, 22)), ("cfg4", "rough", 32768, (41, 42))])
def test_matmul_full_size(cfg, gen, n, seeds, port):
    A, bad_a = _compress_checked(gen, n, seeds[0], 8192)
    B, bad_b = _compress_checked(gen, n, seeds[1], 8192)
    assert bad_a == 0 and bad_b == 0
    scratch = dev.matmul_scratch(A, B)
    # ---- exact mode: compressed output, dense output, the epilogue compress ----
    C = dev.matmul(A, B, mode=blz.GEMM_EXACT, scratch=scratch)
    D = dev.matmul_dense(A, B, mode=blz.GEMM_EXACT, scratch=scratch)
    cD = dev.compress(D)
    ctx = dev.context()
    ctx.set_mode(blz.MODE_EXACT)
    try:
        cD_exact = dev.compress(D)
        dev.sync()
    finally:
        ctx.set_mode(blz.MODE_DEFAULT)
    assert _equal(C, cD), "mat_mul != compress(mat_mul_dense)"
    assert _equal(cD, cD_exact), "GEMM epilogue: fast compress differs from the exact kernel"
    del cD_exact
    # first, middle and last block-rows against the reference's own mat_mul
    nbr = A.block_rows
    brs = [0, nbr // 2, nbr - 1]
    ha, hb = _block_rows(A, brs), B.to_host().blocks
    if O.ref_available():
        want = O.ref().mat_mul(ha, 8 * len(brs), n, hb, n, n, _host_threads())
    else:
        want = port.mat_mul(ha, 8 * len(brs), n, hb, n, n)
    got = _block_rows(C, brs)
    assert _same_blocks(got, want), f"{cfg}: exact-mode block-rows {brs} differ from the reference"
    del hb
    # ---- fused mode against exact mode: counted flips, stated tolerances ----
    Df = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED, scratch=scratch)
    Cf = dev.matmul(A, B, mode=blz.GEMM_FUSED, scratch=scratch)
    assert _equal(Cf, dev.compress(Df))
    st = CMP.cmat_stats(Cf, C)
    st.update(CMP.dense_stats(Df, D))
    s = CMP.summarize(st)
    print(cfg, "fused vs exact:", {k: s[k] for k in ("blocks", "blocks_flipped", "phi_flips", "coeff_flips",
                                                    "max_coeff_delta", "f_normwise", "s_normwise",
                                                    "dense_normwise")})
    assert s["within_tolerance"], s
