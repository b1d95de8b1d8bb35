"""CUDA path vs the oracle / the reference's golden vectors (needs a B200).

Bar: bit-exact.  phi and C[28] byte-exact, f, s and every decompressed /
accumulated double bitwise equal to the reference compiled with
-ffp-contract=off (the exact kernels are built with -fmad=false and follow the
reference's evaluation order).  Calls go through the C ABI (libblaz_cuda.so).
"""
import numpy as np
import pytest
import torch

from conftest import bits, block_diff_report, blocks_equal

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU boxes deselect -m gpu
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import device as dev  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402


def cm_of(golden, n, key, rows, cols):
    return blz.CompressedMatrix(rows, cols, golden[f"m{n}_{key}"])


def test_basis_uploaded_bit_for_bit(golden):
    ctx = blz.default_context()
    assert np.array_equal(bits(ctx.basis()), bits(golden["basis"]))


def test_golden_blocks(golden):
    got = blz.compress_blocks(golden["tiles"])
    assert blocks_equal(got, golden["tiles_c"]), block_diff_report(got, golden["tiles_c"])
    dec = blz.decompress_blocks(golden["tiles_c"])
    assert np.array_equal(bits(dec), bits(golden["tiles_d"]))


def test_golden_ramp_known_answers(golden):
    cb = blz.compress_block(golden["tiles"][0])
    assert cb["scale_factor"] == 20
    assert np.float64(cb["slope"]).view(np.uint64) == np.float64(0.04).view(np.uint64)


def test_golden_pairs(golden):
    pa, pb = golden["pair_a"], golden["pair_b"]
    n = len(pa)
    A = blz.CompressedMatrix(8 * n, 8, pa.reshape(n, 1))
    B = blz.CompressedMatrix(8 * n, 8, pb.reshape(n, 1))
    add = blz.mat_add(A, B).blocks.reshape(-1)
    sub = blz.mat_sub(A, B).blocks.reshape(-1)
    assert blocks_equal(add, golden["pair_add"]), block_diff_report(add, golden["pair_add"])
    assert blocks_equal(sub, golden["pair_sub"]), block_diff_report(sub, golden["pair_sub"])


@pytest.mark.parametrize("n", range(10))
def test_golden_matrices(golden, n):
    rows, cols = (int(v) for v in golden["shapes"][n])
    g = lambda k: golden[f"m{n}_{k}"]  # noqa: E731
    ca = blz.compress_matrix(g("a"))
    assert blocks_equal(ca.blocks, g("ca")), block_diff_report(ca.blocks, g("ca"))
    A, B, BT = cm_of(golden, n, "ca", rows, cols), cm_of(golden, n, "cb", rows, cols), cm_of(golden, n, "cbt", cols, rows)
    assert np.array_equal(bits(blz.decompress_matrix(A)), bits(g("da")))
    assert blocks_equal(blz.mat_add(A, B).blocks, g("add"))
    assert blocks_equal(blz.mat_sub(A, B).blocks, g("sub"))
    assert blocks_equal(blz.mat_scale(A, 3.5).blocks, g("scale"))
    mul = blz.mat_mul(A, BT)
    assert blocks_equal(mul.blocks, g("mul")), block_diff_report(mul.blocks, g("mul"))
    assert np.array_equal(bits(blz.mat_mul_dense(A, BT)), bits(g("muld")))
    dots = [blz.mat_dot(A, BT, int(i), int(j)) for i, j in zip(g("qi"), g("qj"))]
    assert np.array_equal(bits(np.array(dots)), bits(g("dot")))
    r, frob = blz.mat_rowdot(A, B)
    assert np.array_equal(bits(r), bits(g("rowdot")))
    assert np.float64(frob).view(np.uint64) == np.float64(g("frob")).view(np.uint64)


# ---- config 0 at full size (1024 x 1024): every op vs the oracle -------------
@pytest.fixture(scope="module")
def cfg0(port):
    a = W.smooth_field(1024, 1024, seed=1).numpy()
    b = W.smooth_field(1024, 1024, seed=2).numpy()
    return a, b, port.compress_matrix(a), port.compress_matrix(b)


def test_cfg0_compress_decompress(cfg0, port):
    a, b, oa, ob = cfg0
    ca = blz.compress_matrix(a)
    assert blocks_equal(ca.blocks, oa), block_diff_report(ca.blocks, oa)
    assert np.array_equal(bits(blz.decompress_matrix(ca)), bits(port.decompress_matrix(oa, 1024, 1024)))


def test_cfg0_add_sub_scale(cfg0, port):
    a, b, oa, ob = cfg0
    A, B = blz.CompressedMatrix(1024, 1024, oa), blz.CompressedMatrix(1024, 1024, ob)
    for got, want in [(blz.mat_add(A, B).blocks, port.mat_add(oa, ob)),
                      (blz.mat_sub(A, B).blocks, port.mat_sub(oa, ob)),
                      (blz.mat_scale(A, 3.5).blocks, port.mat_scale(oa, 3.5))]:
        assert blocks_equal(got, want), block_diff_report(got, want)


def test_cfg0_device_api_matches_host_api(cfg0):
    a, b, oa, ob = cfg0
    da = dev.compress(torch.from_numpy(a).cuda())
    db = dev.compress(torch.from_numpy(b).cuda())
    s = dev.add(da, db)
    host = s.to_host()
    assert blocks_equal(host.blocks, blz.mat_add(blz.CompressedMatrix(1024, 1024, oa),
                                                 blz.CompressedMatrix(1024, 1024, ob)).blocks)
    back = dev.decompress(s).cpu().numpy()
    assert np.array_equal(bits(back), bits(blz.decompress_matrix(host)))
    dev.sync()


# ---- ragged shapes and edge cases ---------------------------------------------
@pytest.mark.parametrize("rows,cols", [(1, 1), (1, 64), (64, 1), (7, 9), (15, 17), (63, 65), (100, 3)])
def test_ragged_shapes(port, rows, cols):
    rng = np.random.default_rng(rows * 1000 + cols)
    a = rng.normal(size=(rows, cols)).cumsum(axis=1)
    ca = blz.compress_matrix(a)
    oa = port.compress_matrix(a)
    assert blocks_equal(ca.blocks, oa)
    back = blz.decompress_matrix(ca)
    assert back.shape == (rows, cols)
    assert np.array_equal(bits(back), bits(port.decompress_matrix(oa, rows, cols)))


@pytest.mark.parametrize("rows,cols", [(1003, 512), (77, 768), (8, 256), (520, 2304)])
def test_compress_tma_shapes(port, rows, cols):
    """Column counts that are multiples of 256 take the TMA tile loads (whole groups
    of 32 blocks in one block-row); ragged last block-rows and tail groups take the
    direct loads in the same launch.  Bitwise equal to the oracle."""
    for a in (W.smooth_field(rows, cols, seed=rows + cols).numpy(), W.quadratic_blocks(rows, cols, seed=cols).numpy()):
        ca = blz.compress_matrix(a)
        oa = port.compress_matrix(a)
        assert blocks_equal(ca.blocks, oa), block_diff_report(ca.blocks, oa)


def test_errors_match_reference():
    with pytest.raises(blz.InvalidArgument, match="compress_matrix: empty matrix"):
        blz.compress_matrix(np.zeros((0, 4)))
    bad = np.ones((16, 16))
    bad[9, 3] = np.inf
    with pytest.raises(blz.InvalidArgument, match="normalize: non-finite input"):
        blz.compress_matrix(bad)
    a = blz.compress_matrix(np.ones((16, 16)))
    b = blz.compress_matrix(np.ones((16, 24)))
    with pytest.raises(blz.InvalidArgument, match=r"mat_add: dimension mismatch \(16x16 vs 16x24\)"):
        blz.mat_add(a, b)
    with pytest.raises(blz.InvalidArgument, match=r"mat_sub: dimension mismatch"):
        blz.mat_sub(a, b)
    with pytest.raises(blz.InvalidArgument, match="scale: non-finite constant"):
        blz.mat_scale(a, float("nan"))
    c = blz.compress_matrix(np.ones((24, 16)))
    with pytest.raises(blz.InvalidArgument, match="mat_dot: inner dimension mismatch"):
        blz.mat_dot(a, c, 0, 0)
    with pytest.raises(blz.OutOfRange, match="mat_dot: index out of range"):
        blz.mat_dot(a, a, 16, 0)
    with pytest.raises(blz.InvalidArgument, match="mat_mul: inner dimension mismatch"):
        blz.mat_mul(a, c)
    # the context stays usable after errors
    assert blz.compress_matrix(np.ones((8, 8))).blocks["first"][0, 0] == 1.0


def test_identities(port):
    rng = np.random.default_rng(7)
    a = W.smooth_field(40, 56, seed=9).numpy()
    ca = blz.compress_matrix(a)
    assert blocks_equal(blz.mat_scale(ca, 1.0).blocks, ca.blocks)  # matrix_test.cpp:142-149
    zero = blz.decompress_matrix(blz.mat_sub(ca, ca))  # matrix_test.cpp:151-156
    assert not np.any(zero)
    neg = blz.mat_scale(ca, -1.0)  # s1 + s2 == 0 -> dense fallback (block_ops_test.cpp:44-57)
    out = blz.mat_add(ca, neg)
    want = port.mat_add(ca.blocks, neg.blocks)
    assert blocks_equal(out.blocks, want), block_diff_report(out.blocks, want)
    z = blz.mat_scale(ca, 0.0)  # scale by 0 decompresses to zero (block_ops_test.cpp:96-101)
    assert not np.any(blz.decompress_matrix(z))
    b = blz.compress_matrix(rng.normal(size=(40, 56)))
    assert blocks_equal(blz.mat_add(ca, b).blocks, blz.mat_add(b, ca).blocks)  # commutes bitwise


def test_addsub_rounding_ties_and_large_weights(port):
    """Exact ties of w1*C1 + w2*C2 (A + A: w = 1/4 for even phi) and huge
    weights (s1 + s2 nearly cancelling) take the reference rounding sequence."""
    a = W.smooth_field(96, 128, seed=21).numpy()
    ca = blz.compress_matrix(a)
    for other in (ca, blz.mat_scale(ca, 2.0), blz.mat_scale(ca, -0.999999), blz.mat_scale(ca, -1.0000001)):
        for op, ref in ((blz.mat_add, port.mat_add), (blz.mat_sub, port.mat_sub)):
            got = op(ca, other).blocks
            want = ref(ca.blocks, other.blocks)
            assert blocks_equal(got, want), block_diff_report(got, want)
    # ties really occur in A + A
    phis = ca.blocks["scale_factor"]
    assert np.any(phis % 2 == 0)


def test_inplace_add_sub_with_dense_fallback(port):
    """out may be one of the inputs (dev.add(a, b, out=a)): blocks that take the
    s1 + s2 == 0 dense fallback still read the original records."""
    a = W.smooth_field(96, 200, seed=31).numpy()
    ca = dev.compress(torch.from_numpy(a).cuda())
    neg = dev.scale(ca, -1.0)  # every block with s != 0 takes the fallback in ca + neg
    mix = dev.compress(torch.from_numpy(W.rough_uniform(96, 200, seed=32).numpy()).cuda())
    for op, x, y in ((dev.add, ca, neg), (dev.sub, ca, dev.scale(ca, 1.0)), (dev.add, ca, mix), (dev.sub, mix, ca)):
        want = op(x, y)
        for alias in (0, 1):
            xx = dev.DeviceCMat(x.rows, x.cols, buf=x.buf.clone())
            yy = dev.DeviceCMat(y.rows, y.cols, buf=y.buf.clone())
            got = op(xx, yy, out=xx if alias == 0 else yy)
            dev.sync()
            assert _equal_cmats(got, want)
    # a partially overlapping output is rejected (not silently corrupted)
    big = torch.empty(ca.buf.numel() + 512, dtype=torch.uint8, device="cuda")
    v1 = dev.DeviceCMat(ca.rows, ca.cols, buf=big)
    v1.buf[: ca.buf.numel()].copy_(ca.buf)
    v2 = dev.DeviceCMat(ca.rows, ca.cols, buf=big[256:])
    with pytest.raises(blz.InvalidArgument, match="overlaps"):
        dev.add(v1, neg, out=v2)


def test_scale_metadata_only(port):
    """blz_scale_meta_dev (f and s only, phi / C aliased to the input) equals
    mat_scale bitwise, decompresses identically, and keeps the reference's error."""
    a = W.quadratic_blocks(200, 136, seed=33).numpy()
    ca = dev.compress(torch.from_numpy(a).cuda())
    for c in (3.5, -1.0, 0.0, 1e-300, -7.25e12):
        full = dev.scale(ca, c)
        meta = dev.scale_meta(ca, c)
        dev.sync()
        assert meta.c.coeffs == ca.c.coeffs and meta.c.scale == ca.c.scale  # aliased, not copied
        assert _equal_cmats(meta, full)
        want = port.mat_scale(ca.to_host().blocks, c)
        assert blocks_equal(meta.to_host().blocks, want)
        d1, d2 = dev.decompress(meta), dev.decompress(full)
        dev.sync()
        assert torch.equal(d1.view(torch.int64), d2.view(torch.int64))
    with pytest.raises(blz.InvalidArgument, match="scale: non-finite constant"):
        dev.scale_meta(ca, float("inf"))


@pytest.mark.parametrize("gen", ["smooth", "rough"])
def test_batched_block_api_matches_oracle(port, gen):
    """blz_reconstruct_rows_dev / _cols_dev / blz_block_mul_dev over every block
    (pair) of two matrices equal the reference's single-block functions
    (H/block_ops.hpp:87-142) bitwise; dot(b1, b2, i, j) is block_mul's (i, j)."""
    a = W.make(gen, 72, 40, seed=91).numpy()
    b = W.make(gen, 72, 40, seed=92).numpy()
    A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
    ha, hb = A.to_host().blocks.reshape(-1), B.to_host().blocks.reshape(-1)
    for last in (0, 3, 7):
        rr = dev.reconstruct_rows(A, last).cpu().numpy()
        rc = dev.reconstruct_cols(A, last).cpu().numpy()
        for t in range(ha.size):
            assert np.array_equal(bits(rr[t]), bits(port.reconstruct_rows(ha[t], last))), (last, t)
            assert np.array_equal(bits(rc[t]), bits(port.reconstruct_cols(ha[t], last))), (last, t)
    bm = dev.block_mul(A, B).cpu().numpy()
    for t in range(ha.size):
        want = port.block_mul(ha[t], hb[t])
        assert np.array_equal(bits(bm[t]), bits(want)), t
        assert np.float64(bm[t][2, 5]).view(np.uint64) == np.float64(port.dot(ha[t], hb[t], 2, 5)).view(np.uint64)
    with pytest.raises(blz.OutOfRange, match="reconstruct_rows: row index out of range"):
        dev.reconstruct_rows(A, 8)
    with pytest.raises(blz.OutOfRange, match="reconstruct_cols: column index out of range"):
        dev.reconstruct_cols(A, -1)


@pytest.mark.parametrize("rows,cols", [(520, 392), (2056, 4000)])
def test_host_calls_pinned_zero_copy_equal_pageable(rows, cols):
    """Host entry points with page-locked buffers read / write the compressed
    records zero-copy (kernels over PCIe); pageable buffers go through the
    library's page-locked staging slots (parallel host copies, several chunks at
    the larger size); both equal each other bitwise."""
    a = W.smooth_field(rows, cols, seed=61).numpy()
    b = W.quadratic_blocks(rows, cols, seed=62).numpy()
    ctx = blz.default_context()
    lib, h = ctx.lib, ctx.handle
    nb = ((rows + 7) // 8) * ((cols + 7) // 8)

    def pinned_like(x):
        t = torch.empty(x.nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(x.dtype).reshape(x.shape)
        t[...] = x
        return t

    def blocks(pin):
        z = np.zeros(nb, blz.BLOCK_DTYPE)
        return pinned_like(z) if pin else z

    out = {}
    for pin in (False, True):
        xa, xb = (pinned_like(a), pinned_like(b)) if pin else (a.copy(), b.copy())
        ca, cb, cs, cd, ck = (blocks(pin) for _ in range(5))
        dd = pinned_like(np.zeros((rows, cols))) if pin else np.zeros((rows, cols))
        P = lambda v: v.ctypes.data  # noqa: E731
        ctx.check(lib.blz_compress_matrix(h, P(xa), rows, cols, P(ca), 0))
        ctx.check(lib.blz_compress_matrix(h, P(xb), rows, cols, P(cb), 0))
        ctx.check(lib.blz_mat_add(h, P(ca), rows, cols, P(cb), rows, cols, P(cs), 0))
        ctx.check(lib.blz_mat_sub(h, P(ca), rows, cols, P(cb), rows, cols, P(cd), 0))
        ctx.check(lib.blz_mat_scale(h, P(ca), rows, cols, -2.25, P(ck), 0))
        ctx.check(lib.blz_decompress_matrix(h, P(cs), rows, cols, P(dd), 0))
        out[pin] = [x.copy() for x in (ca, cb, cs, cd, ck)] + [dd.copy()]
    for x, y in zip(out[False][:5], out[True][:5]):
        assert blocks_equal(x, y)
    assert np.array_equal(bits(out[False][5]), bits(out[True][5]))


@pytest.mark.parametrize("ar,ac,bc", [(37, 29, 45), (64, 40, 8), (9, 1000, 17)])
def test_mat_dot_reads_one_block_row_and_column(ar, ac, bc, port):
    """mat_dot(i, j) uploads only block-row i / 8 of a and block-column j / 8 of b;
    entries in ragged last block-rows / columns equal the oracle bitwise."""
    a = W.rough_uniform(ar, ac, seed=71).numpy()
    b = W.smooth_field(ac, bc, seed=72).numpy()
    A, B = blz.compress_matrix(a), blz.compress_matrix(b)
    rng = np.random.default_rng(73)
    qs = [(0, 0), (ar - 1, bc - 1), (ar - 1, 0), (0, bc - 1)] + [(int(rng.integers(ar)), int(rng.integers(bc))) for _ in range(12)]
    for i, j in qs:
        got = blz.mat_dot(A, B, i, j)
        want = port.mat_dot(A.blocks, ar, ac, B.blocks, ac, bc, i, j)
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (i, j)


@pytest.mark.parametrize("G", [2, 3, 5])
def test_dot_entries_row_shards_combine(G):
    """blz_dot_entries_rows_dev on each block-row shard of A, combined by the integer
    sum of the 64-bit patterns, equals dot_entries on the whole matrix bitwise
    (the per-rank half of blz_dot_entries_nccl / shard.dot_entries)."""
    from paper_2202_13007_b200 import shard as S
    ar, ac, bc = 8 * 21 + 3, 77, 45
    A = dev.compress(W.rough_uniform(ar, ac, seed=95, device="cuda"))
    B = dev.compress(W.smooth_field(ac, bc, seed=96, device="cuda"))
    g = torch.Generator().manual_seed(97)
    qi = torch.cat([torch.tensor([0, ar - 1]), torch.randint(0, ar, (200,), generator=g)])
    qj = torch.cat([torch.tensor([bc - 1, 0]), torch.randint(0, bc, (200,), generator=g)])
    want = dev.dot_entries(A, B, qi, qj)
    acc = torch.zeros(qi.numel(), dtype=torch.int64, device="cuda")
    for r in range(G):
        lo, hi = S.block_row_range(A.block_rows, r, G)
        r0, nr = 8 * lo, min(ar, 8 * hi) - 8 * lo
        sh = dev.DeviceCMat(nr, ac)
        for f in ("first", "slope", "scale", "coeffs"):
            getattr(sh, f).copy_(getattr(A, f)[lo * A.block_cols:hi * A.block_cols])
        acc += dev.dot_entries_rows(sh, B, qi, qj, r0, ar).view(torch.int64)
    dev.sync()
    assert torch.equal(acc, want.view(torch.int64))
    # one rank: shard.dot_entries is the plain call
    assert torch.equal(S.dot_entries(A, B, ar, ac, bc, qi, qj).view(torch.int64), want.view(torch.int64))
    with pytest.raises(blz.InvalidArgument, match="row shard outside the matrix"):
        dev.dot_entries_rows(A, B, qi, qj, 8, ar)


def test_pageable_staging_slot_reuse_across_ops():
    """A staging slot sized by a one-piece call (scale: one record upload per chunk)
    must grow before a two-piece call (add: both operands' records per chunk) puts
    its first piece in it -- on a fresh context, scale then add then sub."""
    rows = cols = 2040
    a = W.quadratic_blocks(rows, cols, seed=63).numpy()
    b = W.quadratic_blocks(rows, cols, seed=64).numpy()
    A, B = blz.compress_matrix(a), blz.compress_matrix(b)
    ctx = blz.Context()
    try:
        S = blz.mat_scale(A, 0.5, ctx=ctx)
        got = [blz.mat_add(A, B, ctx=ctx), blz.mat_sub(A, B, ctx=ctx), S]
    finally:
        ctx.close()
    want = [blz.mat_add(A, B), blz.mat_sub(A, B), blz.mat_scale(A, 0.5)]
    for x, y in zip(got, want):
        assert blocks_equal(x.blocks, y.blocks)


def test_addsub_every_scale_factor_pair(port):
    """add / sub of records covering every (phi1, phi2) pair in [1, 255]^2 (the
    merged scale factor, H/block_ops.hpp:12-15) equal the oracle."""
    rng = np.random.default_rng(17)
    p1, p2 = np.meshgrid(np.arange(1, 256), np.arange(1, 256))
    n = p1.size
    ra, rb = np.zeros(n, blz.BLOCK_DTYPE), np.zeros(n, blz.BLOCK_DTYPE)
    for r, p in ((ra, p1), (rb, p2)):
        r["first"] = rng.normal(size=n)
        r["slope"] = rng.uniform(0.01, 3.0, size=n)
        r["scale_factor"] = p.reshape(-1).astype(np.uint8)
        r["coeffs"] = rng.integers(-127, 128, size=(n, 28)).astype(np.int8)
    rows, cols = 8 * 255, 8 * 255
    A, B = blz.CompressedMatrix(rows, cols, ra.reshape(255, 255)), blz.CompressedMatrix(rows, cols, rb.reshape(255, 255))
    for got, want in ((blz.mat_add(A, B).blocks, port.mat_add(ra, rb)), (blz.mat_sub(A, B).blocks, port.mat_sub(ra, rb))):
        assert blocks_equal(got, want), block_diff_report(got, want)


def _extreme_records(n, seed):
    rng = np.random.default_rng(seed)
    rec = np.zeros(n, dtype=blz.BLOCK_DTYPE)
    firsts = np.array([0.0, -0.0, 1e-310, -3e-320, 1e300, -1e300, 1.0, -2.5])
    slopes = np.array([0.0, 5e-324, 1e-310, 1e-300, 1.0, -1.0, -1.0000001, 1e300, -3e-5])
    rec["first"] = np.where(rng.random(n) < 0.5, firsts[rng.integers(0, 8, n)], rng.normal(size=n))
    rec["slope"] = np.where(rng.random(n) < 0.7, slopes[rng.integers(0, 9, n)], rng.normal(size=n))
    rec["scale_factor"] = np.array([1, 2, 3, 127, 128, 254, 255], dtype=np.uint8)[rng.integers(0, 7, n)]
    rec["coeffs"] = rng.integers(-127, 128, size=(n, 28)).astype(np.int8)
    return rec


def test_decompress_magnitude_boundaries(port):
    """Records with tiny / subnormal / huge / non-finite f and s and every
    scale-factor class (phi = 0 included) decompress bitwise like the oracle
    (NaN payloads aside)."""
    rng = np.random.default_rng(77)
    fs = [0.0, -0.0, 2.0 ** -955, -(2.0 ** -955), 2.0 ** -956, 3.1 * 2.0 ** -956, 2.0 ** -1000, 5e-324, 1.0, -7.5,
          1e300, -1.7e308]
    ss = [0.0, -0.0, 2.0 ** -834, -(2.0 ** -834), 2.0 ** -835, 1.9 * 2.0 ** -835, 2.0 ** -900, 1e-320, 1.0,
          -3.25, 1e200, np.inf, np.nan]
    recs = []
    for f in fs:
        for sl in ss:
            for phi in (0, 1, 2, 77, 254, 255):
                r = np.zeros(1, blz.BLOCK_DTYPE)
                r["first"], r["slope"], r["scale_factor"] = f, sl, phi
                r["coeffs"] = rng.integers(-127, 128, size=(1, 28)).astype(np.int8)
                recs.append(r)
    ra = np.concatenate(recs)
    n = ra.size - ra.size % 8
    ra = ra[:n]
    rows, cols = 8 * (n // 8), 64
    got = blz.decompress_matrix(blz.CompressedMatrix(rows, cols, ra.reshape(n // 8, 8)))
    want = port.decompress_matrix(ra, rows, cols)
    same = np.array_equal(bits(got), bits(want))
    if not same:  # NaN payloads may differ between x86 and the GPU; compare NaN positions and other bits
        g, w = np.asarray(got), np.asarray(want)
        assert np.array_equal(np.isnan(g), np.isnan(w))
        m = ~np.isnan(w)
        assert np.array_equal(bits(g[m]), bits(w[m]))


def test_records_with_extreme_values(port):
    """add / sub / scale / decompress on records with signed zeros, subnormal and
    huge first values and slopes, cancelling slopes (the dense fallback and the
    huge-weight rounding) and every scale-factor class: equal to the oracle."""
    rows, cols = 64, 96
    nb = (rows // 8) * (cols // 8)
    ra, rb = _extreme_records(nb, 1), _extreme_records(nb, 2)
    A, B = blz.CompressedMatrix(rows, cols, ra), blz.CompressedMatrix(rows, cols, rb)
    for got, want in [(blz.mat_add(A, B).blocks, port.mat_add(ra, rb)),
                      (blz.mat_sub(A, B).blocks, port.mat_sub(ra, rb)),
                      (blz.mat_scale(A, -2.5).blocks, port.mat_scale(ra, -2.5)),
                      (blz.mat_scale(A, 1e10).blocks, port.mat_scale(ra, 1e10))]:
        assert blocks_equal(got, want), block_diff_report(got, want)
    got = blz.decompress_matrix(A)
    want = port.decompress_matrix(ra.reshape(-1), rows, cols)
    assert np.array_equal(bits(got), bits(want))


def test_addsub_zero_scale_factor(port):
    """phi = 0 never comes out of compress, but records read from elsewhere may
    hold it: the weight divisions by 0 (inf / NaN weights, the reference's rounding
    sequence) equal the oracle for add and sub (non-cancelling slopes)."""
    rng = np.random.default_rng(81)
    n = 4096
    ra, rb = np.zeros(n, blz.BLOCK_DTYPE), np.zeros(n, blz.BLOCK_DTYPE)
    for r in (ra, rb):
        r["first"] = rng.normal(size=n)
        r["slope"] = rng.uniform(0.5, 2.0, size=n) * rng.choice([-1.0, 1.0], size=n)
        r["scale_factor"] = rng.integers(0, 256, size=n).astype(np.uint8)
        r["coeffs"] = rng.integers(-127, 128, size=(n, 28)).astype(np.int8)
    ra["scale_factor"][::3] = 0
    rb["scale_factor"][1::3] = 0
    rb["slope"] = np.where(np.abs(ra["slope"] + rb["slope"]) < 0.25, rb["slope"] + 1.0, rb["slope"])
    A = blz.CompressedMatrix(8 * 64, 8 * 64, ra.reshape(64, 64))
    B = blz.CompressedMatrix(8 * 64, 8 * 64, rb.reshape(64, 64))
    for got, want in ((blz.mat_add(A, B).blocks, port.mat_add(ra, rb)), (blz.mat_sub(A, B).blocks, port.mat_sub(ra, rb))):
        assert blocks_equal(got, want), block_diff_report(got, want)


def test_gemm_fused_mode_tolerance(port):
    a = W.smooth_field(64, 96, seed=3).numpy()
    b = W.smooth_field(96, 40, seed=4).numpy()
    A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
    exact = dev.matmul_dense(A, B, mode=blz.GEMM_EXACT).cpu().numpy()
    fused = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED).cpu().numpy()
    want = port.mat_mul_dense(A.to_host().blocks, 64, 96, B.to_host().blocks, 96, 40)
    assert np.array_equal(bits(exact), bits(want))
    # fused (DFMA) mode: normwise tolerance 1e-12 * max(1, ||ref||_inf) * K
    err = np.max(np.abs(fused - want)) / max(1.0, np.max(np.abs(want)))
    assert err <= 1e-12 * 96


# ---- verified fast path vs exact mode vs oracle --------------------------------
def _adversarial_tiles(n_each=2000, seed=5):
    rng = np.random.default_rng(seed)
    tiles = []
    tiles.append(rng.uniform(-100, 100, (n_each, 8, 8)))                       # rough
    tiles.append(np.round(rng.uniform(-5, 5, (n_each, 8, 8))))                 # integer grids (ties)
    tiles.append(np.round(rng.uniform(-5, 5, (n_each, 8, 8))) * 0.25)          # dyadic grids (ties)
    x = np.arange(8.0)
    ramp = x[:, None] * x[None, :]
    tiles.append(ramp[None] * rng.integers(1, 50, (n_each, 1, 1)) / 100.0)     # scaled ramps
    lin = rng.integers(-3, 4, (n_each, 1, 1)) * x[None, :, None] + rng.integers(-3, 4, (n_each, 1, 1)) * x[None, None, :]
    tiles.append(lin.astype(np.float64))                                        # integer planes
    mag = 10.0 ** rng.uniform(-300, 300, (n_each, 1, 1))
    tiles.append(rng.normal(size=(n_each, 8, 8)).cumsum(axis=2) * mag)           # extreme magnitudes
    tiles.append(1e18 + rng.uniform(0, 1e17, (n_each, 8, 8)))                   # INT64 conversion edge
    sparse = np.zeros((n_each, 8, 8))
    sparse[:, 3, 5] = rng.normal(size=n_each)
    tiles.append(sparse)                                                        # one nonzero delta
    const = np.broadcast_to(rng.normal(size=(n_each, 1, 1)), (n_each, 8, 8)).copy()
    tiles.append(const)                                                         # constant blocks
    return np.concatenate(tiles)


def test_fast_path_matches_exact_and_oracle(port):
    tiles = _adversarial_tiles()
    n = tiles.shape[0]
    dense = torch.from_numpy(tiles.reshape(n * 8, 8)).cuda()
    ctx = dev.context()
    assert ctx.fast_path_available()
    before = ctx.stats()["compress_exact_blocks"]
    fast = dev.compress(dense)
    dev.sync()
    used_exact = ctx.stats()["compress_exact_blocks"] - before
    ctx.set_mode(blz.MODE_EXACT)
    try:
        exact = dev.compress(dense)
        dev.sync()
    finally:
        ctx.set_mode(blz.MODE_DEFAULT)
    hf, he = fast.to_host().blocks.reshape(-1), exact.to_host().blocks.reshape(-1)
    want = port.compress_matrix(tiles.reshape(n * 8, 8)).reshape(-1)
    assert blocks_equal(he, want), block_diff_report(he, want)
    assert blocks_equal(hf, want), block_diff_report(hf, want)
    # the exact path must stay the rare path even on these adversarial grids
    assert used_exact < 0.25 * n, used_exact


def _extreme_tiles(n_each=256, seed=11):
    """Blocks at the edges of binary64: subnormal and near-2^-1021 deltas (where
    halving rounds), a subnormal next to a unit delta, 5e307 steps, signed zeros
    with one subnormal."""
    rng = np.random.default_rng(seed)
    tiles = []
    tiles.append(rng.integers(-1000, 1000, size=(n_each, 8, 8)).astype(np.float64) * 5e-324)
    tiles.append(rng.normal(size=(n_each, 8, 8)) * 1e-306)
    mixed = np.zeros((n_each, 8, 8))
    mixed[:, 2, 3] = 3e-310 * rng.integers(1, 9, size=n_each)
    mixed[:, 5, 6] = rng.normal(size=n_each)
    tiles.append(mixed)
    huge = np.zeros((n_each, 8, 8))
    huge[:, 0, 1] = 5e307 * rng.choice([-1.0, 1.0], size=n_each)
    huge[:, 4, 4] = rng.normal(size=n_each)
    tiles.append(huge)
    signed_zero = np.where(rng.random((n_each, 8, 8)) < 0.5, -0.0, 0.0)
    signed_zero[:, 7, 7] = 1e-320
    tiles.append(signed_zero)
    return np.concatenate(tiles)


def test_fast_path_extreme_magnitudes(port):
    """Subnormal and near-2^-1021 deltas, zero tests on subnormal high words,
    overflowing sums: the fast path must certify or hand over every block, so
    fast == exact == oracle on all of them."""
    tiles = _extreme_tiles()
    n = tiles.shape[0]
    dense = torch.from_numpy(tiles.reshape(n * 8, 8)).cuda()
    ctx = dev.context()
    fast = dev.compress(dense)
    dev.sync()
    ctx.set_mode(blz.MODE_EXACT)
    try:
        exact = dev.compress(dense)
        dev.sync()
    finally:
        ctx.set_mode(blz.MODE_DEFAULT)
    hf, he = fast.to_host().blocks.reshape(-1), exact.to_host().blocks.reshape(-1)
    want = port.compress_matrix(tiles.reshape(n * 8, 8)).reshape(-1)
    assert blocks_equal(he, want), block_diff_report(he, want)
    assert blocks_equal(hf, want), block_diff_report(hf, want)


def test_decompress_shared_products_match_plain_kernel(port):
    """The default decompress shares the products of bitwise-repeated basis
    entries; exact mode runs one product per term.  Both equal the oracle."""
    tiles = _adversarial_tiles()
    n = tiles.shape[0]
    a = W.smooth_field(200, 136, seed=5).numpy()
    for m in (tiles.reshape(n * 8, 8), a, np.random.default_rng(3).normal(size=(64, 72)) * 1e3):
        cm = blz.compress_matrix(m)
        fast = blz.decompress_matrix(cm)
        ctx = blz.default_context()
        ctx.set_mode(blz.MODE_EXACT)
        try:
            plain = blz.decompress_matrix(cm)
        finally:
            ctx.set_mode(blz.MODE_DEFAULT)
        want = port.decompress_matrix(cm.blocks.reshape(-1), *m.shape)
        assert np.array_equal(bits(fast), bits(want))
        assert np.array_equal(bits(plain), bits(want))


def test_fast_path_cfg1_sample(port):
    a = W.quadratic_blocks(512, 4096, seed=21)
    ctx = dev.context()
    before = ctx.stats()["compress_exact_blocks"]
    ca = dev.compress(a.cuda())
    dev.sync()
    used_exact = ctx.stats()["compress_exact_blocks"] - before
    assert blocks_equal(ca.to_host().blocks, port.compress_matrix(a.numpy()))
    assert used_exact <= 0.001 * ca.nblocks, used_exact


def test_rowdot_frobenius_medium(port):
    """Config-2 restatement at a CPU-checkable size (512 x 4100, ragged columns)."""
    a = W.smooth_field(512, 4100, seed=31).numpy()
    b = W.smooth_field(512, 4100, seed=32).numpy()
    A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
    r, tot = dev.frobenius(A, B)
    oa, ob = A.to_host().blocks, B.to_host().blocks
    want = port.rowdot(oa, ob, 512, 4100)
    assert np.array_equal(bits(r.cpu().numpy()), bits(want))
    assert np.float64(tot.item()).view(np.uint64) == np.float64(port.sum_ascending(want)).view(np.uint64)


@pytest.mark.parametrize("rows,cols", [(8, 8), (40, 200), (1000, 776), (333, 9000)])
def test_rowdot_total_one_pass_equals_two_calls(rows, cols):
    """blz_rowdot_frobenius_dev (row dots with the ascending total formed inside the
    split kernel, or k_sum after the unsplit one) equals blz_rowdot_dev + blz_sum_dev."""
    A = dev.compress(W.smooth_field(rows, cols, seed=35, device="cuda"))
    B = dev.compress(W.rough_uniform(rows, cols, seed=36, device="cuda"))
    r1, t1 = dev.frobenius(A, B)
    r2 = dev.rowdot(A, B)
    t2 = dev.sum_ascending(r2)
    dev.sync()
    assert torch.equal(r1.view(torch.int64), r2.view(torch.int64))
    assert torch.equal(t1.view(torch.int64), t2.view(torch.int64))


def test_rowdot_block_row_tail(port):
    """Block-row count not a multiple of 4 and a single block column."""
    for rows, cols in [(40, 8), (13, 3), (72, 70)]:
        a = W.smooth_field(rows, cols, seed=rows).numpy()
        b = W.quadratic_blocks(rows, cols, seed=cols).numpy()
        A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
        r = dev.rowdot(A, B).cpu().numpy()
        want = port.rowdot(A.to_host().blocks, B.to_host().blocks, rows, cols)
        assert np.array_equal(bits(r), bits(want)), (rows, cols)


def test_matmul_exact_medium(port):
    """Exact compressed GEMM (SIMT DMUL+DADD, ascending k) vs the oracle, ragged sizes
    spanning several 128 x 128 CTA tiles and a K not a multiple of the k-tile."""
    a = W.smooth_field(264, 333, seed=41).numpy()
    b = W.quadratic_blocks(333, 200, seed=42).numpy()
    A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
    oa, ob = A.to_host().blocks, B.to_host().blocks
    got = dev.matmul_dense(A, B, mode=blz.GEMM_EXACT).cpu().numpy()
    want = port.mat_mul_dense(oa, 264, 333, ob, 333, 200)
    assert np.array_equal(bits(got), bits(want))
    gc = dev.matmul(A, B, mode=blz.GEMM_EXACT).to_host().blocks
    wc = port.mat_mul(oa, 264, 333, ob, 333, 200)
    assert blocks_equal(gc, wc), block_diff_report(gc, wc)


def test_matmul_fused_dmma_tolerance(port):
    """Fused mode = DMMA tensor cores (ascending-k FMA chain): normwise tolerance vs exact."""
    a = W.smooth_field(256, 512, seed=43).numpy()
    b = W.smooth_field(512, 256, seed=44).numpy()
    A, B = dev.compress(torch.from_numpy(a).cuda()), dev.compress(torch.from_numpy(b).cuda())
    exact = dev.matmul_dense(A, B, mode=blz.GEMM_EXACT).cpu().numpy()
    fused = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED).cpu().numpy()
    err = np.max(np.abs(fused - exact)) / max(1.0, np.max(np.abs(exact)))
    assert err <= 1e-13 * 512, err
    assert np.array_equal(bits(fused), bits(dev.matmul_dense(A, B, mode=blz.GEMM_FUSED).cpu().numpy()))  # deterministic


@pytest.mark.parametrize("shape", [(256, 512, 256), (200, 333, 136), (8, 1000, 24)])
def test_matmul_fused_kernels_bitwise_equal(shape):
    """The two fused kernels (DFMA on CUDA cores, DMMA on FP64 tensor cores) compute
    the same ascending-k FMA chain: bitwise equal outputs, ragged shapes included,
    and BLZ_GEMM_FUSED is one of them."""
    m, k, n = shape
    A = dev.compress(W.rough_uniform(m, k, seed=45, device="cuda"))
    B = dev.compress(W.smooth_field(k, n, seed=46, device="cuda"))
    dmma = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED_DMMA).cpu().numpy()
    dfma = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED_DFMA).cpu().numpy()
    fused = dev.matmul_dense(A, B, mode=blz.GEMM_FUSED).cpu().numpy()
    assert np.array_equal(bits(dmma), bits(dfma))
    assert np.array_equal(bits(fused), bits(dfma))
    c_dmma = dev.matmul(A, B, mode=blz.GEMM_FUSED_DMMA)
    c_dfma = dev.matmul(A, B, mode=blz.GEMM_FUSED_DFMA)
    dev.sync()
    assert _equal_cmats(c_dmma, c_dfma)
    with pytest.raises(blz.InvalidArgument, match="bad mode"):
        dev.matmul_dense(A, B, mode=7)


@pytest.mark.parametrize("mode", [blz.GEMM_EXACT, blz.GEMM_FUSED])
@pytest.mark.parametrize("shape,panel", [((200, 333, 136), 4), ((64, 1000, 72), 8), ((40, 96, 48), 12)])
def test_matmul_panels_bitwise_equal_one_pass(shape, panel, mode, port):
    """K-paneled matmul (B decompressed panel by panel, accumulators continued) equals
    the one-pass product bitwise, compressed and dense, ragged K included; exact mode
    also equals the oracle."""
    m, k, n = shape
    A = dev.compress(W.smooth_field(m, k, seed=47, device="cuda"))
    B = dev.compress(W.rough_uniform(k, n, seed=48, device="cuda"))
    one = dev.matmul(A, B, mode=mode)
    pan = dev.matmul_panel(A, B, panel, mode=mode)
    d1 = dev.matmul_dense(A, B, mode=mode)
    d2 = dev.matmul_dense_panel(A, B, panel, mode=mode)
    dev.sync()
    assert _equal_cmats(one, pan)
    assert torch.equal(d1.view(torch.int64), d2.view(torch.int64))
    if mode == blz.GEMM_EXACT:
        want = port.mat_mul(A.to_host().blocks, m, k, B.to_host().blocks, k, n)
        assert blocks_equal(pan.to_host().blocks, want)
    with pytest.raises(blz.InvalidArgument, match="multiple of 4"):
        dev.matmul_panel(A, B, 3, mode=mode)


def test_device_calls_capture_into_cuda_graph():
    """The device API is stream-ordered and allocation-free after the first call, so a
    config-1-style op chain captures into a CUDA graph; replays equal eager calls."""
    rows, cols = 520, 776
    a = W.quadratic_blocks(rows, cols, seed=93, device="cuda")
    b = W.quadratic_blocks(rows, cols, seed=94, device="cuda")
    cA, cB, cS = dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols)
    cK = dev.ScaledCMat(cA)
    oS, oK = torch.empty_like(a), torch.empty_like(a)

    def chain():
        dev.compress(a, cA)
        dev.compress(b, cB)
        dev.sub(cA, cB, cS)
        dev.scale_meta(cA, -2.5, cK)
        dev.decompress(cS, oS)
        dev.decompress(cK, oK)

    def outputs():  # the SoA arrays and dense results (not the layout's padding bytes)
        return [getattr(m, f) for m in (cA, cB, cS, cK) for f in ("first", "slope", "scale", "coeffs")] + [oS, oK]

    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        chain()
    torch.cuda.synchronize()
    want = [x.clone() for x in outputs()]
    for x in outputs():
        x.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        chain()
    g.replay()
    torch.cuda.synchronize()
    for x, y in zip(outputs(), want):
        assert torch.equal(x.contiguous().view(torch.uint8), y.contiguous().view(torch.uint8))


# ---- .blzc container (H/io.hpp:93-134) --------------------------
@pytest.mark.parametrize("n", range(10))
def test_blzc_bytes_match_reference(golden, n):
    rows, cols = (int(v) for v in golden["shapes"][n])
    cm = blz.CompressedMatrix(rows, cols, golden[f"m{n}_ca"])
    data = blz.write_compressed(cm)
    assert data == golden[f"m{n}_blzc"].tobytes()            # byte-identical to the reference writer
    back = blz.read_compressed(data)
    assert (back.rows, back.cols) == (rows, cols)
    assert blocks_equal(back.blocks, cm.blocks)


def test_blzc_device_roundtrip_large():
    a = W.quadratic_blocks(2048, 2056, seed=51)
    A = dev.compress(a.cuda())
    ctx = dev.context()
    n = int(ctx.lib.blz_blzc_bytes(A.rows, A.cols))
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    import ctypes as C
    ctx.check(ctx.lib.blz_pack_blzc_dev(ctx.handle, A.ref(), C.c_void_p(buf.data_ptr())))
    B = dev.DeviceCMat(A.rows, A.cols)
    ctx.check(ctx.lib.blz_unpack_blzc_dev(ctx.handle, C.c_void_p(buf.data_ptr()), n, B.ref()))
    assert blocks_equal(B.to_host().blocks, A.to_host().blocks)
    assert buf.cpu().numpy().tobytes() == blz.write_compressed(A.to_host())


def test_blzc_errors_match_reference(golden):
    good = golden["m7_blzc"].tobytes()  # 40 x 56 -> 35 blocks
    cases = [
        (good[:5], "compressed matrix: truncated header"),
        (b"XLZC" + good[4:], r"compressed matrix: magic mismatch \(not a compressed matrix file\)"),
        (good[:4] + bytes([2]) + good[5:], "compressed matrix: unsupported version 2"),
        (good[:5] + bytes(4) + good[9:], "compressed matrix: zero dimension in header"),
        (good[:13 + 45 * 10 + 7], "compressed matrix: truncated at block 10"),
    ]
    zero_phi = bytearray(good)
    zero_phi[13 + 45 * 3 + 16] = 0
    cases.append((bytes(zero_phi), "compressed matrix: zero scale factor in block 3"))
    both = bytearray(zero_phi[:13 + 45 * 20])  # zero phi at block 3 reported before truncation at 20
    cases.append((bytes(both), "compressed matrix: zero scale factor in block 3"))
    for data, msg in cases:
        with pytest.raises(blz.IoError, match=msg):
            blz.read_compressed(data)
    bad = blz.CompressedMatrix(8, 8, golden["m1_ca"].copy())
    bad.blocks["slope"][0, 0] = np.inf
    with pytest.raises(blz.IoError, match="write_compressed: non-finite block field"):
        blz.write_compressed(bad)


@pytest.mark.parametrize("rows,cols", [(96, 128), (37, 53), (8, 8), (1, 200)])
def test_fused_op_decompress_matches_chain(port, rows, cols):
    """add/sub/scale -> decompress in one pass == the two-call chain, bitwise,
    including the s1 + s2 == 0 fallback, exact ties and huge weights."""
    a = torch.from_numpy(W.smooth_field(rows, cols, seed=31).numpy()).cuda()
    b = torch.from_numpy(np.random.default_rng(4).normal(size=(rows, cols))).cuda()
    ca, cb = dev.compress(a), dev.compress(b)
    others = [cb, ca, dev.scale(ca, -1.0), dev.scale(ca, -1.0000001), dev.scale(ca, 2.0)]
    for other in others:
        for fused, plain in ((dev.add_decompress, dev.add), (dev.sub_decompress, dev.sub)):
            out, dense = fused(ca, other)
            ref_c = plain(ca, other)
            ref_d = dev.decompress(ref_c)
            dev.sync()
            hc, hr = out.to_host().blocks, ref_c.to_host().blocks
            assert blocks_equal(hc, hr), block_diff_report(hc, hr)
            assert torch.equal(dense.view(torch.int64), ref_d.view(torch.int64))
    for k in (3.5, -1.0, 0.0, 1e-300):
        out, dense = dev.scale_decompress(ca, k)
        ref_c = dev.scale(ca, k)
        ref_d = dev.decompress(ref_c)
        dev.sync()
        assert blocks_equal(out.to_host().blocks, ref_c.to_host().blocks)
        assert torch.equal(dense.view(torch.int64), ref_d.view(torch.int64))
    # and against the oracle
    out, dense = dev.add_decompress(ca, cb)
    want = port.mat_add(ca.to_host().blocks.reshape(-1), cb.to_host().blocks.reshape(-1))
    assert blocks_equal(out.to_host().blocks.reshape(-1), want)
    wd = port.decompress_matrix(want, rows, cols)
    assert np.array_equal(bits(dense.cpu().numpy()), bits(wd))


def test_mean_relative_error_serial_order():
    """blz_mean_relative_error (H/bench.hpp:67-84) == the reference's serial loop, bitwise."""
    import ctypes as C
    rng = np.random.default_rng(8)
    n = 5000
    ref = rng.normal(size=n) * 10.0 ** rng.integers(-14, 3, size=n)
    ref[::17] = 0.0
    cand = ref * (1.0 + rng.normal(size=n) * 1e-6) + rng.normal(size=n) * 1e-9
    total, kept = 0.0, 0
    for r, c in zip(ref.tolist(), cand.tolist()):
        if abs(r) < 1e-12:
            continue
        total += abs((c - r) / r)
        kept += 1
    want = total / kept
    ctx = blz.default_context()
    mean, exc = C.c_double(), C.c_uint64()
    a, b = np.ascontiguousarray(ref), np.ascontiguousarray(cand)
    ctx.check(ctx.lib.blz_mean_relative_error(ctx.handle, a.ctypes.data, 50, 100, b.ctypes.data, 50, 100,
                                              C.byref(mean), C.byref(exc)))
    assert np.float64(mean.value).view(np.uint64) == np.float64(want).view(np.uint64)
    assert exc.value == n - kept
    with pytest.raises(blz.InvalidArgument, match="dimension mismatch"):
        ctx.check(ctx.lib.blz_mean_relative_error(ctx.handle, a.ctypes.data, 50, 100, b.ctypes.data, 100, 50,
                                                  C.byref(mean), C.byref(exc)))


def _equal_cmats(x, y):
    return all(torch.equal(getattr(x, f), getattr(y, f)) for f in ("first", "slope", "scale", "coeffs"))


@pytest.mark.parametrize("gen", ["quadratic", "rough"])
def test_full_size_properties(gen):
    """BASELINE config-1 size (16384^2, 4.19 M blocks): size-independent properties.

    * the verified fast compress equals the reference-order exact kernel on EVERY block;
    * the shared-product decompress equals the plain reference-order kernel bitwise;
    * add commutes bitwise; scale by 1 and by 2 then 0.5 are identities; A - A is zero;
    * the fused chains equal the two-call chains.
    """
    n = 16384
    a = W.make(gen, n, n, seed=71, device="cuda")
    b = W.make(gen, n, n, seed=72, device="cuda")
    dctx = dev.context()
    ca, cb = dev.compress(a), dev.compress(b)
    dctx.set_mode(blz.MODE_EXACT)
    try:
        ea = dev.compress(a)
        exact_dense = dev.decompress(ca)
        dev.sync()
    finally:
        dctx.set_mode(blz.MODE_DEFAULT)
    assert _equal_cmats(ca, ea)
    del a, b, ea
    fast_dense = dev.decompress(ca)
    dev.sync()
    assert torch.equal(fast_dense.view(torch.int64), exact_dense.view(torch.int64))
    del exact_dense
    assert _equal_cmats(dev.add(ca, cb), dev.add(cb, ca))
    assert _equal_cmats(dev.scale(ca, 1.0), ca)
    assert _equal_cmats(dev.scale(dev.scale(ca, 2.0), 0.5), ca)
    zero = dev.decompress(dev.sub(ca, ca))
    dev.sync()
    assert not bool(zero.any())
    del zero
    out, dense = dev.sub_decompress(ca, cb, dense=fast_dense)
    ref_c = dev.sub(ca, cb)
    ref_d = dev.decompress(ref_c)
    dev.sync()
    assert _equal_cmats(out, ref_c)
    assert torch.equal(dense.view(torch.int64), ref_d.view(torch.int64))


def _nccl_comm_single_gpu():
    """A one-rank NCCL communicator on cuda:0 (ncclCommInitAll via ctypes)."""
    import ctypes as C
    try:
        lib = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    except OSError:
        pytest.skip("libnccl.so.2 not loadable")
    comm = C.c_void_p()
    devs = (C.c_int * 1)(0)
    assert lib.ncclCommInitAll(C.byref(comm), 1, devs) == 0
    return lib, comm


def test_nccl_sharded_entry_points_one_rank():
    """The NCCL C-ABI variants with G = 1 equal the local operations bitwise
    (rank/row-range logic is shared with shard.py, covered by the gloo tests)."""
    import ctypes as C
    lib_nccl, comm = _nccl_comm_single_gpu()
    ctx = dev.context()
    lib = ctx.lib
    n = 1000
    a = dev.compress(torch.from_numpy(W.smooth_field(n, 776, seed=5).numpy()).cuda())
    b = dev.compress(torch.from_numpy(W.smooth_field(n, 776, seed=6).numpy()).cuda())
    # config 2: gathered row dots + ascending total
    r_all = torch.empty(n, dtype=torch.float64, device="cuda")
    tot = torch.empty(1, dtype=torch.float64, device="cuda")
    ctx.check(lib.blz_rowdot_frobenius_nccl(ctx.handle, comm, a.ref(), b.ref(), n, C.c_void_p(r_all.data_ptr()),
                                            C.c_void_p(tot.data_ptr())))
    r_ref, t_ref = dev.frobenius(a, b)
    dev.sync()
    assert torch.equal(r_all.view(torch.int64), r_ref.view(torch.int64))
    assert torch.equal(tot.view(torch.int64), t_ref.view(torch.int64))
    # allgather of a compressed matrix (one shard = the whole matrix)
    full = dev.DeviceCMat(n, 776)
    ctx.check(lib.blz_allgather_cmat_nccl(ctx.handle, comm, a.ref(), full.ref()))
    dev.sync()
    assert all(torch.equal(getattr(full, f), getattr(a, f)) for f in ("first", "slope", "coeffs", "scale"))
    # config 4: matmul with the gathered B (B^T-shaped second operand)
    bt = dev.compress(torch.from_numpy(W.smooth_field(776, n, seed=7).numpy()).cuda())
    b_full = dev.DeviceCMat(776, n)
    scratch = dev.matmul_scratch(a, b_full)
    c_sh = dev.DeviceCMat(n, n)
    ctx.check(lib.blz_matmul_nccl(ctx.handle, comm, a.ref(), bt.ref(), b_full.ref(), 0,
                                  C.c_void_p(scratch.data_ptr()), c_sh.ref()))
    c_ref = dev.matmul(a, bt, mode=0)
    dev.sync()
    assert all(torch.equal(getattr(c_sh, f), getattr(c_ref, f)) for f in ("first", "slope", "coeffs", "scale"))
    lib_nccl.ncclCommDestroy(comm)


def _np_decompress(blocks, basis, rows, cols):
    """decompress_matrix (H/matrix.hpp:113-126) restated over numpy arrays of blocks with an
    arbitrary basis: dequantize_prediction (H/codec.hpp:150-158, the full 8x8 grid with the
    discarded positions as zeros), idct2 (H/dct.hpp:53-70, every product and sum rounded in
    the reference's order), integrate_rows (H/codec.hpp:164-174).  Vectorised over blocks;
    each array op is one IEEE binary64 operation per block."""
    b = blocks.reshape(-1)
    n = b.shape[0]
    t = np.asarray(basis, np.float64).reshape(8, 8)
    s = b["slope"]
    d = np.zeros((n, 8, 8))
    pos = [(0, c) for c in range(8)] + [(1, c) for c in range(8)] + [(r, 0) for r in range(2, 8)] + \
          [(r, 1) for r in range(2, 8)]
    phi = b["scale_factor"].astype(np.float64)
    for k, (r, c) in enumerate(pos):
        d[:, r, c] = b["coeffs"][:, k].astype(np.float64) / phi
    d[s == 0.0] = 0.0
    tmp = np.zeros((n, 8, 8))
    for u in range(8):
        for j in range(8):
            acc = np.zeros(n)
            for i in range(8):
                acc = acc + t[i, u] * d[:, i, j]
            tmp[:, u, j] = acc
    x = np.zeros((n, 8, 8))
    for u in range(8):
        for v in range(8):
            acc = np.zeros(n)
            for j in range(8):
                acc = acc + tmp[:, u, j] * t[j, v]
            x[:, u, v] = acc
    out = np.zeros((n, 8, 8))
    out[:, 0, 0] = b["first"]
    for j in range(1, 8):
        out[:, 0, j] = out[:, 0, j - 1] + s * x[:, 0, j]
    for i in range(1, 8):
        out[:, i, 0] = out[:, i - 1, 0] + s * x[:, i, 0]
        for j in range(1, 8):
            out[:, i, j] = (out[:, i - 1, j] + out[:, i, j - 1]) / 2.0 + s * x[:, i, j]
    br, bc = (rows + 7) // 8, (cols + 7) // 8
    return out.reshape(br, bc, 8, 8).transpose(0, 2, 1, 3).reshape(br * 8, bc * 8)[:rows, :cols]


@pytest.mark.parametrize("rows,cols", [(8, 8), (5, 3), (13, 8), (8, 21), (203, 141), (64, 1000), (1001, 64)])
def test_decompress_uniform_basis_kernel_crops(port, rows, cols):
    """k_decompress_ub stores the blocks fully inside the crop; k_decompress_edges the
    partial last block-row / block-column.  Device API, contiguous and strided outputs."""
    a = W.smooth_field(rows, cols, seed=rows * 7 + cols).numpy()
    a[: min(rows, 8), : min(cols, 8)] = 0.0  # a constant (s == 0) block
    cm = blz.compress_matrix(a)
    want = port.decompress_matrix(cm.blocks.reshape(-1), rows, cols)
    dcm = dev.DeviceCMat.from_host(cm)
    got = dev.decompress(dcm)
    wide = torch.full((rows, cols + 6), 7.0, dtype=torch.float64, device="cuda")  # ld = cols + 6
    dev.decompress(dcm, out=wide[:, :cols])
    odd = torch.full((rows, cols + 1), 7.0, dtype=torch.float64, device="cuda")  # ld odd: not 16-B aligned rows
    dev.decompress(dcm, out=odd[:, :cols])
    dev.sync()
    for g in (got, wide[:, :cols], odd[:, :cols]):
        assert np.array_equal(bits(g.cpu().numpy()), bits(want))
    assert torch.all(wide[:, cols:] == 7.0) and torch.all(odd[:, cols:] == 7.0)
    assert np.array_equal(bits(_np_decompress(cm.blocks, port.dct_basis(), rows, cols)), bits(want))


def test_decompress_context_with_other_basis():
    """A context whose basis is not the device's bound constant basis runs the
    per-thread-operand kernel, with its own basis; the default context is unaffected."""
    import ctypes as C

    base = blz.default_context()
    t = np.empty(64)
    base.check(base.lib.blz_ctx_basis(base.handle, t.ctypes.data_as(C.c_void_p)))
    other = t.copy()
    other[5 * 8 + 3] = np.nextafter(other[5 * 8 + 3], 1.0)
    other[6 * 8 + 6] *= 1.0 + 2.0 ** -40
    ctx2 = blz.Context(basis=other)
    try:
        a = W.smooth_field(96, 80, seed=11).numpy()
        cm = blz.compress_matrix(a)
        got2 = blz.decompress_matrix(cm, ctx=ctx2)
        got1 = blz.decompress_matrix(cm)
        assert np.array_equal(bits(got2), bits(_np_decompress(cm.blocks, other, 96, 80)))
        assert np.array_equal(bits(got1), bits(_np_decompress(cm.blocks, t, 96, 80)))
        assert not np.array_equal(bits(got1), bits(got2))
    finally:
        ctx2.close()
