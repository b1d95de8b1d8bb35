"""Pins the C restatement (oracle/blaz_oracle.c) before it is trusted.

(1) The reference's own known-answer vectors: the ramp block i*j/100
    (proj/tests/test_util.hpp:28-54; PAPER.md Example 1) -- s == 0.04
    bit-exact (codec_test.cpp:71-74), all 64 quantizer indices
    (codec_test.cpp:103-113), phi == 20 and C within +-2 of the published grid
    (codec_test.cpp:182-210); constant blocks (:212-218, :276-280).
(2) tests/golden/golden.npz, produced by the REAL reference headers compiled
    under oracle/_ref (tests/golden/make_golden.py): bit-for-bit equality.
"""
import numpy as np
import pytest

from conftest import bits, block_diff_report, blocks_equal

RAMP_INDICES = [
    [125, 125, 125, 125, 125, 125, 125, 125],
    [125, 143, 153, 162, 171, 180, 189, 198],
    [125, 153, 162, 171, 180, 189, 198, 207],
    [125, 162, 171, 180, 189, 198, 207, 217],
    [125, 171, 180, 189, 198, 207, 217, 226],
    [125, 180, 189, 198, 207, 217, 226, 235],
    [125, 189, 198, 207, 217, 226, 235, 244],
    [125, 198, 207, 217, 226, 235, 244, 253],
]
RAMP_COEFF_GRID = [
    [122, -51, -11, -14, -8, -8, -4, -2],
    [-51, 15, 7, 7, 5, 4, 3, 1],
    [-11, 7, 0, 0, 0, 0, 0, 0],
    [-14, 7, 0, 1, 0, 0, 0, 0],
    [-8, 5, 0, 0, 0, 0, 0, 0],
    [-8, 4, 0, 0, 0, 0, 0, 0],
    [-4, 3, 0, 0, 0, 0, 0, 0],
    [-2, 1, 0, 0, 0, 0, 0, 0],
]
KEEP = [(0, c) for c in range(8)] + [(1, c) for c in range(8)] + [(r, 0) for r in range(2, 8)] + \
       [(r, 1) for r in range(2, 8)]


def ramp():
    return np.fromfunction(lambda i, j: (i * j) / 100.0, (8, 8))


def test_ramp_known_answers(port):
    first, deltas = port.normalize(ramp())
    assert first == 0.0
    s = port.mean_slope(deltas)
    assert np.float64(s).view(np.uint64) == np.float64(0.04).view(np.uint64)
    idx, _ = port.predict(deltas / s, s)
    assert idx.tolist() == RAMP_INDICES
    cb = port.compress_block(ramp())
    assert cb["scale_factor"] == 20
    assert np.float64(cb["slope"]).view(np.uint64) == np.float64(0.04).view(np.uint64)
    for k, (r, c) in enumerate(KEEP):
        assert abs(int(cb["coeffs"][k]) - RAMP_COEFF_GRID[r][c]) <= 2
    back = port.decompress_block(cb)
    assert np.max(np.abs(back - ramp())) <= 0.02  # codec_test.cpp:268-274


def test_constant_blocks(port):
    cb = port.compress_block(np.full((8, 8), 7.5))
    assert cb["first"] == 7.5 and cb["slope"] == 0.0 and cb["scale_factor"] == 1
    assert not cb["coeffs"].any()
    a = np.full((8, 8), -3.75)
    assert np.array_equal(bits(port.decompress_block(port.compress_block(a))), bits(a))


def test_rounding_rule(port):
    # H/block.hpp:61-67: halfway cases away from zero
    for x, want in [(0.5, 1.0), (-0.5, -1.0), (1.49999, 1.0), (2.5, 3.0), (-2.5, -3.0), (0.0, 0.0)]:
        assert port.round_half_away(x) == want


def test_basis_matches_reference(port, golden):
    assert np.array_equal(bits(port.dct_basis()), bits(golden["basis"]))


def test_blocks_match_reference(port, golden):
    tiles = golden["tiles"]
    got = np.array([port.compress_block(t) for t in tiles], golden["tiles_c"].dtype)
    assert blocks_equal(got, golden["tiles_c"]), block_diff_report(got, golden["tiles_c"])
    dec = np.stack([port.decompress_block(b) for b in golden["tiles_c"]])
    assert np.array_equal(bits(dec), bits(golden["tiles_d"]))
    idx, _ = port.predict(*_slopes(port, tiles[0]))
    assert np.array_equal(idx, golden["ramp_idx"])


def _slopes(port, t):
    _, d = port.normalize(t)
    s = port.mean_slope(d)
    return d / s, s


def test_pairs_match_reference(port, golden):
    pa, pb = golden["pair_a"], golden["pair_b"]
    add = np.array([port.add(a, b) for a, b in zip(pa, pb)], pa.dtype)
    sub = np.array([port.sub(a, b) for a, b in zip(pa, pb)], pa.dtype)
    assert blocks_equal(add, golden["pair_add"]), block_diff_report(add, golden["pair_add"])
    assert blocks_equal(sub, golden["pair_sub"]), block_diff_report(sub, golden["pair_sub"])


@pytest.mark.parametrize("n", range(10))
def test_matrices_match_reference(port, golden, n):
    rows, cols = (int(v) for v in golden["shapes"][n])
    g = lambda k: golden[f"m{n}_{k}"]  # noqa: E731
    ca = port.compress_matrix(g("a"))
    assert blocks_equal(ca, g("ca"))
    assert np.array_equal(bits(port.decompress_matrix(g("ca"), rows, cols)), bits(g("da")))
    assert blocks_equal(port.mat_add(g("ca"), g("cb")), g("add"))
    assert blocks_equal(port.mat_sub(g("ca"), g("cb")), g("sub"))
    assert blocks_equal(port.mat_scale(g("ca"), 3.5), g("scale"))
    assert blocks_equal(port.mat_mul(g("ca"), rows, cols, g("cbt"), cols, rows), g("mul"))
    assert np.array_equal(bits(port.mat_mul_dense(g("ca"), rows, cols, g("cbt"), cols, rows)), bits(g("muld")))
    dots = [port.mat_dot(g("ca"), rows, cols, g("cbt"), cols, rows, int(i), int(j))
            for i, j in zip(g("qi"), g("qj"))]
    assert np.array_equal(bits(np.array(dots)), bits(g("dot")))
    r = port.rowdot(g("ca"), g("cb"), rows, cols)
    assert np.array_equal(bits(r), bits(g("rowdot")))
    assert np.float64(port.sum_ascending(r)).view(np.uint64) == np.float64(g("frob")).view(np.uint64)


def test_oracle_errors(port):
    from oracle.oracle import OracleError
    bad = np.ones((8, 8))
    bad[3, 3] = np.nan
    with pytest.raises(OracleError):
        port.compress_block(bad)
    with pytest.raises(OracleError):
        port.mat_scale(np.zeros(1, port.compress_matrix(np.ones((8, 8))).dtype), float("inf"))


def test_markstein_dequant_exhaustive():
    """C/phi == RN(q + RN? ...) -- the decompress dequantization (blaz_device.cuh::dequant):
    r = RN(1/phi), q = RN(C*r), e = fma(-phi, q, C), result = fma(e, r, q) equals the IEEE
    quotient C/phi for every C in [-128, 127] and phi in [1, 255] (fma emulated exactly)."""
    from fractions import Fraction as F
    bad = 0
    for phi in range(1, 256):
        r = 1.0 / phi
        fr = F(r)
        for c in range(-128, 128):
            q = c * r                                 # DMUL, correctly rounded
            e = float(F(c) - phi * F(q))              # fma(-phi, q, c): one rounding
            res = float(F(e) * fr + F(q))             # fma(e, r, q): one rounding
            if res != c / phi:
                bad += 1
    assert bad == 0


def test_fp32_scale_factor_merge_is_exact():
    """csrc/blaz_device.cuh::merge_scale_factor_u8 computes floor(p1 p2 / (p1 + p2))
    (H/block_ops.hpp:12-15) with one approximate fp32 division: every (p1, p2) in
    [0, 255]^2, with the quotient perturbed by up to 2 ulp either way (the
    documented error of __fdividef), floors to the integer quotient."""
    p1, p2 = np.meshgrid(np.arange(256, dtype=np.int64), np.arange(256, dtype=np.int64))
    N, D = p1 * p2, p1 + p2
    ok = D > 0
    exact = N // np.maximum(D, 1)
    q = N.astype(np.float32) / np.maximum(D, 1).astype(np.float32)
    for ulps in (-2, -1, 0, 1, 2):
        qq = q.copy()
        for _ in range(abs(ulps)):
            qq = np.nextafter(qq, np.float32(np.inf) if ulps > 0 else np.float32(-np.inf))
        got = np.trunc((qq + np.float32(1.0 / 1024.0)).astype(np.float32)).astype(np.int64)
        assert not np.any((got != exact) & ok), ulps
