"""Generates tests/golden/golden.npz from the REAL reference.

Runs the reference headers compiled under oracle/_ref (oracle/ref_shim.cpp ->
/root/reference/proj/include/blaz, -O2 -ffp-contract=off) on seeded inputs and
stores inputs + outputs.  The fixtures pin both the C restatement
(oracle/blaz_oracle.c, tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_parity.py) on machines where /root/reference is absent.

    python tests/golden/make_golden.py       # needs oracle/_ref/libblaz_ref.so
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def smooth_block(rng):
    # same family as the reference's random_smooth_block (proj/tests/test_util.hpp:71-82)
    s = 10.0 ** rng.uniform(-3, 3)
    c = rng.uniform(-1, 1, 6)
    x = np.arange(8) / 7.0
    X, Y = np.meshgrid(x, x)
    return s * (c[0] + c[1] * X + c[2] * Y + c[3] * X * X + c[4] * Y * Y + c[5] * X * Y
                + rng.uniform(-0.02, 0.02, (8, 8)))


def special_blocks():
    out = []
    out.append(np.fromfunction(lambda i, j: i * j / 100.0, (8, 8)))  # ramp (PAPER Example 1)
    out.append(np.full((8, 8), 7.5))
    out.append(np.full((8, 8), -3.75))
    out.append(np.zeros((8, 8)))
    out.append(np.fromfunction(lambda i, j: j * 1.0, (8, 8)))
    one = np.zeros((8, 8)); one[4, 2] = -0.5; out.append(one)
    out.append(np.fromfunction(lambda i, j: (i + j) * 1e-300, (8, 8)))
    out.append(np.fromfunction(lambda i, j: (i - 2 * j) * 1e200, (8, 8)))
    out.append(np.fromfunction(lambda i, j: 1e18 + (i + j) * 1e17, (8, 8)))
    out.append(np.fromfunction(lambda i, j: 5e18 * (i * 8 + j), (8, 8)))
    out.append(np.fromfunction(lambda i, j: (-1.0) ** (i + j), (8, 8)))
    out.append(np.fromfunction(lambda i, j: np.where((i + j) % 3 == 0, 1.0, 0.0), (8, 8)))
    return out


def main():
    r = O.ref()
    rng = np.random.default_rng(20220226)
    g = {}
    g["basis"] = r.dct_basis()

    blocks = special_blocks()
    n_special = len(blocks)
    blocks += [smooth_block(rng) for _ in range(400)]
    blocks += [rng.uniform(-100, 100, (8, 8)) for _ in range(150)]
    blocks += [np.round(rng.uniform(-5, 5, (8, 8))) for _ in range(50)]
    tiles = np.stack(blocks).astype(np.float64)
    g["tiles"] = tiles
    g["n_special"] = np.array(n_special)
    comp = np.zeros(len(tiles), O.BLOCK_DTYPE)
    dec = np.zeros_like(tiles)
    for k, t in enumerate(tiles):
        comp[k] = r.compress_block(t)
        dec[k] = r.decompress_block(comp[k])
    g["tiles_c"] = comp
    g["tiles_d"] = dec
    g["ramp_idx"] = r.predict_indices(tiles[0])

    # add / sub pairs, including the fast paths and the s1+s2 == 0 fallback
    idx_a = rng.integers(0, len(comp), 300)
    idx_b = rng.integers(0, len(comp), 300)
    pa = comp[idx_a].copy()
    pb = comp[idx_b].copy()
    neg = pa[:20].copy()
    neg["first"] *= -1.0
    neg["slope"] *= -1.0  # scale(a, -1): opposite slopes -> dense fallback
    pa = np.concatenate([pa, pa[:20], pa[:10]])
    pb = np.concatenate([pb, neg, pa[:10]])
    g["pair_a"], g["pair_b"] = pa, pb
    g["pair_add"] = np.array([r.add(a, b) for a, b in zip(pa, pb)], O.BLOCK_DTYPE)
    g["pair_sub"] = np.array([r.sub(a, b) for a, b in zip(pa, pb)], O.BLOCK_DTYPE)

    # matrix cases (smooth and quadratic fields, ragged shapes)
    shapes = [(1, 1), (8, 8), (9, 9), (9, 17), (16, 16), (20, 12), (24, 24), (40, 56), (64, 48), (33, 65)]
    for n, (rows, cols) in enumerate(shapes):
        x = np.arange(cols) / max(cols, 1)
        y = np.arange(rows) / max(rows, 1)
        X, Y = np.meshgrid(x, y)
        c = rng.uniform(-1, 1, 4)
        a = c[0] + c[1] * X + c[2] * Y + c[3] * X * Y + rng.uniform(-0.05, 0.05, (rows, cols))
        b = np.sin(3 * X + 2 * Y) + rng.uniform(-0.05, 0.05, (rows, cols))
        ca = r.compress_matrix(a)
        cb = r.compress_matrix(b)
        g[f"m{n}_a"], g[f"m{n}_b"] = a, b
        g[f"m{n}_ca"], g[f"m{n}_cb"] = ca, cb
        g[f"m{n}_da"] = r.decompress_matrix(ca, rows, cols)
        g[f"m{n}_add"] = r.mat_add(ca, cb, rows, cols)
        g[f"m{n}_sub"] = r.mat_sub(ca, cb, rows, cols)
        g[f"m{n}_scale"] = r.mat_scale(ca, rows, cols, 3.5)
        # A (rows x cols) * B^T-shaped operand (cols x rows) via a second compress
        bt = np.ascontiguousarray(b.T)
        cbt = r.compress_matrix(bt)
        g[f"m{n}_cbt"] = cbt
        g[f"m{n}_mul"] = r.mat_mul(ca, rows, cols, cbt, cols, rows)
        g[f"m{n}_muld"] = r.mat_mul_dense(ca, rows, cols, cbt, cols, rows)
        qi = rng.integers(0, rows, 8)
        qj = rng.integers(0, rows, 8)
        g[f"m{n}_qi"], g[f"m{n}_qj"] = qi, qj
        g[f"m{n}_dot"] = np.array([r.mat_dot(ca, rows, cols, cbt, cols, rows, int(i), int(j))
                                   for i, j in zip(qi, qj)])
        # config-2 restatement from reference decompressions: ascending row sums
        da = r.decompress_matrix(ca, rows, cols)
        db = r.decompress_matrix(cb, rows, cols)
        rd = np.zeros(rows)
        for i in range(rows):
            acc = 0.0
            for j in range(cols):
                acc = acc + float(da[i, j]) * float(db[i, j])
            rd[i] = acc
        tot = 0.0
        for v in rd:
            tot = tot + float(v)
        g[f"m{n}_rowdot"], g[f"m{n}_frob"] = rd, np.array(tot)
        # .blzc container bytes written by the reference (H/io.hpp:96-111)
        g[f"m{n}_blzc"] = np.frombuffer(r.write_compressed(ca, rows, cols), np.uint8)
    g["shapes"] = np.array(shapes)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
