"""The `blaz` command-line tool (tools/cli/blaz.cpp).

CPU: usage / argument / I/O exit codes and `gen` (host sampling, glibc math).
GPU: every matrix subcommand against the reference's golden vectors, byte for
byte on the .blzc / .blzd files (tests/golden/golden.npz holds the reference's
own .blzc bytes and results).
"""
import ctypes
import math
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "cli", "blaz")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="tools/cli/blaz not built")


def run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def write_blzd(path, m):
    m = np.ascontiguousarray(m, np.float64)
    with open(path, "wb") as f:
        f.write(b"BLZD" + bytes([1]) + struct.pack("<II", *m.shape) + m.tobytes())


def read_blzd(path):
    b = open(path, "rb").read()
    assert b[:5] == b"BLZD\x01"
    r, c = struct.unpack("<II", b[5:13])
    return np.frombuffer(b[13:], np.float64).reshape(r, c)


def blzc_bytes(blocks, rows, cols):
    blocks = np.ascontiguousarray(blocks).reshape(-1)
    out = bytearray(b"BLZC" + bytes([1]) + struct.pack("<II", rows, cols))
    for bl in blocks:
        out += struct.pack("<dd", float(bl["first"]), float(bl["slope"]))
        out += bytes([int(bl["scale_factor"])]) + np.asarray(bl["coeffs"], np.int8).tobytes()
    return bytes(out)


def test_usage_errors(tmp_path):
    assert run()[0] == 1
    assert run("frobnicate")[0] == 1
    assert run("compress")[0] == 1  # missing input and output
    assert run("--bogus", "info", "x")[0] == 1
    assert run("accuracy", "-n", "1", "-o", str(tmp_path / "a.csv"))[0] == 3
    assert run("bench", "--repeats", "4", "-o", str(tmp_path / "b.csv"))[0] == 3
    assert run("bench", "--ops", "frob", "-o", str(tmp_path / "b.csv"))[0] == 3
    code, out, _ = run("--help")
    assert code == 0 and "compress" in out


def test_gen_matches_glibc_sampling(tmp_path):
    libm = ctypes.CDLL("libm.so.6")
    for name in ("cos", "sqrt", "exp"):
        getattr(libm, name).restype = ctypes.c_double
        getattr(libm, name).argtypes = [ctypes.c_double]
    fns = {
        "f1": lambda x, y: x * y,
        "f2": lambda x, y: x * y / (1.0 + x * x + y * y),
        "f3": lambda x, y: x * x - y,
        "f4": lambda x, y: (x * x) * (y * y),
        "f5": lambda x, y: libm.cos(libm.sqrt(x * x + y * y)),
        "f6": lambda x, y: libm.cos(x * x + y * y) * libm.exp(-0.1 * (x * x + y * y)),
    }
    n = 13
    nodes = [-2.0 + 4.0 * j / (n - 1) for j in range(n)]
    for fid, f in fns.items():
        path = tmp_path / f"{fid}.blzd"
        assert run("gen", fid, str(n), "-o", str(path))[0] == 0
        got = read_blzd(path)
        want = np.array([[f(nodes[j], nodes[i]) for j in range(n)] for i in range(n)])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), fid
    # argument errors: exit 3; existing output without --force: exit 2
    assert run("gen", "f7", "8", "-o", str(tmp_path / "x.blzd"))[0] == 3
    assert run("gen", "f1", "1", "-o", str(tmp_path / "x.blzd"))[0] == 3
    assert run("gen", "f1", "8", "-o", str(tmp_path / "f1.blzd"))[0] == 2
    assert run("--force", "gen", "f1", "8", "-o", str(tmp_path / "f1.blzd"))[0] == 0
    assert not any(p.name.endswith(".tmp") for p in tmp_path.iterdir())


def test_missing_input_is_io_error(tmp_path):
    assert run("decompress", str(tmp_path / "nope.blzc"), "-o", str(tmp_path / "o.blzd"))[0] == 2


@pytest.mark.gpu
@pytest.mark.parametrize("n", [3, 9])  # each call pays a CUDA context start-up
def test_matrix_commands_match_reference(golden, tmp_path, n):
    rows, cols = (int(v) for v in golden["shapes"][n])
    g = lambda k: golden[f"m{n}_{k}"]  # noqa: E731
    a, b = tmp_path / "a.blzd", tmp_path / "b.blzd"
    write_blzd(a, g("a"))
    write_blzd(b, g("b"))
    ca, cb = tmp_path / "a.blzc", tmp_path / "b.blzc"
    assert run("compress", str(a), "-o", str(ca))[0] == 0
    assert run("compress", str(b), "-o", str(cb))[0] == 0
    assert open(ca, "rb").read() == g("blzc").tobytes()  # the reference's own .blzc bytes
    assert open(cb, "rb").read() == blzc_bytes(g("cb"), rows, cols)
    d = tmp_path / "a_d.blzd"
    assert run("decompress", str(ca), "-o", str(d))[0] == 0
    assert np.array_equal(read_blzd(d).view(np.uint64), g("da").view(np.uint64))
    for cmd, key in (("add", "add"), ("sub", "sub")):
        o = tmp_path / f"{cmd}.blzc"
        assert run(cmd, str(ca), str(cb), "-o", str(o))[0] == 0
        assert open(o, "rb").read() == blzc_bytes(g(key), rows, cols)
    o = tmp_path / "scale.blzc"
    assert run("scale", str(ca), "3.5", "-o", str(o))[0] == 0
    assert open(o, "rb").read() == blzc_bytes(g("scale"), rows, cols)
    # dot / matmul against B^T (cols x rows), as the fixtures were made
    bt = tmp_path / "bt.blzd"
    write_blzd(bt, np.ascontiguousarray(g("b").T))
    cbt = tmp_path / "bt.blzc"
    assert run("compress", str(bt), "-o", str(cbt))[0] == 0
    for q, (i, j) in list(enumerate(zip(g("qi"), g("qj"))))[:2]:
        code, out, _ = run("dot", str(ca), str(cbt), str(int(i)), str(int(j)))
        assert code == 0
        assert np.float64(float(out)).view(np.uint64) == np.float64(g("dot")[q]).view(np.uint64)
    o = tmp_path / "mul.blzc"
    assert run("matmul", str(ca), str(cbt), "-o", str(o))[0] == 0
    assert open(o, "rb").read() == blzc_bytes(g("mul"), rows, rows)
    if n == 3:  # the harness subcommands (GPU mean_relative_error, timing)
        acc = tmp_path / "acc.csv"
        assert run("accuracy", "-n", "24", "-o", str(acc))[0] == 0
        lines = acc.read_text().splitlines()
        assert lines[0] == "op,lhs,rhs,n,error,excluded" and len(lines) == 64
        bench = tmp_path / "bench.csv"
        assert run("bench", "--sizes", "16", "--ops", "add,compress", "-o", str(bench))[0] == 0
        assert bench.read_text().splitlines()[0] == "op,n,variant,seconds"
    code, out, _ = run("info", str(ca))
    assert code == 0 and f"dimensions:       {rows} x {cols}" in out
    # errors: dimension mismatch -> 3, out-of-range dot -> 3, corrupt file -> 2
    if rows != cols:
        assert run("add", str(ca), str(cbt), "-o", str(tmp_path / "bad.blzc"))[0] == 3
    assert run("dot", str(ca), str(cbt), str(rows), "0")[0] == 3
    bad = tmp_path / "bad.blzc"
    bad.write_bytes(b"BLZX" + open(ca, "rb").read()[4:])
    assert run("info", str(bad))[0] == 2
