"""CPU ORACLE bindings (test infrastructure only).

ctypes wrappers over
  * ``oracle/liboracle.so``       -- the plain-C restatement (``blaz_oracle.c``), and
  * ``oracle/_ref/libblaz_ref.so`` -- the real reference headers compiled from
    /root/reference (``ref_shim.cpp``), present only where it was built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker.
The product package (``paper_2202_13007_b200``) never imports it.

Blocks are exchanged as numpy structured arrays with the reference's 48-byte
in-memory layout of ``blaz::compressed_block`` (H/block.hpp:33-38).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libblaz_ref.so")

BLOCK_DTYPE = np.dtype(
    {"names": ["first", "slope", "scale_factor", "coeffs"],
     "formats": ["<f8", "<f8", "u1", ("i1", 28)],
     "offsets": [0, 8, 16, 17], "itemsize": 48})

_P = C.c_void_p
_SZ = C.c_size_t


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/include")
    if ref:
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def _nb(n: int) -> int:
    return (n + 7) // 8


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name, restype=C.c_int, argtypes=()):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        f.argtypes = list(argtypes)
        return f


class Port:
    """The C restatement (scalar, single thread)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = _Lib(path, "orc_")
        self.lib = L.lib
        self._basis = L.fn("dct_basis", None, [_P])
        self._cb = L.fn("compress_block", C.c_int, [_P, _P])
        self._db = L.fn("decompress_block", None, [_P, _P])
        self._add = L.fn("add", C.c_int, [_P, _P, _P])
        self._sub = L.fn("sub", C.c_int, [_P, _P, _P])
        self._dot = L.fn("dot", C.c_double, [_P, _P, C.c_int, C.c_int])
        self._norm = L.fn("normalize", C.c_int, [_P, _P, _P])
        self._mean = L.fn("mean_slope", C.c_double, [_P])
        self._pred = L.fn("predict", None, [_P, C.c_double, _P, _P])
        self._rha = L.fn("round_half_away", C.c_double, [C.c_double])
        self._cm = L.fn("compress_matrix", C.c_int, [_P, _SZ, _SZ, _P])
        self._dm = L.fn("decompress_matrix", None, [_P, _SZ, _SZ, _P])
        self._madd = L.fn("mat_add", C.c_int, [_P, _P, _SZ, _P])
        self._msub = L.fn("mat_sub", C.c_int, [_P, _P, _SZ, _P])
        self._mscale = L.fn("mat_scale", C.c_int, [_P, C.c_double, _SZ, _P])
        self._mdot = L.fn("mat_dot", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P])
        self._mmd = L.fn("mat_mul_dense", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _P])
        self._mm = L.fn("mat_mul", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _P])
        self._rowdot = L.fn("rowdot", C.c_int, [_P, _P, _SZ, _SZ, _P])
        self._rrows = L.fn("reconstruct_rows", None, [_P, C.c_int, _P])
        self._rcols = L.fn("reconstruct_cols", None, [_P, C.c_int, _P])
        self._bmul = L.fn("block_mul", None, [_P, _P, _P])
        self._sum = L.fn("sum_ascending", C.c_double, [_P, _SZ])

    # block level
    def dct_basis(self) -> np.ndarray:
        t = np.zeros(64, np.float64)
        self._basis(_ptr(t))
        return t

    def compress_block(self, m) -> np.ndarray:
        m = np.ascontiguousarray(m, np.float64).reshape(64)
        out = np.zeros(1, BLOCK_DTYPE)
        st = self._cb(_ptr(m), _ptr(out))
        if st:
            raise OracleError(st)
        return out[0]

    def decompress_block(self, b) -> np.ndarray:
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(64, np.float64)
        self._db(_ptr(b), _ptr(out))
        return out.reshape(8, 8)

    def normalize(self, m):
        m = np.ascontiguousarray(m, np.float64).reshape(64)
        f = np.zeros(1, np.float64)
        d = np.zeros(64, np.float64)
        st = self._norm(_ptr(m), _ptr(f), _ptr(d))
        if st:
            raise OracleError(st)
        return float(f[0]), d.reshape(8, 8)

    def mean_slope(self, d) -> float:
        d = np.ascontiguousarray(d, np.float64).reshape(64)
        return self._mean(_ptr(d))

    def predict(self, slopes, s):
        slopes = np.ascontiguousarray(slopes, np.float64).reshape(64)
        idx = np.zeros(64, np.uint8)
        snapped = np.zeros(64, np.float64)
        self._pred(_ptr(slopes), C.c_double(s), _ptr(idx), _ptr(snapped))
        return idx.reshape(8, 8), snapped.reshape(8, 8)

    def round_half_away(self, x: float) -> float:
        return self._rha(x)

    def add(self, a, b):
        return self._binop(self._add, a, b)

    def sub(self, a, b):
        return self._binop(self._sub, a, b)

    def _binop(self, f, a, b):
        a = np.array([a], BLOCK_DTYPE)
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(1, BLOCK_DTYPE)
        st = f(_ptr(a), _ptr(b), _ptr(out))
        if st:
            raise OracleError(st)
        return out[0]

    def dot(self, a, b, i, j) -> float:
        a = np.array([a], BLOCK_DTYPE)
        b = np.array([b], BLOCK_DTYPE)
        return self._dot(_ptr(a), _ptr(b), i, j)

    def reconstruct_rows(self, b, last_row: int) -> np.ndarray:
        """partial_reconstruction.values (H/block_ops.hpp:87-95): rows > last_row stay +0.0."""
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(64, np.float64)
        self._rrows(_ptr(b), last_row, _ptr(out))
        return out.reshape(8, 8)

    def reconstruct_cols(self, b, last_col: int) -> np.ndarray:
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(64, np.float64)
        self._rcols(_ptr(b), last_col, _ptr(out))
        return out.reshape(8, 8)

    def block_mul(self, a, b) -> np.ndarray:
        a = np.array([a], BLOCK_DTYPE)
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(64, np.float64)
        self._bmul(_ptr(a), _ptr(b), _ptr(out))
        return out.reshape(8, 8)

    # matrix level
    def compress_matrix(self, m: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(m, np.float64)
        rows, cols = m.shape
        out = np.zeros(max(1, _nb(rows) * _nb(cols)), BLOCK_DTYPE)
        st = self._cm(_ptr(m), rows, cols, _ptr(out))
        if st:
            raise OracleError(st)
        return out.reshape(_nb(rows), _nb(cols))

    def decompress_matrix(self, blocks: np.ndarray, rows: int, cols: int) -> np.ndarray:
        blocks = np.ascontiguousarray(blocks, BLOCK_DTYPE)
        out = np.zeros((rows, cols), np.float64)
        self._dm(_ptr(blocks), rows, cols, _ptr(out))
        return out

    def mat_add(self, a, b):
        return self._mbin(self._madd, a, b)

    def mat_sub(self, a, b):
        return self._mbin(self._msub, a, b)

    def _mbin(self, f, a, b):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros_like(a)
        st = f(_ptr(a), _ptr(b), a.size, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def mat_scale(self, a, c: float):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        out = np.zeros_like(a)
        st = self._mscale(_ptr(a), C.c_double(c), a.size, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def mat_dot(self, a, ar, ac, b, br, bc, i, j) -> float:
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros(1, np.float64)
        st = self._mdot(_ptr(a), ar, ac, _ptr(b), br, bc, i, j, _ptr(out))
        if st:
            raise OracleError(st)
        return float(out[0])

    def mat_mul_dense(self, a, ar, ac, b, br, bc) -> np.ndarray:
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros((ar, bc), np.float64)
        st = self._mmd(_ptr(a), ar, ac, _ptr(b), br, bc, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def mat_mul(self, a, ar, ac, b, br, bc) -> np.ndarray:
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros((_nb(ar), _nb(bc)), BLOCK_DTYPE)
        st = self._mm(_ptr(a), ar, ac, _ptr(b), br, bc, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def rowdot(self, a, b, rows, cols) -> np.ndarray:
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros(rows, np.float64)
        self._rowdot(_ptr(a), _ptr(b), rows, cols, _ptr(out))
        return out

    def sum_ascending(self, v) -> float:
        v = np.ascontiguousarray(v, np.float64)
        return self._sum(_ptr(v), v.size)


class Ref:
    """The reference headers themselves, compiled under oracle/_ref."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        L = _Lib(path, "ref_")
        self.lib = L.lib
        self._err = L.fn("last_error", C.c_char_p, [])
        self.hardware_threads = L.fn("hardware_threads", C.c_uint, [])()
        self._basis = L.fn("dct_basis", None, [_P])
        self._cb = L.fn("compress_block", C.c_int, [_P, _P])
        self._db = L.fn("decompress_block", None, [_P, _P])
        self._pred = L.fn("predict_indices", C.c_int, [_P, _P])
        self._add = L.fn("add", C.c_int, [_P, _P, _P])
        self._sub = L.fn("sub", C.c_int, [_P, _P, _P])
        self._dot = L.fn("dot", C.c_int, [_P, _P, C.c_int, C.c_int, _P])
        self._cm = L.fn("compress_matrix", C.c_int, [_P, _SZ, _SZ, C.c_uint, _P])
        self._dm = L.fn("decompress_matrix", C.c_int, [_P, _SZ, _SZ, C.c_uint, _P])
        self._mbin = L.fn("mat_binop", C.c_int, [C.c_int, _P, _P, _SZ, _SZ, C.c_uint, _P])
        self._mscale = L.fn("mat_scale", C.c_int, [_P, _SZ, _SZ, C.c_double, C.c_uint, _P])
        self._mdot = L.fn("mat_dot", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P])
        self._mm = L.fn("mat_mul", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, C.c_uint, _P])
        self._mmd = L.fn("mat_mul_dense", C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, C.c_uint, _P])
        self._wc = L.fn("write_compressed", C.c_longlong, [_P, _SZ, _SZ, _P, _SZ])
        self._rc = L.fn("read_compressed", C.c_int, [_P, _SZ, C.POINTER(_SZ), C.POINTER(_SZ), _P, _SZ])
        # handle API (timing)
        self.dense_new = L.fn("dense_new", _P, [_P, _SZ, _SZ])
        self.dense_free = L.fn("dense_free", None, [_P])
        self.cm_free = L.fn("cm_free", None, [_P])
        self.h_compress = L.fn("h_compress", _P, [_P, C.c_uint])
        self.h_decompress = L.fn("h_decompress", _P, [_P, C.c_uint])
        self.h_add = L.fn("h_add", _P, [_P, _P, C.c_uint])
        self.h_sub = L.fn("h_sub", _P, [_P, _P, C.c_uint])
        self.h_scale = L.fn("h_scale", _P, [_P, C.c_double, C.c_uint])
        self.h_mul = L.fn("h_mul", _P, [_P, _P, C.c_uint])
        self.dense_data = L.fn("dense_data", _P, [_P])
        self.cm_blocks = L.fn("cm_blocks", _P, [_P])

    def _check(self, st):
        if st:
            raise OracleError(st, self._err().decode())

    def dct_basis(self) -> np.ndarray:
        t = np.zeros(64, np.float64)
        self._basis(_ptr(t))
        return t

    def compress_block(self, m):
        m = np.ascontiguousarray(m, np.float64).reshape(64)
        out = np.zeros(1, BLOCK_DTYPE)
        self._check(self._cb(_ptr(m), _ptr(out)))
        return out[0]

    def decompress_block(self, b):
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(64, np.float64)
        self._db(_ptr(b), _ptr(out))
        return out.reshape(8, 8)

    def predict_indices(self, m):
        m = np.ascontiguousarray(m, np.float64).reshape(64)
        idx = np.zeros(64, np.uint8)
        self._check(self._pred(_ptr(m), _ptr(idx)))
        return idx.reshape(8, 8)

    def add(self, a, b):
        return self._binop(self._add, a, b)

    def sub(self, a, b):
        return self._binop(self._sub, a, b)

    def _binop(self, f, a, b):
        a = np.array([a], BLOCK_DTYPE)
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(1, BLOCK_DTYPE)
        self._check(f(_ptr(a), _ptr(b), _ptr(out)))
        return out[0]

    def dot(self, a, b, i, j):
        a = np.array([a], BLOCK_DTYPE)
        b = np.array([b], BLOCK_DTYPE)
        out = np.zeros(1, np.float64)
        self._check(self._dot(_ptr(a), _ptr(b), i, j, _ptr(out)))
        return float(out[0])

    def compress_matrix(self, m, threads=1):
        m = np.ascontiguousarray(m, np.float64)
        rows, cols = m.shape
        out = np.zeros(max(1, _nb(rows) * _nb(cols)), BLOCK_DTYPE)
        self._check(self._cm(_ptr(m), rows, cols, threads, _ptr(out)))
        return out.reshape(_nb(rows), _nb(cols))

    def decompress_matrix(self, blocks, rows, cols, threads=1):
        blocks = np.ascontiguousarray(blocks, BLOCK_DTYPE)
        out = np.zeros((rows, cols), np.float64)
        self._check(self._dm(_ptr(blocks), rows, cols, threads, _ptr(out)))
        return out

    def mat_add(self, a, b, rows, cols, threads=1):
        return self._mb(0, a, b, rows, cols, threads)

    def mat_sub(self, a, b, rows, cols, threads=1):
        return self._mb(1, a, b, rows, cols, threads)

    def _mb(self, op, a, b, rows, cols, threads):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros_like(a)
        self._check(self._mbin(op, _ptr(a), _ptr(b), rows, cols, threads, _ptr(out)))
        return out

    def mat_scale(self, a, rows, cols, c, threads=1):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        out = np.zeros_like(a)
        self._check(self._mscale(_ptr(a), rows, cols, C.c_double(c), threads, _ptr(out)))
        return out

    def mat_dot(self, a, ar, ac, b, br, bc, i, j):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros(1, np.float64)
        self._check(self._mdot(_ptr(a), ar, ac, _ptr(b), br, bc, i, j, _ptr(out)))
        return float(out[0])

    def mat_mul(self, a, ar, ac, b, br, bc, threads=1):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros((_nb(ar), _nb(bc)), BLOCK_DTYPE)
        self._check(self._mm(_ptr(a), ar, ac, _ptr(b), br, bc, threads, _ptr(out)))
        return out

    def mat_mul_dense(self, a, ar, ac, b, br, bc, threads=1):
        a = np.ascontiguousarray(a, BLOCK_DTYPE)
        b = np.ascontiguousarray(b, BLOCK_DTYPE)
        out = np.zeros((ar, bc), np.float64)
        self._check(self._mmd(_ptr(a), ar, ac, _ptr(b), br, bc, threads, _ptr(out)))
        return out

    def write_compressed(self, blocks, rows, cols) -> bytes:
        blocks = np.ascontiguousarray(blocks, BLOCK_DTYPE)
        cap = 13 + 45 * blocks.size
        buf = np.zeros(cap, np.uint8)
        n = self._wc(_ptr(blocks), rows, cols, _ptr(buf), cap)
        if n < 0:
            raise OracleError(3, self._err().decode())
        return buf[:n].tobytes()

    def read_compressed(self, data: bytes):
        raw = np.frombuffer(data, np.uint8).copy()
        rows, cols = _SZ(), _SZ()
        cap = max(1, (len(data) // 45) + 1)
        out = np.zeros(cap, BLOCK_DTYPE)
        self._check(self._rc(_ptr(raw), raw.size, C.byref(rows), C.byref(cols), _ptr(out), cap))
        nb = _nb(rows.value) * _nb(cols.value)
        return rows.value, cols.value, out[:nb].copy()


def port() -> Port:
    return Port()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Ref:
    return Ref()
