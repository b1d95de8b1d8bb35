"""Host-side mirror of the reference matrix API (proj/include/blaz/matrix.hpp).

Same names, argument meaning and error behaviour as namespace blaz:

=====================  ==========================================  =====================
this module            reference                                   C ABI entry
=====================  ==========================================  =====================
compress_matrix        compress_matrix  (H/matrix.hpp:97-111)      blz_compress_matrix
decompress_matrix      decompress_matrix (:113-126)                blz_decompress_matrix
mat_add / mat_sub      mat_add / mat_sub (:128-144)                blz_mat_add / _sub
mat_scale              mat_scale (:146-151)                        blz_mat_scale
mat_dot                mat_dot (:157-173)                          blz_mat_dot
mat_mul                mat_mul (:223-235)                          blz_mat_mul
mat_mul_dense          mat_mul_dense (:239-250)                    blz_mat_mul_dense
mat_rowdot             (config-2 restatement)        blz_mat_rowdot
compress_block(s)      compress_block (H/codec.hpp:130-146)        blz_compress_blocks
decompress_block(s)    decompress_block (H/codec.hpp:180-185)      blz_decompress_blocks
=====================  ==========================================  =====================

std::invalid_argument -> InvalidArgument (a ValueError), std::out_of_range ->
OutOfRange (an IndexError), with the reference's messages.  Inputs and outputs
are host numpy arrays (dense: 2-D float64 row-major; compressed: the 48-byte
AoS block grid), so every call copies host->device and back, exactly as a
drop-in for the reference's value-returning functions must.  ``threads`` is
accepted for signature parity and ignored: all arithmetic runs in CUDA.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading

import numpy as np

from . import _native as N
from ._native import BLOCK_DTYPE, InvalidArgument, IoError, OutOfRange  # noqa: F401

block_dim = 8
block_cells = 64
kept_coeff_count = 28
block_payload_bytes = 8 + 8 + 1 + kept_coeff_count  # 45, H/block.hpp:18
compression_rate = (block_cells * 8 * 8) / (block_payload_bytes * 8)  # H/block.hpp:19-20


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Context:
    """One blz_ctx (device, stream, uploaded DCT basis, scratch)."""

    def __init__(self, device: int = 0, basis: np.ndarray | None = None):
        self.lib = N.load()
        h = C.c_void_p()
        b = None
        if basis is not None:
            b = np.ascontiguousarray(basis, np.float64).reshape(64)
        st = self.lib.blz_ctx_create(device, _ptr(b) if b is not None else None, C.byref(h))
        if st != N.BLZ_OK:
            raise N.BlazError(f"blz_ctx_create failed with status {st}")
        self.handle = h
        self.device = device
        self._basis_keepalive = b

    def close(self):
        if self.handle:
            self.lib.blz_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int):
        N.raise_for(st, self.handle)

    def sync(self):
        self.check(self.lib.blz_ctx_sync(self.handle))

    def basis(self) -> np.ndarray:
        t = np.zeros(64, np.float64)
        self.check(self.lib.blz_ctx_basis(self.handle, _ptr(t)))
        return t

    def launches(self) -> int:
        return int(self.lib.blz_ctx_launches(self.handle))

    def set_mode(self, mode: int):
        """MODE_DEFAULT (verified fast compress) or MODE_EXACT (reference order everywhere)."""
        self.check(self.lib.blz_ctx_set_mode(self.handle, mode))

    def fast_path_available(self) -> bool:
        return bool(self.lib.blz_ctx_fast_path_available(self.handle))

    def stats(self) -> dict:
        a, b = C.c_uint64(), C.c_uint64()
        self.check(self.lib.blz_ctx_stats(self.handle, C.byref(a), C.byref(b)))
        return {"compress_exact_blocks": a.value, "addsub_fallback_blocks": b.value}

    def set_stream(self, stream_ptr: int | None):
        self.check(self.lib.blz_ctx_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


@dataclasses.dataclass
class CompressedMatrix:
    """blaz::compressed_matrix (H/matrix.hpp:31-40): logical dims + row-major block grid."""

    rows: int
    cols: int
    blocks: np.ndarray  # BLOCK_DTYPE, shape (block_rows, block_cols)

    @property
    def block_rows(self) -> int:
        return (self.rows + 7) // 8

    @property
    def block_cols(self) -> int:
        return (self.cols + 7) // 8

    def block(self, br: int, bc: int):
        return self.blocks[br, bc]


def _nb(n: int) -> int:
    return (n + 7) // 8


def _blocks(cm: CompressedMatrix) -> np.ndarray:
    b = np.ascontiguousarray(cm.blocks, BLOCK_DTYPE)
    if b.size != cm.block_rows * cm.block_cols:
        raise InvalidArgument("compressed matrix: block count does not match dimensions")
    return b


def compress_matrix(m, threads: int = 1, ctx: Context | None = None) -> CompressedMatrix:
    ctx = ctx or default_context()
    m = np.asarray(m, np.float64)
    if m.ndim != 2 or m.shape[0] == 0 or m.shape[1] == 0:
        raise InvalidArgument("compress_matrix: empty matrix")
    m = np.ascontiguousarray(m)
    rows, cols = m.shape
    out = np.zeros((_nb(rows), _nb(cols)), BLOCK_DTYPE)
    ctx.check(ctx.lib.blz_compress_matrix(ctx.handle, _ptr(m), rows, cols, _ptr(out), threads))
    return CompressedMatrix(rows, cols, out)


def decompress_matrix(cm: CompressedMatrix, threads: int = 1, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    b = _blocks(cm)
    out = np.zeros((cm.rows, cm.cols), np.float64)
    ctx.check(ctx.lib.blz_decompress_matrix(ctx.handle, _ptr(b), cm.rows, cm.cols, _ptr(out), threads))
    return out


def _binop(fn, a: CompressedMatrix, b: CompressedMatrix, threads, ctx) -> CompressedMatrix:
    ctx = ctx or default_context()
    ba, bb = _blocks(a), _blocks(b)
    out = np.zeros_like(ba)
    ctx.check(fn(ctx.handle, _ptr(ba), a.rows, a.cols, _ptr(bb), b.rows, b.cols, _ptr(out), threads))
    return CompressedMatrix(a.rows, a.cols, out)


def mat_add(a: CompressedMatrix, b: CompressedMatrix, threads: int = 1, ctx: Context | None = None):
    ctx = ctx or default_context()
    return _binop(ctx.lib.blz_mat_add, a, b, threads, ctx)


def mat_sub(a: CompressedMatrix, b: CompressedMatrix, threads: int = 1, ctx: Context | None = None):
    ctx = ctx or default_context()
    return _binop(ctx.lib.blz_mat_sub, a, b, threads, ctx)


def mat_scale(a: CompressedMatrix, c: float, threads: int = 1, ctx: Context | None = None):
    ctx = ctx or default_context()
    ba = _blocks(a)
    out = np.zeros_like(ba)
    ctx.check(ctx.lib.blz_mat_scale(ctx.handle, _ptr(ba), a.rows, a.cols, C.c_double(c), _ptr(out), threads))
    return CompressedMatrix(a.rows, a.cols, out)


def mat_dot(a: CompressedMatrix, b: CompressedMatrix, i: int, j: int, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    if i < 0 or j < 0:
        raise OutOfRange("mat_dot: index out of range")
    ba, bb = _blocks(a), _blocks(b)
    out = np.zeros(1, np.float64)
    ctx.check(ctx.lib.blz_mat_dot(ctx.handle, _ptr(ba), a.rows, a.cols, _ptr(bb), b.rows, b.cols, i, j, _ptr(out)))
    return float(out[0])


def mat_mul(a: CompressedMatrix, b: CompressedMatrix, threads: int = 1, ctx: Context | None = None):
    ctx = ctx or default_context()
    ba, bb = _blocks(a), _blocks(b)
    out = np.zeros((_nb(a.rows), _nb(b.cols)), BLOCK_DTYPE)
    ctx.check(ctx.lib.blz_mat_mul(ctx.handle, _ptr(ba), a.rows, a.cols, _ptr(bb), b.rows, b.cols, _ptr(out), threads))
    return CompressedMatrix(a.rows, b.cols, out)


def mat_mul_dense(a: CompressedMatrix, b: CompressedMatrix, threads: int = 1, ctx: Context | None = None):
    ctx = ctx or default_context()
    ba, bb = _blocks(a), _blocks(b)
    out = np.zeros((a.rows, b.cols), np.float64)
    ctx.check(ctx.lib.blz_mat_mul_dense(ctx.handle, _ptr(ba), a.rows, a.cols, _ptr(bb), b.rows, b.cols,
                                        _ptr(out), threads))
    return out


def mat_rowdot(a: CompressedMatrix, b: CompressedMatrix, ctx: Context | None = None):
    """Row-wise dots r_i = sum_j Ahat(i,j) Bhat(i,j) and their ascending total."""
    ctx = ctx or default_context()
    if a.rows != b.rows or a.cols != b.cols:
        raise InvalidArgument(f"mat_rowdot: dimension mismatch ({a.rows}x{a.cols} vs {b.rows}x{b.cols})")
    ba, bb = _blocks(a), _blocks(b)
    r = np.zeros(a.rows, np.float64)
    frob = np.zeros(1, np.float64)
    ctx.check(ctx.lib.blz_mat_rowdot(ctx.handle, _ptr(ba), _ptr(bb), a.rows, a.cols, _ptr(r), _ptr(frob)))
    return r, float(frob[0])


def compress_blocks(tiles, ctx: Context | None = None) -> np.ndarray:
    """Batched compress_block over an (n, 8, 8) array."""
    ctx = ctx or default_context()
    t = np.ascontiguousarray(tiles, np.float64).reshape(-1, 64)
    out = np.zeros(t.shape[0], BLOCK_DTYPE)
    ctx.check(ctx.lib.blz_compress_blocks(ctx.handle, _ptr(t), t.shape[0], _ptr(out)))
    return out


def decompress_blocks(blocks, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    b = np.ascontiguousarray(blocks, BLOCK_DTYPE).reshape(-1)
    out = np.zeros((b.size, 8, 8), np.float64)
    ctx.check(ctx.lib.blz_decompress_blocks(ctx.handle, _ptr(b), b.size, _ptr(out)))
    return out


def compress_block(tile, ctx: Context | None = None):
    return compress_blocks(np.asarray(tile).reshape(1, 8, 8), ctx)[0]


def decompress_block(block, ctx: Context | None = None) -> np.ndarray:
    return decompress_blocks(np.array([block], BLOCK_DTYPE), ctx)[0]


def write_compressed(cm: CompressedMatrix, ctx: Context | None = None) -> bytes:
    """write_compressed (H/io.hpp:96-111): the .blzc byte stream, packed on the GPU."""
    ctx = ctx or default_context()
    b = _blocks(cm)
    n = int(ctx.lib.blz_blzc_bytes(cm.rows, cm.cols))
    out = np.zeros(n, np.uint8)
    written = C.c_uint64()
    ctx.check(ctx.lib.blz_write_compressed(ctx.handle, _ptr(b), cm.rows, cm.cols, _ptr(out), n, C.byref(written)))
    return out[: written.value].tobytes()


def read_compressed(data: bytes, ctx: Context | None = None) -> CompressedMatrix:
    """read_compressed (H/io.hpp:113-134): parses and validates on the GPU;
    malformed input raises IoError with the reference's message."""
    ctx = ctx or default_context()
    raw = np.frombuffer(bytes(data), np.uint8).copy()
    rows, cols = C.c_uint64(), C.c_uint64()
    ctx.check(ctx.lib.blz_read_compressed(ctx.handle, _ptr(raw), raw.size, C.byref(rows), C.byref(cols), None, 0))
    out = np.zeros((_nb(rows.value), _nb(cols.value)), BLOCK_DTYPE)
    ctx.check(ctx.lib.blz_read_compressed(ctx.handle, _ptr(raw), raw.size, C.byref(rows), C.byref(cols), _ptr(out),
                                          out.size))
    return CompressedMatrix(rows.value, cols.value, out)
