"""Device-resident API: compressed matrices living in HBM (SoA, 45 B/block).

Torch is used only for device memory and streams; every operation is one
C-ABI call (``blz_*_dev``) that launches the sm_100a kernels on the context
stream, which is bound to torch's current CUDA stream at each call.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .matrix import BLOCK_DTYPE, CompressedMatrix, Context


def _nb(n: int) -> int:
    return (n + 7) // 8


_ctxs: dict[tuple[int, int], Context] = {}


def context(device: int | None = None) -> Context:
    """The context bound to torch's current stream on `device`.  Each stream gets
    its own context (own scratch and exact-path worklist), so operations issued
    on different streams may run concurrently."""
    dev = torch.cuda.current_device() if device is None else device
    stream = torch.cuda.current_stream(dev).cuda_stream
    ctx = _ctxs.get((dev, stream))
    if ctx is None:
        ctx = Context(dev)
        ctx.set_stream(stream)
        _ctxs[(dev, stream)] = ctx
    return ctx


def contexts(device: int | None = None) -> list[Context]:
    """All contexts created on `device` (one per stream used)."""
    dev = torch.cuda.current_device() if device is None else device
    return [c for (d, _), c in _ctxs.items() if d == dev]


class DeviceCMat:
    """A blz_cmat laid over one torch uint8 buffer."""

    def __init__(self, rows: int, cols: int, device=None, buf: torch.Tensor | None = None):
        lib = N.load()
        self.rows, self.cols = int(rows), int(cols)
        nbytes = int(lib.blz_cmat_bytes(self.rows, self.cols))
        if buf is None:
            buf = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device or "cuda")
        assert buf.numel() >= nbytes and buf.is_cuda
        self.buf = buf
        self.c = N.blz_cmat()
        st = lib.blz_cmat_view(self.rows, self.cols, C.c_void_p(buf.data_ptr()), C.byref(self.c))
        assert st == 0

    @property
    def block_rows(self):
        return _nb(self.rows)

    @property
    def block_cols(self):
        return _nb(self.cols)

    @property
    def nblocks(self):
        return self.block_rows * self.block_cols

    def ref(self):
        return C.byref(self.c)

    # SoA views (torch tensors aliasing the buffer)
    def _view(self, ptr_attr: str, dtype, count):
        off = getattr(self.c, ptr_attr) - self.buf.data_ptr()
        item = torch.empty(0, dtype=dtype).element_size()
        return self.buf[off:off + count * item].view(dtype)

    @property
    def first(self):
        return self._view("first", torch.float64, self.nblocks)

    @property
    def slope(self):
        return self._view("slope", torch.float64, self.nblocks)

    @property
    def scale(self):
        return self._view("scale", torch.uint8, self.nblocks)

    @property
    def coeffs(self):
        return self._view("coeffs", torch.int8, self.nblocks * 28).view(self.nblocks, 28)

    def to_host(self, ctx: Context | None = None) -> CompressedMatrix:
        ctx = ctx or context(self.buf.device.index)
        aos = torch.empty(max(1, self.nblocks) * 48, dtype=torch.uint8, device=self.buf.device)
        ctx.check(ctx.lib.blz_pack_aos_dev(ctx.handle, self.ref(), C.c_void_p(aos.data_ptr())))
        host = aos.cpu().numpy().view(BLOCK_DTYPE)[: self.nblocks]
        return CompressedMatrix(self.rows, self.cols, host.reshape(self.block_rows, self.block_cols).copy())

    @staticmethod
    def from_host(cm: CompressedMatrix, device="cuda", ctx: Context | None = None) -> "DeviceCMat":
        out = DeviceCMat(cm.rows, cm.cols, device=device)
        ctx = ctx or context(out.buf.device.index)
        raw = np.ascontiguousarray(cm.blocks, BLOCK_DTYPE).view(np.uint8).reshape(-1)
        aos = torch.from_numpy(raw.copy()).to(out.buf.device)
        ctx.check(ctx.lib.blz_unpack_aos_dev(ctx.handle, C.c_void_p(aos.data_ptr()), out.ref()))
        torch.cuda.current_stream(out.buf.device).synchronize()
        return out


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


def compress(dense: torch.Tensor, out: DeviceCMat | None = None) -> DeviceCMat:
    """compress_matrix on a device fp64 2-D tensor (row stride = ld)."""
    assert dense.is_cuda and dense.dtype == torch.float64 and dense.dim() == 2 and dense.stride(1) == 1
    rows, cols = dense.shape
    ctx = context(dense.device.index)
    if rows == 0 or cols == 0:
        raise N.InvalidArgument("compress_matrix: empty matrix")
    out = out or DeviceCMat(rows, cols, device=dense.device)
    ctx.check(ctx.lib.blz_compress_dev(ctx.handle, _ptr(dense), rows, cols, dense.stride(0), out.ref()))
    return out


def decompress(cm: DeviceCMat, out: torch.Tensor | None = None) -> torch.Tensor:
    ctx = context(cm.buf.device.index)
    if out is None:
        out = torch.empty((cm.rows, cm.cols), dtype=torch.float64, device=cm.buf.device)
    ctx.check(ctx.lib.blz_decompress_dev(ctx.handle, cm.ref(), _ptr(out), out.stride(0)))
    return out


def _shard_array(shards):
    arr = (N.blz_cmat * len(shards))()
    for k, sh in enumerate(shards):
        arr[k] = sh.c
    return arr


def decompress_gather(shards, out: torch.Tensor | None = None) -> torch.Tensor:
    """Decompresses a matrix held as consecutive block-row shards (separate
    DeviceCMats: the ranks' shards, possibly other GPUs' memory opened as peer
    views) in one kernel -- the fused all-gather + decompress
    (blz_decompress_gather_dev)."""
    dev0 = torch.device("cuda", torch.cuda.current_device())
    ctx = context(dev0.index)
    rows, cols = sum(sh.rows for sh in shards), shards[0].cols
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float64, device=dev0)
    arr = _shard_array(shards)
    ctx.check(ctx.lib.blz_decompress_gather_dev(ctx.handle, arr, len(shards), _ptr(out), out.stride(0)))
    return out


def matmul_gather(a: DeviceCMat, b_shards, mode: int = N.GEMM_EXACT, out: DeviceCMat | None = None,
                  scratch: torch.Tensor | None = None) -> DeviceCMat:
    """mat_mul with B given as block-row shards (blz_matmul_gather_dev): B is
    decompressed straight from the shards, bitwise the same product as matmul."""
    ctx = context(a.buf.device.index)
    b_rows, b_cols = sum(sh.rows for sh in b_shards), b_shards[0].cols
    if scratch is None:
        dims = N.blz_cmat(rows=b_rows, cols=b_cols, block_rows=_nb(b_rows), block_cols=_nb(b_cols))
        n = int(N.load().blz_matmul_scratch_bytes(a.ref(), C.byref(dims)))
        scratch = torch.empty(n, dtype=torch.uint8, device=a.buf.device)
    out = out or DeviceCMat(a.rows, b_cols, device=a.buf.device)
    arr = _shard_array(b_shards)
    ctx.check(ctx.lib.blz_matmul_gather_dev(ctx.handle, a.ref(), arr, len(b_shards), mode, _ptr(scratch), out.ref()))
    return out


def add(a: DeviceCMat, b: DeviceCMat, out: DeviceCMat | None = None) -> DeviceCMat:
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    ctx.check(ctx.lib.blz_add_dev(ctx.handle, a.ref(), b.ref(), out.ref()))
    return out


def sub(a: DeviceCMat, b: DeviceCMat, out: DeviceCMat | None = None) -> DeviceCMat:
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    ctx.check(ctx.lib.blz_sub_dev(ctx.handle, a.ref(), b.ref(), out.ref()))
    return out


def scale(a: DeviceCMat, c: float, out: DeviceCMat | None = None) -> DeviceCMat:
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    ctx.check(ctx.lib.blz_scale_dev(ctx.handle, a.ref(), C.c_double(c), out.ref()))
    return out


class ScaledCMat(DeviceCMat):
    """Result of `scale_meta`: own f / s arrays, phi / C shared with the source
    matrix (kept alive by this object)."""

    def __init__(self, a: DeviceCMat, fs: torch.Tensor | None = None):
        nb = a.nblocks
        self.rows, self.cols = a.rows, a.cols
        self.src = a
        self.buf = fs if fs is not None else torch.empty(max(2 * nb, 2), dtype=torch.float64, device=a.buf.device)
        assert self.buf.dtype == torch.float64 and self.buf.numel() >= 2 * nb
        self.c = N.blz_cmat()
        self.c.rows, self.c.cols = a.rows, a.cols
        self.c.block_rows, self.c.block_cols = a.block_rows, a.block_cols
        self.c.first = self.buf.data_ptr()
        self.c.slope = self.buf.data_ptr() + 8 * nb
        self.c.scale, self.c.coeffs = a.c.scale, a.c.coeffs

    @property
    def first(self):
        return self.buf[: self.nblocks]

    @property
    def slope(self):
        return self.buf[self.nblocks: 2 * self.nblocks]

    @property
    def scale(self):
        return self.src.scale

    @property
    def coeffs(self):
        return self.src.coeffs


def scale_meta(a: DeviceCMat, c: float, out: ScaledCMat | None = None) -> ScaledCMat:
    """mat_scale as a metadata-only update (H/block_ops.hpp:74-77 changes only f
    and s): 16 B/block read and written; phi / C stay in `a`'s arrays."""
    ctx = context(a.buf.device.index)
    out = out if out is not None else ScaledCMat(a)
    if out.src is not a:
        out.src = a
    ctx.check(ctx.lib.blz_scale_meta_dev(ctx.handle, a.ref(), C.c_double(c), out.ref()))
    return out


def _dense_for(a: DeviceCMat, dense: torch.Tensor | None) -> torch.Tensor:
    if dense is None:
        dense = torch.empty((a.rows, a.cols), dtype=torch.float64, device=a.buf.device)
    assert dense.is_cuda and dense.dtype == torch.float64 and dense.dim() == 2 and dense.stride(1) == 1
    return dense


def add_decompress(a: DeviceCMat, b: DeviceCMat, out: DeviceCMat | None = None,
                   dense: torch.Tensor | None = None) -> tuple[DeviceCMat, torch.Tensor]:
    """Fused mat_add -> decompress_matrix: (compressed A+B, its decompression)."""
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    dense = _dense_for(a, dense)
    ctx.check(ctx.lib.blz_add_decompress_dev(ctx.handle, a.ref(), b.ref(), out.ref(), _ptr(dense), dense.stride(0)))
    return out, dense


def sub_decompress(a: DeviceCMat, b: DeviceCMat, out: DeviceCMat | None = None,
                   dense: torch.Tensor | None = None) -> tuple[DeviceCMat, torch.Tensor]:
    """Fused mat_sub -> decompress_matrix."""
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    dense = _dense_for(a, dense)
    ctx.check(ctx.lib.blz_sub_decompress_dev(ctx.handle, a.ref(), b.ref(), out.ref(), _ptr(dense), dense.stride(0)))
    return out, dense


def scale_decompress(a: DeviceCMat, c: float, out: DeviceCMat | None = None,
                     dense: torch.Tensor | None = None) -> tuple[DeviceCMat, torch.Tensor]:
    """Fused mat_scale -> decompress_matrix."""
    ctx = context(a.buf.device.index)
    out = out or DeviceCMat(a.rows, a.cols, device=a.buf.device)
    dense = _dense_for(a, dense)
    ctx.check(ctx.lib.blz_scale_decompress_dev(ctx.handle, a.ref(), C.c_double(c), out.ref(), _ptr(dense),
                                               dense.stride(0)))
    return out, dense


def dot_entries(a: DeviceCMat, b: DeviceCMat, i: torch.Tensor, j: torch.Tensor) -> torch.Tensor:
    ctx = context(a.buf.device.index)
    i = i.to(device=a.buf.device, dtype=torch.int64).contiguous()
    j = j.to(device=a.buf.device, dtype=torch.int64).contiguous()
    out = torch.empty(i.numel(), dtype=torch.float64, device=a.buf.device)
    ctx.check(ctx.lib.blz_dot_entries_dev(ctx.handle, a.ref(), b.ref(), _ptr(i), _ptr(j), i.numel(), _ptr(out)))
    return out


def dot_entries_rows(a_rows: DeviceCMat, b: DeviceCMat, i: torch.Tensor, j: torch.Tensor, row0: int,
                     rows_total: int) -> torch.Tensor:
    """dot_entries against a row shard: a_rows holds rows [row0, row0 + a_rows.rows)
    of a rows_total-row matrix, i are global rows; entries on other shards' rows are
    +0.0 (all bits zero), so shards combine by an integer sum of the bit patterns
    (blz_dot_entries_rows_dev)."""
    ctx = context(b.buf.device.index)
    i = i.to(device=b.buf.device, dtype=torch.int64).contiguous()
    j = j.to(device=b.buf.device, dtype=torch.int64).contiguous()
    out = torch.empty(i.numel(), dtype=torch.float64, device=b.buf.device)
    ctx.check(ctx.lib.blz_dot_entries_rows_dev(ctx.handle, a_rows.ref(), b.ref(), _ptr(i), _ptr(j), i.numel(),
                                               row0, rows_total, _ptr(out)))
    return out


def rowdot(a: DeviceCMat, b: DeviceCMat, out: torch.Tensor | None = None) -> torch.Tensor:
    ctx = context(a.buf.device.index)
    if out is None:
        out = torch.empty(a.rows, dtype=torch.float64, device=a.buf.device)
    ctx.check(ctx.lib.blz_rowdot_dev(ctx.handle, a.ref(), b.ref(), _ptr(out)))
    return out


def sum_ascending(v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    ctx = context(v.device.index)
    v = v.contiguous()
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=v.device)
    ctx.check(ctx.lib.blz_sum_dev(ctx.handle, _ptr(v), v.numel(), _ptr(out)))
    return out


def frobenius(a: DeviceCMat, b: DeviceCMat):
    """Row dots and their ascending total, in one pass (blz_rowdot_frobenius_dev)."""
    ctx = context(a.buf.device.index)
    r = torch.empty(a.rows, dtype=torch.float64, device=a.buf.device)
    total = torch.empty(1, dtype=torch.float64, device=a.buf.device)
    ctx.check(ctx.lib.blz_rowdot_frobenius_dev(ctx.handle, a.ref(), b.ref(), _ptr(r), _ptr(total)))
    return r, total


def _tiles(cm: DeviceCMat) -> torch.Tensor:
    return torch.empty((cm.nblocks, 8, 8), dtype=torch.float64, device=cm.buf.device)


def reconstruct_rows(cm: DeviceCMat, last_row: int) -> torch.Tensor:
    """partial_reconstruction.values of every block (H/block_ops.hpp:87-95): (n, 8, 8)."""
    ctx = context(cm.buf.device.index)
    out = _tiles(cm)
    ctx.check(ctx.lib.blz_reconstruct_rows_dev(ctx.handle, cm.ref(), int(last_row), _ptr(out)))
    return out


def reconstruct_cols(cm: DeviceCMat, last_col: int) -> torch.Tensor:
    """partial_reconstruction.values of every block (H/block_ops.hpp:99-115): (n, 8, 8)."""
    ctx = context(cm.buf.device.index)
    out = _tiles(cm)
    ctx.check(ctx.lib.blz_reconstruct_cols_dev(ctx.handle, cm.ref(), int(last_col), _ptr(out)))
    return out


def block_mul(a: DeviceCMat, b: DeviceCMat) -> torch.Tensor:
    """block_mul of every block pair (H/block_ops.hpp:131-142): (n, 8, 8)."""
    ctx = context(a.buf.device.index)
    out = _tiles(a)
    ctx.check(ctx.lib.blz_block_mul_dev(ctx.handle, a.ref(), b.ref(), _ptr(out)))
    return out


def matmul_scratch(a: DeviceCMat, b: DeviceCMat) -> torch.Tensor:
    n = int(N.load().blz_matmul_scratch_bytes(a.ref(), b.ref()))
    return torch.empty(n, dtype=torch.uint8, device=a.buf.device)


def matmul(a: DeviceCMat, b: DeviceCMat, mode: int = N.GEMM_EXACT, out: DeviceCMat | None = None,
           scratch: torch.Tensor | None = None) -> DeviceCMat:
    ctx = context(a.buf.device.index)
    if a.cols != b.rows:
        raise N.InvalidArgument("mat_mul: inner dimension mismatch")
    scratch = scratch if scratch is not None else matmul_scratch(a, b)
    out = out or DeviceCMat(a.rows, b.cols, device=a.buf.device)
    ctx.check(ctx.lib.blz_matmul_dev(ctx.handle, a.ref(), b.ref(), mode, _ptr(scratch), out.ref()))
    return out


def matmul_dense(a: DeviceCMat, b: DeviceCMat, mode: int = N.GEMM_EXACT, out: torch.Tensor | None = None,
                 scratch: torch.Tensor | None = None) -> torch.Tensor:
    ctx = context(a.buf.device.index)
    if a.cols != b.rows:
        raise N.InvalidArgument("mat_mul: inner dimension mismatch")
    scratch = scratch if scratch is not None else matmul_scratch(a, b)
    if out is None:
        out = torch.empty((a.rows, b.cols), dtype=torch.float64, device=a.buf.device)
    ctx.check(ctx.lib.blz_matmul_dense_dev(ctx.handle, a.ref(), b.ref(), mode, _ptr(scratch), _ptr(out),
                                           out.stride(0)))
    return out


def matmul_panel_scratch(a: DeviceCMat, b: DeviceCMat, panel_block_rows: int) -> torch.Tensor:
    n = int(N.load().blz_matmul_panel_scratch_bytes(a.ref(), b.ref(), int(panel_block_rows)))
    return torch.empty(n, dtype=torch.uint8, device=a.buf.device)


def matmul_panel(a: DeviceCMat, b: DeviceCMat, panel_block_rows: int, mode: int = N.GEMM_EXACT,
                 out: DeviceCMat | None = None, scratch: torch.Tensor | None = None) -> DeviceCMat:
    """mat_mul with B decompressed panel_block_rows block-rows at a time (bitwise = matmul)."""
    ctx = context(a.buf.device.index)
    scratch = scratch if scratch is not None else matmul_panel_scratch(a, b, panel_block_rows)
    out = out or DeviceCMat(a.rows, b.cols, device=a.buf.device)
    ctx.check(ctx.lib.blz_matmul_panel_dev(ctx.handle, a.ref(), b.ref(), mode, int(panel_block_rows),
                                           _ptr(scratch), out.ref()))
    return out


def matmul_dense_panel(a: DeviceCMat, b: DeviceCMat, panel_block_rows: int, mode: int = N.GEMM_EXACT,
                       out: torch.Tensor | None = None, scratch: torch.Tensor | None = None) -> torch.Tensor:
    ctx = context(a.buf.device.index)
    scratch = scratch if scratch is not None else matmul_panel_scratch(a, b, panel_block_rows)
    if out is None:
        out = torch.empty((a.rows, b.cols), dtype=torch.float64, device=a.buf.device)
    ctx.check(ctx.lib.blz_matmul_dense_panel_dev(ctx.handle, a.ref(), b.ref(), mode, int(panel_block_rows),
                                                 _ptr(scratch), _ptr(out), out.stride(0)))
    return out


def sync(device: int | None = None):
    context(device).sync()
