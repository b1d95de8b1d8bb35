"""ctypes binding of the C ABI in include/blaz_cuda.h (libblaz_cuda.so).

The shared library is built in-tree by ``paper_2202_13007_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing this module raises
on import, so nothing can silently run on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libblaz_cuda.so")

# blaz::compressed_block (H/block.hpp:33-38), 48 bytes in memory.
BLOCK_DTYPE = np.dtype(
    {"names": ["first", "slope", "scale_factor", "coeffs"],
     "formats": ["<f8", "<f8", "u1", ("i1", 28)],
     "offsets": [0, 8, 16, 17], "itemsize": 48})

BLZ_OK, BLZ_INVALID_ARGUMENT, BLZ_OUT_OF_RANGE, BLZ_CUDA_ERROR, BLZ_OUT_OF_MEMORY, BLZ_NOT_SUPPORTED, BLZ_IO_ERROR = range(7)
GEMM_EXACT, GEMM_FUSED, GEMM_FUSED_DMMA, GEMM_FUSED_DFMA = 0, 1, 2, 3
MODE_DEFAULT, MODE_EXACT = 0, 1


class BlazError(RuntimeError):
    """CUDA / allocation failure inside the library."""


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(IndexError):
    """std::out_of_range in the reference."""


class IoError(RuntimeError):
    """blaz::io_error (H/io.hpp:20-23)."""


class NotBuilt(ImportError):
    pass


class blz_cmat(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64),
                ("block_rows", C.c_uint64), ("block_cols", C.c_uint64),
                ("first", C.c_void_p), ("slope", C.c_void_p),
                ("scale", C.c_void_p), ("coeffs", C.c_void_p)]


_P = C.c_void_p
_U64 = C.c_uint64
_I = C.c_int
_ST = C.c_int

# name -> (restype, argtypes); the full exported surface of include/blaz_cuda.h
SIGNATURES = {
    "blz_abi_version": (_I, []),
    "blz_ctx_create": (_ST, [_I, _P, C.POINTER(_P)]),
    "blz_ctx_destroy": (None, [_P]),
    "blz_ctx_set_stream": (_ST, [_P, _P]),
    "blz_ctx_get_stream": (_P, [_P]),
    "blz_last_error": (C.c_char_p, [_P]),
    "blz_ctx_sync": (_ST, [_P]),
    "blz_ctx_basis": (_ST, [_P, _P]),
    "blz_ctx_launches": (_U64, [_P]),
    "blz_ctx_set_mode": (_ST, [_P, _I]),
    "blz_ctx_get_mode": (_I, [_P]),
    "blz_ctx_fast_path_available": (_I, [_P]),
    "blz_ctx_stats": (_ST, [_P, C.POINTER(_U64), C.POINTER(_U64)]),
    "blz_cmat_bytes": (_U64, [_U64, _U64]),
    "blz_cmat_view": (_ST, [_U64, _U64, _P, C.POINTER(blz_cmat)]),
    "blz_cmat_alloc": (_ST, [_P, _U64, _U64, C.POINTER(blz_cmat)]),
    "blz_cmat_free": (None, [_P, C.POINTER(blz_cmat)]),
    "blz_compress_dev": (_ST, [_P, _P, _U64, _U64, _U64, C.POINTER(blz_cmat)]),
    "blz_decompress_dev": (_ST, [_P, C.POINTER(blz_cmat), _P, _U64]),
    "blz_add_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat)]),
    "blz_sub_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat)]),
    "blz_scale_dev": (_ST, [_P, C.POINTER(blz_cmat), C.c_double, C.POINTER(blz_cmat)]),
    "blz_scale_meta_dev": (_ST, [_P, C.POINTER(blz_cmat), C.c_double, C.POINTER(blz_cmat)]),
    "blz_matmul_panel_scratch_bytes": (_U64, [C.POINTER(blz_cmat), C.POINTER(blz_cmat), _U64]),
    "blz_matmul_panel_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.c_int, _U64, _P,
                                   C.POINTER(blz_cmat)]),
    "blz_matmul_dense_panel_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.c_int, _U64, _P, _P,
                                         _U64]),
    "blz_rowdot_frobenius_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _P]),
    "blz_reconstruct_rows_dev": (_ST, [_P, C.POINTER(blz_cmat), C.c_int, _P]),
    "blz_reconstruct_cols_dev": (_ST, [_P, C.POINTER(blz_cmat), C.c_int, _P]),
    "blz_block_mul_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P]),
    "blz_allgather_cmat_nccl": (_ST, [_P, _P, C.POINTER(blz_cmat), C.POINTER(blz_cmat)]),
    "blz_rowdot_frobenius_nccl": (_ST, [_P, _P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _U64, _P, _P]),
    "blz_frobenius_allreduce_nccl": (_ST, [_P, _P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _P]),
    "blz_matmul_nccl": (_ST, [_P, _P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.c_int, _P,
                               C.POINTER(blz_cmat)]),
    "blz_normalize_blocks": (_ST, [_P, _P, _U64, _P, _P]),
    "blz_denormalize_blocks": (_ST, [_P, _P, _P, _U64, _P]),
    "blz_mean_slope_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_predict_blocks": (_ST, [_P, _P, _P, _U64, _P, _P, _P, _P]),
    "blz_quantize_coeffs_blocks": (_ST, [_P, _P, _U64, _P, _P]),
    "blz_dct2_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_idct2_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_mean_relative_error_dev": (_ST, [_P, _P, _P, _U64, _P, _P]),
    "blz_mean_relative_error": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _P, _P]),
    "blz_add_decompress_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _U64]),
    "blz_sub_decompress_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _U64]),
    "blz_scale_decompress_dev": (_ST, [_P, C.POINTER(blz_cmat), C.c_double, C.POINTER(blz_cmat), _P, _U64]),
    "blz_dot_entries_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _P, _U64, _P]),
    "blz_decompress_gather_dev": (_ST, [_P, _P, _I, _P, _U64]),
    "blz_matmul_gather_dev": (_ST, [_P, C.POINTER(blz_cmat), _P, _I, _I, _P, C.POINTER(blz_cmat)]),
    "blz_dot_entries_rows_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P, _P, _U64, _U64, _U64, _P]),
    "blz_dot_entries_nccl": (_ST, [_P, _P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), C.POINTER(blz_cmat), _U64, _P,
                                   _P, _U64, _P]),
    "blz_rowdot_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _P]),
    "blz_sum_dev": (_ST, [_P, _P, _U64, _P]),
    "blz_matmul_scratch_bytes": (_U64, [C.POINTER(blz_cmat), C.POINTER(blz_cmat)]),
    "blz_matmul_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _I, _P, C.POINTER(blz_cmat)]),
    "blz_matmul_dense_dev": (_ST, [_P, C.POINTER(blz_cmat), C.POINTER(blz_cmat), _I, _P, _P, _U64]),
    "blz_pack_aos_dev": (_ST, [_P, C.POINTER(blz_cmat), _P]),
    "blz_unpack_aos_dev": (_ST, [_P, _P, C.POINTER(blz_cmat)]),
    "blz_compress_matrix": (_ST, [_P, _P, _U64, _U64, _P, C.c_uint]),
    "blz_decompress_matrix": (_ST, [_P, _P, _U64, _U64, _P, C.c_uint]),
    "blz_mat_add": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _P, C.c_uint]),
    "blz_mat_sub": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _P, C.c_uint]),
    "blz_mat_scale": (_ST, [_P, _P, _U64, _U64, C.c_double, _P, C.c_uint]),
    "blz_mat_dot": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _U64, _U64, _P]),
    "blz_mat_mul": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _P, C.c_uint]),
    "blz_mat_mul_dense": (_ST, [_P, _P, _U64, _U64, _P, _U64, _U64, _P, C.c_uint]),
    "blz_mat_rowdot": (_ST, [_P, _P, _P, _U64, _U64, _P, _P]),
    "blz_compress_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_decompress_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_dequantize_blocks": (_ST, [_P, _P, _U64, _P]),
    "blz_blzc_bytes": (_U64, [_U64, _U64]),
    "blz_pack_blzc_dev": (_ST, [_P, C.POINTER(blz_cmat), _P]),
    "blz_unpack_blzc_dev": (_ST, [_P, _P, _U64, C.POINTER(blz_cmat)]),
    "blz_write_compressed": (_ST, [_P, _P, _U64, _U64, _P, _U64, C.POINTER(_U64)]),
    "blz_read_compressed": (_ST, [_P, _P, _U64, C.POINTER(_U64), C.POINTER(_U64), _P, _U64]),
}

_lib = None


def load(path: str | None = None):
    """Loads libblaz_cuda.so (raises NotBuilt when absent -- no fallback).

    BLZ_LIB_PATH overrides the in-tree library (A/B builds of the same ABI)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("BLZ_LIB_PATH") or LIB_PATH
    if not os.path.exists(path):
        raise NotBuilt(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    ab = path != LIB_PATH  # an A/B build of an older revision may lack newer entry points
    for name, (res, args) in SIGNATURES.items():
        if ab and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def raise_for(status: int, ctx_handle) -> None:
    if status == BLZ_OK:
        return
    msg = load().blz_last_error(ctx_handle)
    msg = msg.decode() if msg else ""
    if status == BLZ_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == BLZ_OUT_OF_RANGE:
        raise OutOfRange(msg)
    if status == BLZ_IO_ERROR:
        raise IoError(msg)
    if status == BLZ_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise BlazError(f"status {status}: {msg}")
