"""B200-native (sm_100a) compressed-matrix hot path of arXiv 2202.13007 ("blaz").

Host API mirroring the reference's ``namespace blaz`` matrix functions
(proj/include/blaz/matrix.hpp) over the C ABI in ``include/blaz_cuda.h``;
all arithmetic runs in hand-written CUDA kernels (``csrc/``).  Importing the
package requires the built library ``lib/libblaz_cuda.so`` -- there is no
CPU fallback.
"""
from ._native import (BLOCK_DTYPE, GEMM_EXACT, GEMM_FUSED, GEMM_FUSED_DFMA, GEMM_FUSED_DMMA, MODE_DEFAULT, MODE_EXACT, BlazError, InvalidArgument, IoError,  # noqa: F401
                      NotBuilt, OutOfRange, load)
from .matrix import (CompressedMatrix, Context, block_dim, block_payload_bytes,  # noqa: F401
                     compress_block, compress_blocks, compress_matrix, compression_rate,
                     decompress_block, decompress_blocks, decompress_matrix, default_context,
                     kept_coeff_count, mat_add, mat_dot, mat_mul, mat_mul_dense, mat_rowdot,
                     mat_scale, mat_sub, read_compressed, write_compressed)

load()  # fail loudly at import when the CUDA library is missing
