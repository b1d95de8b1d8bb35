/*
 * blaz_cuda.h -- C ABI of the B200 (sm_100a) compressed-matrix library.
 *
 * Drop-in boundary for the reference's matrix API (namespace blaz,
 * proj/include/blaz/matrix.hpp).  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary.  Two levels:
 *
 *   blz_*_dev   device-resident, stream-ordered, caller-owned buffers (the
 *               throughput path; SoA compressed layout, see blz_cmat).
 *   blz_*_host  host buffers in the reference's own in-memory layout (dense
 *               row-major double, AoS 48-byte blz_block); copies in/out are part
 *               of the call and the call is synchronous, like the reference's
 *               value-returning functions.
 *
 * Every entry returns a blz_status.  On failure blz_last_error(ctx) holds the
 * reference's exception message (e.g. "mat_add: dimension mismatch (16x16 vs
 * 16x24)"); BLZ_INVALID_ARGUMENT maps to std::invalid_argument and
 * BLZ_OUT_OF_RANGE to std::out_of_range (see include/blaz/blaz.hpp).
 *
 * Data-dependent errors found on the device (non-finite input to compress,
 * "normalize: non-finite input", H/codec.hpp:21) are latched in the context:
 * _host calls report them directly; after _dev calls use blz_ctx_sync().
 *
 * Exact mode (default): every kernel is compiled with -fmad=false and follows
 * the reference's evaluation order, so phi/C are byte-exact and f/s/values
 * bit-exact against the reference built with -ffp-contract=off.
 */
#ifndef BLAZ_CUDA_H
#define BLAZ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLZ_ABI_VERSION 1

typedef enum blz_status {
    BLZ_OK = 0,
    BLZ_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    BLZ_OUT_OF_RANGE = 2,     /* std::out_of_range in the reference */
    BLZ_CUDA_ERROR = 3,
    BLZ_OUT_OF_MEMORY = 4,
    BLZ_NOT_SUPPORTED = 5,
    BLZ_IO_ERROR = 6          /* blaz::io_error in the reference (H/io.hpp:20-23) */
} blz_status;

/* Reference compressed_block (H/block.hpp:33-38), 48 bytes in memory:
 * first@0, slope@8, scale_factor@16, coeffs@17..44, 3 pad bytes. */
typedef struct blz_block {
    double first;
    double slope;
    uint8_t scale_factor;
    int8_t coeffs[28];
} blz_block;

/* Device-resident compressed matrix, SoA over the row-major block grid
 * (block (br,bc) is index br*block_cols+bc, as H/matrix.hpp:38-39).
 * first/slope: nb doubles; scale: nb bytes; coeffs: nb*28 bytes, block t's
 * 28 coefficients at coeffs[28*t .. 28*t+27] in the frozen keep-set order
 * (H/block.hpp:48-56).  45 bytes per block, the on-disk payload size. */
typedef struct blz_cmat {
    uint64_t rows, cols;             /* logical dimensions */
    uint64_t block_rows, block_cols; /* ceil(rows/8), ceil(cols/8) */
    double* first;
    double* slope;
    uint8_t* scale;
    int8_t* coeffs;
} blz_cmat;

typedef struct blz_ctx blz_ctx;

/* GEMM accumulation modes for blz_matmul_* (H/matrix.hpp:188-202 accumulates
 * acc = 0.0; acc += a*b over k ascending, products and sums rounded separately) */
typedef enum blz_gemm_mode {
    BLZ_GEMM_EXACT = 0,      /* DMUL+DADD, ascending k: bitwise equal to mat_mul/mat_dot */
    BLZ_GEMM_FUSED = 1,      /* acc = fma(a, b, acc), ascending k: tolerance parity; runs the
                                faster of the two kernels below (their results are bitwise equal) */
    BLZ_GEMM_FUSED_DMMA = 2, /* the fused chain on FP64 tensor cores (mma.sync m8n8k4 f64) */
    BLZ_GEMM_FUSED_DFMA = 3  /* the fused chain as CUDA-core DFMA */
} blz_gemm_mode;

/* ---- context --------------------------------------------------------------- */
int blz_abi_version(void);
/* Creates a context on `device`.  `basis` may be NULL (the library evaluates
 * the reference expression H/dct.hpp:17-21 with the host libm) or 64 doubles
 * to upload bit-for-bit.  The first context created on a device also binds its
 * basis to the device's constant copy used by the main decompress kernel;
 * contexts with another basis decompress through a slower kernel (same
 * results for their basis). */
blz_status blz_ctx_create(int device, const double* basis, blz_ctx** out);
void blz_ctx_destroy(blz_ctx* ctx);
/* Stream for all subsequent calls (cudaStream_t as void*; NULL = legacy). */
blz_status blz_ctx_set_stream(blz_ctx* ctx, void* stream);
void* blz_ctx_get_stream(const blz_ctx* ctx);
const char* blz_last_error(const blz_ctx* ctx);
/* Synchronizes the context stream and reports latched device-side errors. */
blz_status blz_ctx_sync(blz_ctx* ctx);
/* Copies the 64-entry basis in use into `out`. */
blz_status blz_ctx_basis(const blz_ctx* ctx, double* out);
/* Number of kernel launches issued through this context so far. */
uint64_t blz_ctx_launches(const blz_ctx* ctx);
/* Kernel selection.  BLZ_MODE_DEFAULT: compress runs the verified fast path
 * (fused arithmetic + certified integer decisions, uncertified blocks re-run in
 * reference order -- results identical to the reference).  BLZ_MODE_EXACT:
 * every kernel follows the reference's evaluation order literally. */
#define BLZ_MODE_DEFAULT 0
#define BLZ_MODE_EXACT 1
blz_status blz_ctx_set_mode(blz_ctx* ctx, int mode);
int blz_ctx_get_mode(const blz_ctx* ctx);
/* 1 if the uploaded basis admits the verified fast path (the reference basis does). */
int blz_ctx_fast_path_available(const blz_ctx* ctx);
/* Cumulative counters (synchronizes): blocks compressed on the exact path
 * because a decision was not certified, and add/sub blocks that took the
 * s1 + s2 == 0 dense fallback (H/block_ops.hpp:36-44). */
blz_status blz_ctx_stats(blz_ctx* ctx, uint64_t* compress_exact_blocks, uint64_t* addsub_fallback_blocks);

/* ---- device-resident compressed matrices --------------------------------- */
/* Bytes of device memory one SoA matrix of rows x cols needs. */
uint64_t blz_cmat_bytes(uint64_t rows, uint64_t cols);
/* Lays out `m` over caller-owned device memory `mem` (blz_cmat_bytes bytes). */
blz_status blz_cmat_view(uint64_t rows, uint64_t cols, void* mem, blz_cmat* m);
/* Allocates with cudaMalloc (freed by blz_cmat_free). */
blz_status blz_cmat_alloc(blz_ctx* ctx, uint64_t rows, uint64_t cols, blz_cmat* m);
void blz_cmat_free(blz_ctx* ctx, blz_cmat* m);

/* ---- device-level operations (stream-ordered, no hidden allocation) ------- */
/* compress_matrix (H/matrix.hpp:97-111): dense row-major with leading
 * dimension ld (elements); out must be rows x cols. */
blz_status blz_compress_dev(blz_ctx* ctx, const double* dense, uint64_t rows, uint64_t cols,
                            uint64_t ld, const blz_cmat* out);
/* decompress_matrix (H/matrix.hpp:113-126): crops to rows x cols. */
blz_status blz_decompress_dev(blz_ctx* ctx, const blz_cmat* in, double* dense, uint64_t ld);
/* mat_add / mat_sub / mat_scale (H/matrix.hpp:128-151) */
blz_status blz_add_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out);
blz_status blz_sub_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out);
blz_status blz_scale_dev(blz_ctx* ctx, const blz_cmat* a, double c, const blz_cmat* out);
/* mat_scale as a metadata-only update (H/block_ops.hpp:74-77
 * changes only f and s): writes out->first / out->slope (c * a's) and points
 * out->scale / out->coeffs at a's arrays, so 16 B/block are read and 16 B
 * written instead of 45 + 45.  The result shares a's phi/C storage: it is valid
 * while a's arrays are alive and unchanged.  out may be a itself (in place). */
blz_status blz_scale_meta_dev(blz_ctx* ctx, const blz_cmat* a, double c, blz_cmat* out);
/* Op chains: the op of blz_add_dev / blz_sub_dev /
 * blz_scale_dev writing `out`, followed by blz_decompress_dev(out, dense, ld);
 * results are bitwise those of the two calls.  scale (and add / sub on views
 * that are not 16-byte aligned) run as one fused pass over the operands; add /
 * sub otherwise run their two kernels back to back, which measured faster.
 * Replaces the reference sequence mat_add(...) -> decompress_matrix(...)
 * (H/matrix.hpp:128-151, :113-126). */
blz_status blz_add_decompress_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out,
                                  double* dense, uint64_t ld);
blz_status blz_sub_decompress_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, const blz_cmat* out,
                                  double* dense, uint64_t ld);
blz_status blz_scale_decompress_dev(blz_ctx* ctx, const blz_cmat* a, double c, const blz_cmat* out,
                                    double* dense, uint64_t ld);
/* Batched mat_dot (H/matrix.hpp:157-173): out[q] = (Ahat Bhat)(i[q], j[q]).
 * i, j, out are device arrays of n entries; indices are validated on device
 * (an out-of-range index latches BLZ_OUT_OF_RANGE). */
blz_status blz_dot_entries_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b,
                               const uint64_t* i, const uint64_t* j, uint64_t n, double* out);
/* The same entries against a row shard: a_rows holds rows [row0, row0 + a_rows->rows)
 * (row0 a multiple of 8) of a matrix with rows_total rows; i are global row
 * indices.  Entries on rows of other shards are +0.0 (all bits zero), so the
 * results of all shards combine exactly by an integer sum of their 64-bit
 * patterns (blz_dot_entries_nccl).  Replaces nothing in the reference: the
 * batched mat_dot of SURVEY.md 8(e), routed to the rank owning row i. */
blz_status blz_dot_entries_rows_dev(blz_ctx* ctx, const blz_cmat* a_rows, const blz_cmat* b,
                                    const uint64_t* i, const uint64_t* j, uint64_t n, uint64_t row0,
                                    uint64_t rows_total, double* out);
/* Row-wise dot products (config 2; restated):
 * r[i] = sum_j Ahat(i,j)*Bhat(i,j), ascending j from +0.0, for the rows of a
 * and b (same dims).  r has a->rows entries. */
blz_status blz_rowdot_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, double* r);
/* Ascending serial sum of n doubles (the Frobenius total from row dots). */
blz_status blz_sum_dev(blz_ctx* ctx, const double* v, uint64_t n, double* out);
/* blz_rowdot_dev and the ascending total of r (blz_sum_dev) in one pass: bitwise the same. */
blz_status blz_rowdot_frobenius_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, double* r, double* total);
/* mat_mul (H/matrix.hpp:223-235) and mat_mul_dense (:239-250).
 * scratch: device buffer of blz_matmul_scratch_bytes(a,b) bytes. */
uint64_t blz_matmul_scratch_bytes(const blz_cmat* a, const blz_cmat* b);
blz_status blz_matmul_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, int mode,
                          void* scratch, const blz_cmat* out);
blz_status blz_matmul_dense_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, int mode,
                                void* scratch, double* out, uint64_t ld);
/* K-paneled variants (HBM capacity): B is decompressed
 * panel_block_rows block-rows at a time (a positive multiple of 4) and each
 * panel's product accumulated into C; bitwise the results of the one-pass calls.
 * scratch: blz_matmul_panel_scratch_bytes(a, b, panel_block_rows) bytes (dense A,
 * one B panel and, for the compressed output, dense C). */
uint64_t blz_matmul_panel_scratch_bytes(const blz_cmat* a, const blz_cmat* b, uint64_t panel_block_rows);
blz_status blz_matmul_panel_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, int mode,
                                uint64_t panel_block_rows, void* scratch, const blz_cmat* out);
blz_status blz_matmul_dense_panel_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, int mode,
                                      uint64_t panel_block_rows, void* scratch, double* out, uint64_t ld);
/* ---- block-row sharded operations over NCCL --------
 * `nccl_comm` is an ncclComm_t of G ranks (one GPU each); rank r owns
 * block-rows [BR*r/G, BR*(r+1)/G) of every operand and result.  NCCL is
 * loaded at run time (libnccl.so.2); without it these return
 * BLZ_NOT_SUPPORTED.  Stream-ordered on the context stream.
 *   allgather_cmat: the whole compressed matrix `full` from the row shards
 *     (45 B per block over NVLink instead of 512 B of binary64);
 *   rowdot_frobenius: config 2 -- local row dots, all r_i gathered in row order
 *     into r_all (rows_total entries) and their ascending total (bit-identical
 *     to the one-GPU result for every G);
 *   frobenius_allreduce: per-rank ascending partials summed by one allreduce
 *     (tolerance parity); r_local has a_local->rows entries;
 *   matmul: config 4 -- gathers B into b_full, then C rows = A rows x B
 *     (H/matrix.hpp:223-235); scratch: blz_matmul_scratch_bytes(a_local, b_full);
 *   dot_entries: batched mat_dot (H/matrix.hpp:157-173) -- gathers B into
 *     b_full, each rank evaluates the queries on its own rows of A, and one
 *     allreduce (integer sum of the 64-bit patterns) gives every rank all n
 *     entries, bit-identical to the one-GPU result; i, j, out are device arrays
 *     of n entries (i global row indices, the same on every rank). */
blz_status blz_allgather_cmat_nccl(blz_ctx* ctx, void* nccl_comm, const blz_cmat* local, const blz_cmat* full);
blz_status blz_rowdot_frobenius_nccl(blz_ctx* ctx, void* nccl_comm, const blz_cmat* a_local,
                                     const blz_cmat* b_local, uint64_t rows_total, double* r_all, double* total);
blz_status blz_frobenius_allreduce_nccl(blz_ctx* ctx, void* nccl_comm, const blz_cmat* a_local,
                                        const blz_cmat* b_local, double* r_local, double* total);
blz_status blz_matmul_nccl(blz_ctx* ctx, void* nccl_comm, const blz_cmat* a_local, const blz_cmat* b_local,
                           const blz_cmat* b_full, int mode, void* scratch, const blz_cmat* c_local);
blz_status blz_dot_entries_nccl(blz_ctx* ctx, void* nccl_comm, const blz_cmat* a_local, const blz_cmat* b_local,
                                const blz_cmat* b_full, uint64_t rows_total, const uint64_t* i, const uint64_t* j,
                                uint64_t n, double* out);
/* Fused all-gather + decompress: a matrix held as
 * nshards (<= 16) consecutive block-row shards in separate SoA arrays --
 * typically the ranks' own shards, opened as peer pointers (CUDA IPC) so the
 * kernel reads them over NVLink -- decompressed into one dense array (rows =
 * the shards' rows summed; every shard but the last holds whole block-rows).
 * blz_matmul_gather_dev: mat_mul with B given as such shards, bitwise equal
 * to blz_matmul_dev on the whole B (scratch: blz_matmul_scratch_bytes(a, b)
 * for the whole B's dimensions).  No collective library involved: the
 * transfer is the decompression kernel's own loads. */
blz_status blz_decompress_gather_dev(blz_ctx* ctx, const blz_cmat* shards, int nshards, double* dense,
                                     uint64_t ld);
blz_status blz_matmul_gather_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b_shards, int nshards, int mode,
                                 void* scratch, const blz_cmat* out);

/* AoS (48-byte blz_block, device memory) <-> SoA conversions. */
blz_status blz_pack_aos_dev(blz_ctx* ctx, const blz_cmat* in, blz_block* out);
blz_status blz_unpack_aos_dev(blz_ctx* ctx, const blz_block* in, const blz_cmat* out);

/* ---- host-level drop-in entry points (synchronous) ------------------------ */
/* Each mirrors one reference function; blocks are host AoS arrays of
 * ceil(rows/8)*ceil(cols/8) entries.  `threads` is accepted for signature
 * parity with the reference and ignored (there is no CPU fallback). */
blz_status blz_compress_matrix(blz_ctx* ctx, const double* values, uint64_t rows, uint64_t cols,
                               blz_block* out, unsigned threads);
blz_status blz_decompress_matrix(blz_ctx* ctx, const blz_block* in, uint64_t rows, uint64_t cols,
                                 double* out, unsigned threads);
blz_status blz_mat_add(blz_ctx* ctx, const blz_block* a, uint64_t a_rows, uint64_t a_cols,
                       const blz_block* b, uint64_t b_rows, uint64_t b_cols, blz_block* out,
                       unsigned threads);
blz_status blz_mat_sub(blz_ctx* ctx, const blz_block* a, uint64_t a_rows, uint64_t a_cols,
                       const blz_block* b, uint64_t b_rows, uint64_t b_cols, blz_block* out,
                       unsigned threads);
blz_status blz_mat_scale(blz_ctx* ctx, const blz_block* a, uint64_t rows, uint64_t cols,
                         double c, blz_block* out, unsigned threads);
blz_status blz_mat_dot(blz_ctx* ctx, const blz_block* a, uint64_t a_rows, uint64_t a_cols,
                       const blz_block* b, uint64_t b_rows, uint64_t b_cols, uint64_t i,
                       uint64_t j, double* out);
blz_status blz_mat_mul(blz_ctx* ctx, const blz_block* a, uint64_t a_rows, uint64_t a_cols,
                       const blz_block* b, uint64_t b_rows, uint64_t b_cols, blz_block* out,
                       unsigned threads);
blz_status blz_mat_mul_dense(blz_ctx* ctx, const blz_block* a, uint64_t a_rows, uint64_t a_cols,
                             const blz_block* b, uint64_t b_rows, uint64_t b_cols, double* out,
                             unsigned threads);
/* Config-2 restatement on host buffers: row dots r[rows] and their ascending
 * total (*frob, may be NULL). */
blz_status blz_mat_rowdot(blz_ctx* ctx, const blz_block* a, const blz_block* b, uint64_t rows,
                          uint64_t cols, double* r, double* frob);

/* ---- block-level entry points (H/codec.hpp, H/block_ops.hpp), batched ------ */
/* n independent 8x8 blocks (64 row-major doubles each) <-> n blz_block. */
blz_status blz_compress_blocks(blz_ctx* ctx, const double* tiles, uint64_t n, blz_block* out);
blz_status blz_decompress_blocks(blz_ctx* ctx, const blz_block* in, uint64_t n, double* tiles);
/* dequantize_prediction (H/codec.hpp:150-158): the 8x8 slope grid of each block. */
blz_status blz_dequantize_blocks(blz_ctx* ctx, const blz_block* in, uint64_t n, double* tiles);

/* Device-batched block-level API (H/block_ops.hpp:87-142):
 * the n = rows/8-by-cols/8 blocks of `in` (or block pairs of a, b with equal
 * grids) in block order, results as n row-major 8x8 tiles (64 doubles each) in
 * device memory.
 *   reconstruct_rows(b, last_row): rows 0..last_row of decompress_block(b)
 *     (bitwise), other rows +0.0; last_row outside [0, 7] -> BLZ_OUT_OF_RANGE
 *     "reconstruct_rows: row index out of range"
 *   reconstruct_cols(b, last_col): columns 0..last_col, other columns +0.0
 *   block_mul(b1, b2): out(i,j) = sum_k d1(i,k) * d2(k,j), k ascending (= dot). */
blz_status blz_reconstruct_rows_dev(blz_ctx* ctx, const blz_cmat* in, int last_row, double* tiles);
blz_status blz_reconstruct_cols_dev(blz_ctx* ctx, const blz_cmat* in, int last_col, double* tiles);
blz_status blz_block_mul_dev(blz_ctx* ctx, const blz_cmat* a, const blz_cmat* b, double* tiles);

/* ---- stage functions of the codec, batched ---------------
 * Host arrays of n blocks (64 doubles each, row-major), computed on the GPU one
 * thread per block in the reference's order:
 *   normalize (H/codec.hpp:20-32): first[n], deltas[n*64]; non-finite input
 *     -> BLZ_INVALID_ARGUMENT "normalize: non-finite input"
 *   denormalize (:35-44), mean_slope (:47-57)
 *   predict (:61-98): indices[n*64], snapped[n*64], quantizer lo[n], step[n];
 *     slope_mean <= 0 -> "predict: mean slope must be positive"
 *   quantize_coeffs (:108-125): scale[n], coeffs[n*28] (keep-set order)
 *   dct2 / idct2 (H/dct.hpp:32-70) with the context's basis */
blz_status blz_normalize_blocks(blz_ctx* ctx, const double* m, uint64_t n, double* first, double* deltas);
blz_status blz_denormalize_blocks(blz_ctx* ctx, const double* first, const double* deltas, uint64_t n, double* m);
blz_status blz_mean_slope_blocks(blz_ctx* ctx, const double* deltas, uint64_t n, double* s);
blz_status blz_predict_blocks(blz_ctx* ctx, const double* slopes, const double* slope_mean, uint64_t n,
                              uint8_t* indices, double* snapped, double* lo, double* step);
blz_status blz_quantize_coeffs_blocks(blz_ctx* ctx, const double* d, uint64_t n, uint8_t* scale, int8_t* coeffs);
blz_status blz_dct2_blocks(blz_ctx* ctx, const double* x, uint64_t n, double* d);
blz_status blz_idct2_blocks(blz_ctx* ctx, const double* d, uint64_t n, double* x);

/* ---- evaluation harness --------------------------------
 * mean_relative_error (H/bench.hpp:67-84): mean of |(cand - ref) / ref| over
 * the entries with |ref| >= 1e-12 (serial sum in index order, as the
 * reference), and the count of excluded entries.  _dev: device arrays of n
 * entries, results written to device memory; host variant: host matrices with
 * the reference's dimension check ("mean_relative_error: dimension mismatch"). */
blz_status blz_mean_relative_error_dev(blz_ctx* ctx, const double* ref, const double* cand, uint64_t n,
                                       double* mean, uint64_t* excluded);
blz_status blz_mean_relative_error(blz_ctx* ctx, const double* ref, uint64_t ref_rows, uint64_t ref_cols,
                                   const double* cand, uint64_t cand_rows, uint64_t cand_cols, double* mean,
                                   uint64_t* excluded);

/* ---- .blzc container (H/io.hpp:93-134) --------------------------------------- */
/* 13-byte header ("BLZC", version 1, rows, cols as LE u32) + 45-byte records
 * (f, s LE binary64, scale byte, 28 coefficients) in row-major block order. */
uint64_t blz_blzc_bytes(uint64_t rows, uint64_t cols);
/* write_compressed on the device: `out` (device) receives blz_blzc_bytes bytes;
 * a non-finite f or s latches "write_compressed: non-finite block field". */
blz_status blz_pack_blzc_dev(blz_ctx* ctx, const blz_cmat* in, uint8_t* out);
/* read_compressed on the device (synchronizes for the header): validates
 * magic, version, zero dims, zero scale factors and truncation with the
 * reference's messages; `out` must have the header's dimensions. */
blz_status blz_unpack_blzc_dev(blz_ctx* ctx, const uint8_t* in, uint64_t nbytes, const blz_cmat* out);
/* Host-buffer variants.  blz_read_compressed with out == NULL only parses the
 * header into rows/cols. */
blz_status blz_write_compressed(blz_ctx* ctx, const blz_block* blocks, uint64_t rows, uint64_t cols,
                                uint8_t* out, uint64_t capacity, uint64_t* written);
blz_status blz_read_compressed(blz_ctx* ctx, const uint8_t* bytes, uint64_t nbytes, uint64_t* rows,
                               uint64_t* cols, blz_block* out, uint64_t out_capacity);

#ifdef __cplusplus
}
#endif
#endif /* BLAZ_CUDA_H */
