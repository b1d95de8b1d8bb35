/*
 * blaz_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's per-8x8-block codec and compressed
 * operations (arXiv 2202.13007, reference at proj/include/blaz/).  It exists
 * only as the CHECKER for the CUDA path: tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may call it; the product
 * (paper_2202_13007_b200/) never links or imports it.
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement bit-for-bit
 * against (1) the reference's own known-answer vectors (ramp block,
 * proj/tests/test_util.hpp:28-54, codec_test.cpp) and (2) golden fixtures
 * produced by the real reference headers compiled under oracle/_ref
 * (tests/golden/make_golden.py).
 *
 * Build contract: compiled with -O2 -ffp-contract=off, the same pin the
 * reference uses (proj/CMakeLists.txt:15-18), so every multiply and add is
 * rounded separately.
 */
#ifndef BLAZ_ORACLE_H
#define BLAZ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same member order/layout as blaz::compressed_block (H/block.hpp:33-38):
 * 48 bytes in memory (f@0, s@8, phi@16, C@17..44, 3 pad bytes). */
typedef struct orc_block {
    double first;
    double slope;
    uint8_t scale_factor;
    int8_t coeffs[28];
} orc_block;

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_RANGE = 2 };

/* block level ------------------------------------------------------------ */
void   orc_dct_basis(double t[64]);
void   orc_dct2(const double x[64], double d[64]);
void   orc_idct2(const double d[64], double x[64]);
int    orc_normalize(const double m[64], double* first, double deltas[64]);
double orc_mean_slope(const double deltas[64]);
void   orc_predict(const double slopes[64], double slope_mean, uint8_t idx[64], double snapped[64]);
void   orc_quantize_coeffs(const double d[64], uint8_t* phi, int8_t c[28]);
int    orc_compress_block(const double m[64], orc_block* out);
void   orc_dequantize_prediction(const orc_block* b, double slopes[64]);
void   orc_decompress_block(const orc_block* b, double out[64]);
int    orc_add(const orc_block* a, const orc_block* b, orc_block* out);
int    orc_sub(const orc_block* a, const orc_block* b, orc_block* out);
int    orc_scale(const orc_block* a, double c, orc_block* out);
void   orc_reconstruct_rows(const orc_block* b, int last_row, double out[64]);
void   orc_reconstruct_cols(const orc_block* b, int last_col, double out[64]);
double orc_dot(const orc_block* a, const orc_block* b, int i, int j);
void   orc_block_mul(const orc_block* a, const orc_block* b, double out[64]);
double orc_round_half_away(double x);

/* matrix level (row-major block grid, AoS blocks) -------------------------- */
int    orc_compress_matrix(const double* values, size_t rows, size_t cols, orc_block* out);
void   orc_decompress_matrix(const orc_block* in, size_t rows, size_t cols, double* out);
int    orc_mat_add(const orc_block* a, const orc_block* b, size_t nblocks, orc_block* out);
int    orc_mat_sub(const orc_block* a, const orc_block* b, size_t nblocks, orc_block* out);
int    orc_mat_scale(const orc_block* a, double c, size_t nblocks, orc_block* out);
int    orc_mat_dot(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                   size_t b_rows, size_t b_cols, size_t i, size_t j, double* out);
int    orc_mat_mul_dense(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                         size_t b_rows, size_t b_cols, double* out);
int    orc_mat_mul(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                   size_t b_rows, size_t b_cols, orc_block* out);
/* Config-2 restatement (not a reference function):
 * r_i = sum_j Ahat(i,j)*Bhat(i,j) ascending j from +0.0, frob = sum_i r_i ascending. */
int    orc_rowdot(const orc_block* a, const orc_block* b, size_t rows, size_t cols, double* r);
double orc_sum_ascending(const double* v, size_t n);

#ifdef __cplusplus
}
#endif
#endif
