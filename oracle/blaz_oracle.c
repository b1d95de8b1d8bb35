/*
 * blaz_oracle.c -- CPU ORACLE (test infrastructure only; see blaz_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Every function cites the
 * reference lines it follows (H/ = proj/include/blaz/).  Compile with
 * -O2 -ffp-contract=off (oracle/Makefile) so products and sums round
 * separately, exactly as the reference build pins (proj/CMakeLists.txt:15-18).
 *
 * This file is the checker, never the product: the CUDA library in
 * paper_2202_13007_b200/ does not link it.
 */
#include "blaz_oracle.h"

#include <math.h>
#include <string.h>

#define BD 8
#define BC 64
#define KEPT 28

/* H/block.hpp:48-56: frozen keep-set order (row 0, row 1, col 0 rows 2..7,
 * col 1 rows 2..7). */
static const uint8_t KROW[KEPT] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1,
                                   1, 1, 2, 3, 4, 5, 6, 7, 2, 3, 4, 5, 6, 7};
static const uint8_t KCOL[KEPT] = {0, 1, 2, 3, 4, 5, 6, 7, 0, 1, 2, 3, 4, 5,
                                   6, 7, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1};

/* std::max(a, b) == (a < b) ? b : a  -- keeps a when b is NaN. */
static inline double stdmax(double a, double b) { return (a < b) ? b : a; }

/* H/block.hpp:61-67.  The long long truncation is spelled out with the
 * x86-64 cvttsd2si result for out-of-range / NaN inputs (INT64_MIN), which is
 * what the reference build executes for those inputs. */
double orc_round_half_away(double x) {
    double t;
    if (x >= -9223372036854775808.0 && x < 9223372036854775808.0)
        t = (double)(long long)x;
    else
        t = -9223372036854775808.0;
    const double frac = x - t;
    if (frac >= 0.5) return t + 1.0;
    if (frac <= -0.5) return t - 1.0;
    return t;
}

/* H/block.hpp:69-74 */
static int clamp_index(double x) {
    const double r = orc_round_half_away(x);
    if (r <= 0.0) return 0;
    if (r >= 255.0) return 255;
    return (int)r;
}

/* H/block.hpp:76-81 */
static int8_t clamp_coeff(double x) {
    const double r = orc_round_half_away(x);
    if (r <= -127.0) return -127;
    if (r >= 127.0) return 127;
    return (int8_t)r;
}

/* H/dct.hpp:14-26: t(i,u) = a_i cos((2u+1) i pi / 16), evaluated with libm
 * in the same expression order, so the table is bit-identical. */
void orc_dct_basis(double t[64]) {
    const double pi = acos(-1.0);
    for (int i = 0; i < BD; ++i) {
        const double ai = (i == 0) ? sqrt(1.0 / 8.0) : sqrt(1.0 / 4.0);
        for (int u = 0; u < BD; ++u) t[i * BD + u] = ai * cos((2 * u + 1) * i * pi / 16.0);
    }
}

static const double* basis(void) {
    static double t[64];
    static int init = 0;
    if (!init) {
        orc_dct_basis(t);
        init = 1;
    }
    return t;
}

/* H/dct.hpp:32-49: tmp = T x (ascending u from +0.0), d = tmp T' (ascending v). */
void orc_dct2(const double x[64], double d[64]) {
    const double* t = basis();
    double tmp[64];
    for (int i = 0; i < BD; ++i)
        for (int v = 0; v < BD; ++v) {
            double acc = 0.0;
            for (int u = 0; u < BD; ++u) acc += t[i * BD + u] * x[u * BD + v];
            tmp[i * BD + v] = acc;
        }
    for (int i = 0; i < BD; ++i)
        for (int j = 0; j < BD; ++j) {
            double acc = 0.0;
            for (int v = 0; v < BD; ++v) acc += tmp[i * BD + v] * t[j * BD + v];
            d[i * BD + j] = acc;
        }
}

/* H/dct.hpp:53-70: tmp = T' d (ascending i), x = tmp T (ascending j). */
void orc_idct2(const double d[64], double x[64]) {
    const double* t = basis();
    double tmp[64];
    for (int u = 0; u < BD; ++u)
        for (int j = 0; j < BD; ++j) {
            double acc = 0.0;
            for (int i = 0; i < BD; ++i) acc += t[i * BD + u] * d[i * BD + j];
            tmp[u * BD + j] = acc;
        }
    for (int u = 0; u < BD; ++u)
        for (int v = 0; v < BD; ++v) {
            double acc = 0.0;
            for (int j = 0; j < BD; ++j) acc += tmp[u * BD + j] * t[j * BD + v];
            x[u * BD + v] = acc;
        }
}

/* H/block.hpp:83-87 + H/codec.hpp:20-32 */
int orc_normalize(const double m[64], double* first, double d[64]) {
    for (int k = 0; k < BC; ++k)
        if (!isfinite(m[k])) return ORC_INVALID; /* "normalize: non-finite input" */
    *first = m[0];
    d[0] = 0.0;
    for (int j = 1; j < BD; ++j) d[j] = m[j] - m[j - 1];
    for (int i = 1; i < BD; ++i) d[i * BD] = m[i * BD] - m[(i - 1) * BD];
    for (int i = 1; i < BD; ++i)
        for (int j = 1; j < BD; ++j)
            d[i * BD + j] =
                ((m[i * BD + j] - m[(i - 1) * BD + j]) + (m[i * BD + j] - m[i * BD + j - 1])) / 2.0;
    return ORC_OK;
}

/* H/codec.hpp:47-57: serial row-major sum of |delta| over nonzero entries. */
double orc_mean_slope(const double d[64]) {
    double sum = 0.0;
    int nonzero = 0;
    for (int k = 0; k < BC; ++k) {
        if (d[k] != 0.0) {
            sum += fabs(d[k]);
            ++nonzero;
        }
    }
    return nonzero == 0 ? 0.0 : sum / nonzero;
}

/* H/codec.hpp:61-71 (slope_quantizer) + :85-98 (predict).  The caller has
 * already checked slope_mean > 0 (predict throws otherwise, :86). */
void orc_predict(const double slopes[64], double slope_mean, uint8_t idx[64], double snapped[64]) {
    double s_max = 0.0;
    for (int k = 0; k < BC; ++k) s_max = stdmax(s_max, fabs(slopes[k]));
    const double lo = slope_mean - s_max;
    const double step = 2.0 * s_max / 256;
    for (int k = 0; k < BC; ++k) {
        const int q = (step == 0.0) ? 0 : clamp_index((slopes[k] - lo) / step);
        idx[k] = (uint8_t)q;
        snapped[k] = lo + q * step;
    }
}

/* H/codec.hpp:108-125 */
void orc_quantize_coeffs(const double d[64], uint8_t* phi_out, int8_t c[28]) {
    double m = 0.0;
    for (int k = 0; k < BC; ++k) m = stdmax(m, fabs(d[k]));
    memset(c, 0, KEPT);
    if (m == 0.0) {
        *phi_out = 1;
        return;
    }
    double phi = floor(127.0 / m);
    if (phi < 1.0) phi = 1.0;
    if (phi > 255.0) phi = 255.0;
    *phi_out = (uint8_t)phi;
    for (int k = 0; k < KEPT; ++k) c[k] = clamp_coeff(phi * d[KROW[k] * BD + KCOL[k]]);
}

/* H/codec.hpp:130-146.  Returns ORC_INVALID for non-finite input
 * ("normalize: non-finite input") and ORC_RANGE when predict would throw
 * ("predict: mean slope must be positive": s is NaN). */
int orc_compress_block(const double m[64], orc_block* out) {
    double d[64];
    memset(out, 0, sizeof *out);
    out->scale_factor = 1;
    if (orc_normalize(m, &out->first, d) != ORC_OK) return ORC_INVALID;
    const double s = orc_mean_slope(d);
    out->slope = s;
    if (s == 0.0) return ORC_OK;
    if (!(s > 0.0)) return ORC_RANGE;
    double slopes[64], snapped[64], dct[64];
    uint8_t idx[64];
    for (int k = 0; k < BC; ++k) slopes[k] = d[k] / s;
    orc_predict(slopes, s, idx, snapped);
    orc_dct2(snapped, dct);
    orc_quantize_coeffs(dct, &out->scale_factor, out->coeffs);
    return ORC_OK;
}

/* H/codec.hpp:150-158 */
void orc_dequantize_prediction(const orc_block* b, double slopes[64]) {
    double d[64];
    if (b->slope == 0.0) {
        memset(slopes, 0, 64 * sizeof(double));
        return;
    }
    memset(d, 0, sizeof d);
    for (int k = 0; k < KEPT; ++k)
        d[KROW[k] * BD + KCOL[k]] = (double)b->coeffs[k] / (double)b->scale_factor;
    orc_idct2(d, slopes);
}

/* H/codec.hpp:164-174 (integrate_rows) */
static void integrate_rows(const orc_block* b, const double* p, int last_row, double* o) {
    const double s = b->slope;
    o[0] = b->first;
    for (int j = 1; j < BD; ++j) o[j] = o[j - 1] + s * p[j];
    for (int i = 1; i <= last_row; ++i) {
        o[i * BD] = o[(i - 1) * BD] + s * p[i * BD];
        for (int j = 1; j < BD; ++j)
            o[i * BD + j] = (o[(i - 1) * BD + j] + o[i * BD + j - 1]) / 2.0 + s * p[i * BD + j];
    }
}

/* H/codec.hpp:180-185 */
void orc_decompress_block(const orc_block* b, double out[64]) {
    double p[64];
    memset(out, 0, 64 * sizeof(double));
    orc_dequantize_prediction(b, p);
    integrate_rows(b, p, BD - 1, out);
}

/* H/block_ops.hpp:12-15.  phi1 + phi2 == 0 only for invalid blocks (the
 * reference reader rejects phi == 0, H/io.hpp:129-130); defined here as 1. */
static int merge_scale_factor(int p1, int p2) {
    if (p1 + p2 == 0) return 1;
    const int phi = (p1 * p2) / (p1 + p2);
    return phi < 1 ? 1 : (phi > 255 ? 255 : phi);
}

/* H/block_ops.hpp:20-58 */
static int combine(const orc_block* b1, const orc_block* b2, double rhs_sign, orc_block* out) {
    const double f = b1->first + rhs_sign * b2->first;
    if (b2->slope == 0.0) {
        *out = *b1;
        out->first = f;
        return ORC_OK;
    }
    if (b1->slope == 0.0) {
        *out = *b2;
        out->first = f;
        if (rhs_sign < 0.0)
            for (int k = 0; k < KEPT; ++k)
                out->coeffs[k] = (out->coeffs[k] == -127) ? (int8_t)127 : (int8_t)(-out->coeffs[k]);
        return ORC_OK;
    }
    const double s = b1->slope + b2->slope;
    if (s == 0.0) {
        double d1[64], d2[64], sum[64];
        orc_decompress_block(b1, d1);
        orc_decompress_block(b2, d2);
        for (int k = 0; k < BC; ++k) sum[k] = d1[k] + rhs_sign * d2[k];
        return orc_compress_block(sum, out);
    }
    memset(out, 0, sizeof *out);
    out->first = f;
    out->slope = s;
    const int phi = merge_scale_factor(b1->scale_factor, b2->scale_factor);
    out->scale_factor = (uint8_t)phi;
    const double a1 = b1->slope / s;
    const double a2 = rhs_sign * b2->slope / s;
    const double w1 = a1 / (double)b1->scale_factor * (double)phi;
    const double w2 = a2 / (double)b2->scale_factor * (double)phi;
    for (int k = 0; k < KEPT; ++k)
        out->coeffs[k] = clamp_coeff(w1 * (double)b1->coeffs[k] + w2 * (double)b2->coeffs[k]);
    return ORC_OK;
}

int orc_add(const orc_block* a, const orc_block* b, orc_block* out) { return combine(a, b, +1.0, out); }
int orc_sub(const orc_block* a, const orc_block* b, orc_block* out) { return combine(a, b, -1.0, out); }

/* H/block_ops.hpp:74-77 */
int orc_scale(const orc_block* a, double c, orc_block* out) {
    if (!isfinite(c)) return ORC_INVALID; /* "scale: non-finite constant" */
    *out = *a;
    out->first = a->first * c;
    out->slope = a->slope * c;
    return ORC_OK;
}

/* H/block_ops.hpp:87-95 */
void orc_reconstruct_rows(const orc_block* b, int last_row, double out[64]) {
    double p[64];
    memset(out, 0, 64 * sizeof(double));
    orc_dequantize_prediction(b, p);
    integrate_rows(b, p, last_row, out);
}

/* H/block_ops.hpp:99-115 */
void orc_reconstruct_cols(const orc_block* b, int last_col, double out[64]) {
    double p[64];
    memset(out, 0, 64 * sizeof(double));
    orc_dequantize_prediction(b, p);
    const double s = b->slope;
    out[0] = b->first;
    for (int i = 1; i < BD; ++i) out[i * BD] = out[(i - 1) * BD] + s * p[i * BD];
    for (int j = 1; j <= last_col; ++j) {
        out[j] = out[j - 1] + s * p[j];
        for (int i = 1; i < BD; ++i)
            out[i * BD + j] = (out[(i - 1) * BD + j] + out[i * BD + j - 1]) / 2.0 + s * p[i * BD + j];
    }
}

/* H/block_ops.hpp:119-127 */
double orc_dot(const orc_block* a, const orc_block* b, int i, int j) {
    double rows[64], cols[64];
    orc_reconstruct_rows(a, i, rows);
    orc_reconstruct_cols(b, j, cols);
    double r = 0.0;
    for (int k = 0; k < BD; ++k) r += rows[i * BD + k] * cols[k * BD + j];
    return r;
}

/* H/block_ops.hpp:131-142 */
void orc_block_mul(const orc_block* a, const orc_block* b, double out[64]) {
    double d1[64], d2[64];
    orc_decompress_block(a, d1);
    orc_decompress_block(b, d2);
    for (int i = 0; i < BD; ++i)
        for (int j = 0; j < BD; ++j) {
            double r = 0.0;
            for (int k = 0; k < BD; ++k) r += d1[i * BD + k] * d2[k * BD + j];
            out[i * BD + j] = r;
        }
}

/* ---- matrix level: H/matrix.hpp ------------------------------------------ */

static size_t nblk(size_t n) { return (n + BD - 1) / BD; }

/* H/matrix.hpp:97-111 with extract_tile/padded_at (:72-84): edge replication. */
int orc_compress_matrix(const double* v, size_t rows, size_t cols, orc_block* out) {
    if (rows == 0 || cols == 0) return ORC_INVALID; /* "compress_matrix: empty matrix" */
    const size_t br = nblk(rows), bc = nblk(cols);
    int status = ORC_OK;
    for (size_t t = 0; t < br * bc; ++t) {
        const size_t bi = t / bc, bj = t % bc;
        double tile[64];
        for (int i = 0; i < BD; ++i)
            for (int j = 0; j < BD; ++j) {
                size_t r = bi * BD + i, c = bj * BD + j;
                if (r >= rows) r = rows - 1;
                if (c >= cols) c = cols - 1;
                tile[i * BD + j] = v[r * cols + c];
            }
        const int st = orc_compress_block(tile, &out[t]);
        if (st != ORC_OK && status == ORC_OK) status = st;
    }
    return status;
}

/* H/matrix.hpp:113-126: decompress every tile, crop the padding. */
void orc_decompress_matrix(const orc_block* in, size_t rows, size_t cols, double* out) {
    const size_t br = nblk(rows), bc = nblk(cols);
    for (size_t t = 0; t < br * bc; ++t) {
        const size_t bi = t / bc, bj = t % bc;
        double tile[64];
        orc_decompress_block(&in[t], tile);
        for (size_t i = 0; i < BD && bi * BD + i < rows; ++i)
            for (size_t j = 0; j < BD && bj * BD + j < cols; ++j)
                out[(bi * BD + i) * cols + bj * BD + j] = tile[i * BD + j];
    }
}

/* H/matrix.hpp:128-151 (dimension checks are the caller's job here). */
int orc_mat_add(const orc_block* a, const orc_block* b, size_t n, orc_block* out) {
    int status = ORC_OK;
    for (size_t t = 0; t < n; ++t) {
        const int st = orc_add(&a[t], &b[t], &out[t]);
        if (st != ORC_OK && status == ORC_OK) status = st;
    }
    return status;
}

int orc_mat_sub(const orc_block* a, const orc_block* b, size_t n, orc_block* out) {
    int status = ORC_OK;
    for (size_t t = 0; t < n; ++t) {
        const int st = orc_sub(&a[t], &b[t], &out[t]);
        if (st != ORC_OK && status == ORC_OK) status = st;
    }
    return status;
}

int orc_mat_scale(const orc_block* a, double c, size_t n, orc_block* out) {
    for (size_t t = 0; t < n; ++t)
        if (orc_scale(&a[t], c, &out[t]) != ORC_OK) return ORC_INVALID;
    return ORC_OK;
}

/* H/matrix.hpp:157-173 */
int orc_mat_dot(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                size_t b_rows, size_t b_cols, size_t i, size_t j, double* out) {
    if (a_cols != b_rows) return ORC_INVALID; /* "mat_dot: inner dimension mismatch" */
    if (i >= a_rows || j >= b_cols) return ORC_RANGE; /* "mat_dot: index out of range" */
    const size_t a_bc = nblk(a_cols), b_bc = nblk(b_cols);
    const size_t bi = i / BD, bj = j / BD;
    const int ri = (int)(i % BD), cj = (int)(j % BD);
    double r = 0.0;
    for (size_t t = 0; t < a_bc; ++t) {
        double rows[64], cols[64];
        orc_reconstruct_rows(&a[bi * a_bc + t], ri, rows);
        orc_reconstruct_cols(&b[t * b_bc + bj], cj, cols);
        const size_t rem = a_cols - t * BD;
        const int klim = (int)(rem < BD ? rem : BD);
        for (int k = 0; k < klim; ++k) r += rows[ri * BD + k] * cols[k * BD + cj];
    }
    *out = r;
    return ORC_OK;
}

/* H/matrix.hpp:188-202 (accumulate_product_tile): ascending t, then i, k, j. */
static void product_tile(const double* ta, const double* tb, size_t a_bc, size_t b_bc,
                         size_t inner, size_t I, size_t J, double acc[64]) {
    memset(acc, 0, 64 * sizeof(double));
    for (size_t t = 0; t < a_bc; ++t) {
        const double* da = ta + (I * a_bc + t) * 64;
        const double* db = tb + (t * b_bc + J) * 64;
        const size_t rem = inner - t * BD;
        const int klim = (int)(rem < BD ? rem : BD);
        for (int i = 0; i < BD; ++i)
            for (int k = 0; k < klim; ++k) {
                const double av = da[i * BD + k];
                for (int j = 0; j < BD; ++j) acc[i * BD + j] += av * db[k * BD + j];
            }
    }
}

#include <stdlib.h>

static double* decompress_tiles(const orc_block* m, size_t n) {
    double* t = (double*)malloc(n * 64 * sizeof(double));
    for (size_t k = 0; k < n; ++k) orc_decompress_block(&m[k], t + k * 64);
    return t;
}

/* H/matrix.hpp:239-250 */
int orc_mat_mul_dense(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                      size_t b_rows, size_t b_cols, double* out) {
    if (a_cols != b_rows) return ORC_INVALID; /* "mat_mul: inner dimension mismatch" */
    const size_t a_br = nblk(a_rows), a_bc = nblk(a_cols), b_br = nblk(b_rows), b_bc = nblk(b_cols);
    double* ta = decompress_tiles(a, a_br * a_bc);
    double* tb = decompress_tiles(b, b_br * b_bc);
    for (size_t I = 0; I < a_br; ++I)
        for (size_t J = 0; J < b_bc; ++J) {
            double acc[64];
            product_tile(ta, tb, a_bc, b_bc, a_cols, I, J, acc);
            for (size_t i = 0; i < BD && I * BD + i < a_rows; ++i)
                for (size_t j = 0; j < BD && J * BD + j < b_cols; ++j)
                    out[(I * BD + i) * b_cols + J * BD + j] = acc[i * BD + j];
        }
    free(ta);
    free(tb);
    return ORC_OK;
}

/* H/matrix.hpp:223-235: each full 8x8 accumulator tile (padding rows and
 * columns included) is compressed once. */
int orc_mat_mul(const orc_block* a, size_t a_rows, size_t a_cols, const orc_block* b,
                size_t b_rows, size_t b_cols, orc_block* out) {
    if (a_cols != b_rows) return ORC_INVALID;
    const size_t a_br = nblk(a_rows), a_bc = nblk(a_cols), b_br = nblk(b_rows), b_bc = nblk(b_cols);
    double* ta = decompress_tiles(a, a_br * a_bc);
    double* tb = decompress_tiles(b, b_br * b_bc);
    int status = ORC_OK;
    for (size_t I = 0; I < a_br; ++I)
        for (size_t J = 0; J < b_bc; ++J) {
            double acc[64];
            product_tile(ta, tb, a_bc, b_bc, a_cols, I, J, acc);
            const int st = orc_compress_block(acc, &out[I * b_bc + J]);
            if (st != ORC_OK && status == ORC_OK) status = st;
        }
    free(ta);
    free(tb);
    return status;
}

/* Config-2 restatement built only from decompress_matrix (H/matrix.hpp:113-126)
 * and the ascending loop of ref::dot (H/matrix.hpp:280-286). */
int orc_rowdot(const orc_block* a, const orc_block* b, size_t rows, size_t cols, double* r) {
    const size_t bc = nblk(cols);
    for (size_t i = 0; i < rows; ++i) r[i] = 0.0;
    /* walk block-rows so only one strip of tiles is live */
    for (size_t bi = 0; bi < nblk(rows); ++bi) {
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (size_t t = 0; t < bc; ++t) {
            double da[64], db[64];
            orc_decompress_block(&a[bi * bc + t], da);
            orc_decompress_block(&b[bi * bc + t], db);
            const size_t rem = cols - t * BD;
            const int jlim = (int)(rem < BD ? rem : BD);
            for (int i = 0; i < BD; ++i)
                for (int j = 0; j < jlim; ++j) acc[i] += da[i * BD + j] * db[i * BD + j];
        }
        for (int i = 0; i < BD && bi * BD + i < rows; ++i) r[bi * BD + i] = acc[i];
    }
    return ORC_OK;
}

double orc_sum_ascending(const double* v, size_t n) {
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += v[k];
    return s;
}
