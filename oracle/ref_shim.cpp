// ref_shim.cpp -- CPU ORACLE build of the REAL reference (test infrastructure only).
//
// This translation unit is compiled by oracle/Makefile against the reference's
// own headers where they lie (-I /root/reference/proj/include), with the
// reference's pinned flags (-std=c++20 -O2 -ffp-contract=off,
// proj/CMakeLists.txt:15-18), into oracle/_ref/libblaz_ref.so.  It copies no
// reference source: it only adapts blaz::compress_matrix & co.
// (H/matrix.hpp:97-250) to plain C entry points so Python tests can
//   * pin the C restatement (oracle/blaz_oracle.c) and generate golden vectors,
//   * time the reference CPU path (bench.py --impl reference / cpu_baseline).
// Blocks cross this boundary as the reference's own 48-byte
// blaz::compressed_block (H/block.hpp:33-38).
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>

#include "blaz/blaz.hpp"

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 out_of_range, 3 other
int run(auto&& fn) {
    try {
        fn();
        g_err.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

blaz::compressed_matrix make_cm(const blaz::compressed_block* blocks, std::size_t rows,
                                std::size_t cols) {
    blaz::compressed_matrix cm;
    cm.rows = rows;
    cm.cols = cols;
    cm.block_rows = (rows + 7) / 8;
    cm.block_cols = (cols + 7) / 8;
    cm.blocks.assign(blocks, blocks + cm.block_rows * cm.block_cols);
    return cm;
}

}  // namespace

static_assert(sizeof(blaz::compressed_block) == 48, "AoS block layout");

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

void ref_dct_basis(double* t) {
    const blaz::block8& b = blaz::detail::dct_basis();
    std::memcpy(t, b.a.data(), 64 * sizeof(double));
}

int ref_compress_block(const double* m, blaz::compressed_block* out) {
    return run([&] {
        blaz::block8 b;
        std::memcpy(b.a.data(), m, 64 * sizeof(double));
        *out = blaz::compress_block(b);
    });
}

void ref_decompress_block(const blaz::compressed_block* b, double* out) {
    const blaz::block8 d = blaz::decompress_block(*b);
    std::memcpy(out, d.a.data(), 64 * sizeof(double));
}

int ref_predict_indices(const double* m, unsigned char* idx) {
    return run([&] {
        blaz::block8 b;
        std::memcpy(b.a.data(), m, 64 * sizeof(double));
        const auto n = blaz::normalize(b);
        const double s = blaz::mean_slope(n.deltas);
        blaz::block8 slopes;
        for (int k = 0; k < 64; ++k) slopes.a[k] = n.deltas.a[k] / s;
        const auto p = blaz::predict(slopes, s);
        std::memcpy(idx, p.prediction.indices.data(), 64);
    });
}

int ref_add(const blaz::compressed_block* a, const blaz::compressed_block* b,
            blaz::compressed_block* out) {
    return run([&] { *out = blaz::add(*a, *b); });
}
int ref_sub(const blaz::compressed_block* a, const blaz::compressed_block* b,
            blaz::compressed_block* out) {
    return run([&] { *out = blaz::sub(*a, *b); });
}
int ref_dot(const blaz::compressed_block* a, const blaz::compressed_block* b, int i, int j,
            double* out) {
    return run([&] { *out = blaz::dot(*a, *b, i, j); });
}

// ---- matrix level, array in / array out -----------------------------------
int ref_compress_matrix(const double* v, std::size_t rows, std::size_t cols, unsigned threads,
                        blaz::compressed_block* out) {
    return run([&] {
        blaz::dense_matrix m;
        m.rows = rows;
        m.cols = cols;
        m.values.assign(v, v + rows * cols);
        const auto cm = blaz::compress_matrix(m, threads);
        std::memcpy(out, cm.blocks.data(), cm.blocks.size() * sizeof(blaz::compressed_block));
    });
}

int ref_decompress_matrix(const blaz::compressed_block* in, std::size_t rows, std::size_t cols,
                          unsigned threads, double* out) {
    return run([&] {
        const auto d = blaz::decompress_matrix(make_cm(in, rows, cols), threads);
        std::memcpy(out, d.values.data(), d.values.size() * sizeof(double));
    });
}

int ref_mat_binop(int op, const blaz::compressed_block* a, const blaz::compressed_block* b,
                  std::size_t rows, std::size_t cols, unsigned threads,
                  blaz::compressed_block* out) {
    return run([&] {
        const auto ca = make_cm(a, rows, cols);
        const auto cb = make_cm(b, rows, cols);
        const auto r = op == 0 ? blaz::mat_add(ca, cb, threads) : blaz::mat_sub(ca, cb, threads);
        std::memcpy(out, r.blocks.data(), r.blocks.size() * sizeof(blaz::compressed_block));
    });
}

int ref_mat_scale(const blaz::compressed_block* a, std::size_t rows, std::size_t cols, double c,
                  unsigned threads, blaz::compressed_block* out) {
    return run([&] {
        const auto r = blaz::mat_scale(make_cm(a, rows, cols), c, threads);
        std::memcpy(out, r.blocks.data(), r.blocks.size() * sizeof(blaz::compressed_block));
    });
}

int ref_mat_dot(const blaz::compressed_block* a, std::size_t ar, std::size_t ac,
                const blaz::compressed_block* b, std::size_t br, std::size_t bc, std::size_t i,
                std::size_t j, double* out) {
    return run([&] { *out = blaz::mat_dot(make_cm(a, ar, ac), make_cm(b, br, bc), i, j); });
}

int ref_mat_mul(const blaz::compressed_block* a, std::size_t ar, std::size_t ac,
                const blaz::compressed_block* b, std::size_t br, std::size_t bc,
                unsigned threads, blaz::compressed_block* out) {
    return run([&] {
        const auto r = blaz::mat_mul(make_cm(a, ar, ac), make_cm(b, br, bc), threads);
        std::memcpy(out, r.blocks.data(), r.blocks.size() * sizeof(blaz::compressed_block));
    });
}

int ref_mat_mul_dense(const blaz::compressed_block* a, std::size_t ar, std::size_t ac,
                      const blaz::compressed_block* b, std::size_t br, std::size_t bc,
                      unsigned threads, double* out) {
    return run([&] {
        const auto r = blaz::mat_mul_dense(make_cm(a, ar, ac), make_cm(b, br, bc), threads);
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
    });
}

// ---- .blzc container through the reference's io.hpp (H/io.hpp:93-134) ------
long long ref_write_compressed(const blaz::compressed_block* blocks, std::size_t rows, std::size_t cols,
                               unsigned char* out, std::size_t cap) {
    long long n = -1;
    const int st = run([&] {
        std::ostringstream os;
        blaz::write_compressed(make_cm(blocks, rows, cols), os);
        const std::string b = os.str();
        if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
        n = (long long)b.size();
    });
    return st ? -1 : n;
}

int ref_read_compressed(const unsigned char* bytes, std::size_t n, std::size_t* rows, std::size_t* cols,
                        blaz::compressed_block* out, std::size_t cap) {
    return run([&] {
        std::istringstream is(std::string(reinterpret_cast<const char*>(bytes), n));
        const auto cm = blaz::read_compressed(is);
        *rows = cm.rows;
        *cols = cm.cols;
        if (cm.blocks.size() <= cap) std::memcpy(out, cm.blocks.data(), cm.blocks.size() * sizeof(blaz::compressed_block));
    });
}

// ---- handle API for timing the reference without per-call marshalling -----
void* ref_dense_new(const double* v, std::size_t rows, std::size_t cols) {
    auto* m = new blaz::dense_matrix;
    m->rows = rows;
    m->cols = cols;
    m->values.assign(v, v + rows * cols);
    return m;
}
void ref_dense_free(void* h) { delete static_cast<blaz::dense_matrix*>(h); }
void ref_cm_free(void* h) { delete static_cast<blaz::compressed_matrix*>(h); }

void* ref_h_compress(void* dense, unsigned threads) {
    void* out = nullptr;
    run([&] {
        out = new blaz::compressed_matrix(
            blaz::compress_matrix(*static_cast<blaz::dense_matrix*>(dense), threads));
    });
    return out;
}
void* ref_h_decompress(void* cm, unsigned threads) {
    return new blaz::dense_matrix(
        blaz::decompress_matrix(*static_cast<blaz::compressed_matrix*>(cm), threads));
}
void* ref_h_add(void* a, void* b, unsigned threads) {
    return new blaz::compressed_matrix(blaz::mat_add(
        *static_cast<blaz::compressed_matrix*>(a), *static_cast<blaz::compressed_matrix*>(b), threads));
}
void* ref_h_sub(void* a, void* b, unsigned threads) {
    return new blaz::compressed_matrix(blaz::mat_sub(
        *static_cast<blaz::compressed_matrix*>(a), *static_cast<blaz::compressed_matrix*>(b), threads));
}
void* ref_h_scale(void* a, double c, unsigned threads) {
    return new blaz::compressed_matrix(
        blaz::mat_scale(*static_cast<blaz::compressed_matrix*>(a), c, threads));
}
void* ref_h_mul(void* a, void* b, unsigned threads) {
    return new blaz::compressed_matrix(blaz::mat_mul(
        *static_cast<blaz::compressed_matrix*>(a), *static_cast<blaz::compressed_matrix*>(b), threads));
}
const double* ref_dense_data(void* h) { return static_cast<blaz::dense_matrix*>(h)->values.data(); }
const void* ref_cm_blocks(void* h) { return static_cast<blaz::compressed_matrix*>(h)->blocks.data(); }

}  // extern "C"
