// blaz/blaz.hpp -- C++ drop-in for the reference's public API, backed by the
// sm_100a kernels of libblaz_cuda.so through the C ABI (include/blaz_cuda.h).
//
// A program written against the reference (proj/include/blaz/blaz.hpp) builds
// against this header unchanged and links -lblaz_cuda: the same types
// (block8, compressed_block, dense_matrix, compressed_matrix,
// partial_reconstruction) with the same member layout, and the same functions
// with the same signatures, exception types and messages:
//
//   compress_matrix / decompress_matrix      H/matrix.hpp:97-126
//   mat_add / mat_sub / mat_scale            H/matrix.hpp:128-151
//   mat_dot                                  H/matrix.hpp:157-173
//   mat_mul / mat_mul_dense                  H/matrix.hpp:223-250
//   compress_block / decompress_block        H/codec.hpp:130-146, :180-185
//   dequantize_prediction                    H/codec.hpp:150-158
//   add / sub / scale / dot / block_mul      H/block_ops.hpp:65-142
//   reconstruct_rows / reconstruct_cols      H/block_ops.hpp:87-115
//   normalize / denormalize / mean_slope / predict / quantize_coeffs,
//   dct2 / idct2 (stage functions)           H/codec.hpp:12-125, H/dct.hpp:14-70
//   round_half_away / clamp_index / clamp_coeff / all_finite  H/block.hpp:61-87
//   write/read_compressed, write/read_dense,
//   import_csv                               H/io.hpp:93-190
//   gen_matrix, mean_relative_error, accuracy_suite, bench_suite, ...
//                                            H/bench.hpp (blaz/harness.hpp)
//   ref::add/sub/scale/dot/mul               H/matrix.hpp:253-300 (dense baselines)
//
// Every compressed-domain result is computed on the GPU (one process-wide
// context on device $BLZ_DEVICE, default 0); `threads` is accepted and ignored.
// The ref:: functions are the reference's uncompressed CPU baselines, kept for
// source compatibility of benchmarks and tests.
#ifndef BLAZ_DROPIN_BLAZ_HPP
#define BLAZ_DROPIN_BLAZ_HPP

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <iterator>
#include <mutex>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../blaz_cuda.h"

namespace blaz {

inline constexpr int block_dim = 8;
inline constexpr int block_cells = block_dim * block_dim;
inline constexpr int kept_coeff_count = 28;
inline constexpr int block_payload_bytes = 8 + 8 + 1 + kept_coeff_count;
inline constexpr double compression_rate =
    double(block_cells * 8 * 8) / double(block_payload_bytes * 8);

struct block8 {
    std::array<double, block_cells> a{};
    double& operator()(int r, int c) { return a[r * block_dim + c]; }
    const double& operator()(int r, int c) const { return a[r * block_dim + c]; }
};

struct compressed_block {
    double first = 0.0;
    double slope = 0.0;
    std::uint8_t scale_factor = 1;
    std::array<std::int8_t, kept_coeff_count> coeffs{};
};
static_assert(sizeof(compressed_block) == sizeof(blz_block), "48-byte AoS record");
static_assert(offsetof(compressed_block, scale_factor) == offsetof(blz_block, scale_factor), "layout");
static_assert(offsetof(compressed_block, coeffs) == offsetof(blz_block, coeffs), "layout");

struct coeff_position {
    std::uint8_t row;
    std::uint8_t col;
};

// Frozen keep-set order: row 0, row 1, column 0 rows 2..7, column 1 rows 2..7.
inline constexpr std::array<coeff_position, kept_coeff_count> kept_coeff_positions = [] {
    std::array<coeff_position, kept_coeff_count> p{};
    for (int k = 0; k < kept_coeff_count; ++k) {
        if (k < 16) p[k] = {std::uint8_t(k / 8), std::uint8_t(k % 8)};
        else if (k < 22) p[k] = {std::uint8_t(k - 14), 0};
        else p[k] = {std::uint8_t(k - 20), 1};
    }
    return p;
}();

struct dense_matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> values;

    dense_matrix() = default;
    dense_matrix(std::size_t r, std::size_t c) : rows(r), cols(c), values(r * c, 0.0) {}
    double& operator()(std::size_t r, std::size_t c) { return values[r * cols + c]; }
    const double& operator()(std::size_t r, std::size_t c) const { return values[r * cols + c]; }
};

struct compressed_matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::size_t block_rows = 0;
    std::size_t block_cols = 0;
    std::vector<compressed_block> blocks;

    compressed_block& block(std::size_t br, std::size_t bc) { return blocks[br * block_cols + bc]; }
    const compressed_block& block(std::size_t br, std::size_t bc) const { return blocks[br * block_cols + bc]; }
};

// File-format failures (H/io.hpp:20-23).
class io_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

struct partial_reconstruction {
    block8 values;
    int extent = 0;
};

namespace gpu {

// One context per calling thread (created on first use, destroyed at thread
// exit).  A context owns its stream, scratch buffers, worklists and error
// string, so concurrent calls from several threads never share mutable state:
// the reference's functions are pure and re-entrant, and so are these.
struct thread_context {
    blz_ctx* ctx = nullptr;
    ~thread_context() {
        if (ctx) blz_ctx_destroy(ctx);
    }
};

inline blz_ctx* context() {
    thread_local thread_context tc;
    if (!tc.ctx) {
        const char* d = std::getenv("BLZ_DEVICE");
        if (blz_ctx_create(d ? std::atoi(d) : 0, nullptr, &tc.ctx) != BLZ_OK) {
            tc.ctx = nullptr;
            throw std::runtime_error("blaz: cannot create the CUDA context");
        }
    }
    return tc.ctx;
}

inline void check(blz_status st) {
    if (st == BLZ_OK) return;
    const std::string msg = blz_last_error(context());
    if (st == BLZ_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == BLZ_OUT_OF_RANGE) throw std::out_of_range(msg);
    if (st == BLZ_OUT_OF_MEMORY) throw std::bad_alloc();
    if (st == BLZ_IO_ERROR) throw io_error(msg);
    throw std::runtime_error("blaz: " + msg);
}

inline blz_block* raw(compressed_block* b) { return reinterpret_cast<blz_block*>(b); }
inline const blz_block* raw(const compressed_block* b) { return reinterpret_cast<const blz_block*>(b); }

inline compressed_matrix shaped(std::size_t rows, std::size_t cols) {
    compressed_matrix m;
    m.rows = rows;
    m.cols = cols;
    m.block_rows = (rows + block_dim - 1) / block_dim;
    m.block_cols = (cols + block_dim - 1) / block_dim;
    m.blocks.resize(m.block_rows * m.block_cols);
    return m;
}

}  // namespace gpu

// ---- matrix level ------------------------------------------------------------
inline compressed_matrix compress_matrix(const dense_matrix& m, unsigned threads = 1) {
    if (m.rows == 0 || m.cols == 0) throw std::invalid_argument("compress_matrix: empty matrix");
    compressed_matrix cm = gpu::shaped(m.rows, m.cols);
    gpu::check(blz_compress_matrix(gpu::context(), m.values.data(), m.rows, m.cols, gpu::raw(cm.blocks.data()),
                                   threads));
    return cm;
}

inline dense_matrix decompress_matrix(const compressed_matrix& cm, unsigned threads = 1) {
    dense_matrix m(cm.rows, cm.cols);
    if (cm.blocks.empty()) return m;
    gpu::check(blz_decompress_matrix(gpu::context(), gpu::raw(cm.blocks.data()), cm.rows, cm.cols,
                                     m.values.data(), threads));
    return m;
}

inline compressed_matrix mat_add(const compressed_matrix& a, const compressed_matrix& b, unsigned threads = 1) {
    compressed_matrix out = gpu::shaped(a.rows, a.cols);
    gpu::check(blz_mat_add(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols, gpu::raw(b.blocks.data()),
                           b.rows, b.cols, gpu::raw(out.blocks.data()), threads));
    return out;
}

inline compressed_matrix mat_sub(const compressed_matrix& a, const compressed_matrix& b, unsigned threads = 1) {
    compressed_matrix out = gpu::shaped(a.rows, a.cols);
    gpu::check(blz_mat_sub(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols, gpu::raw(b.blocks.data()),
                           b.rows, b.cols, gpu::raw(out.blocks.data()), threads));
    return out;
}

inline compressed_matrix mat_scale(const compressed_matrix& a, double c, unsigned threads = 1) {
    compressed_matrix out = gpu::shaped(a.rows, a.cols);
    out.blocks.resize(a.blocks.size());
    if (a.blocks.empty()) return out;
    gpu::check(blz_mat_scale(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols, c,
                             gpu::raw(out.blocks.data()), threads));
    return out;
}

inline double mat_dot(const compressed_matrix& a, const compressed_matrix& b, std::size_t i, std::size_t j) {
    double r = 0.0;
    gpu::check(blz_mat_dot(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols, gpu::raw(b.blocks.data()),
                           b.rows, b.cols, i, j, &r));
    return r;
}

inline compressed_matrix mat_mul(const compressed_matrix& a, const compressed_matrix& b, unsigned threads = 1) {
    if (a.cols != b.rows) throw std::invalid_argument("mat_mul: inner dimension mismatch");
    compressed_matrix out = gpu::shaped(a.rows, b.cols);
    gpu::check(blz_mat_mul(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols, gpu::raw(b.blocks.data()),
                           b.rows, b.cols, gpu::raw(out.blocks.data()), threads));
    return out;
}

inline dense_matrix mat_mul_dense(const compressed_matrix& a, const compressed_matrix& b, unsigned threads = 1) {
    if (a.cols != b.rows) throw std::invalid_argument("mat_mul: inner dimension mismatch");
    dense_matrix out(a.rows, b.cols);
    gpu::check(blz_mat_mul_dense(gpu::context(), gpu::raw(a.blocks.data()), a.rows, a.cols,
                                 gpu::raw(b.blocks.data()), b.rows, b.cols, out.values.data(), threads));
    return out;
}

// ---- scalar helpers of the codec (H/block.hpp:61-87) ---------------------------
// Reference semantics, including the x86 conversion of out-of-range values to
// INT64_MIN inside round_half_away; used by callers and by slope_quantizer.
inline double round_half_away(double x) {
    const double t = (x >= -9223372036854775808.0 && x < 9223372036854775808.0)
                         ? double(static_cast<long long>(x))
                         : -9223372036854775808.0;
    const double frac = x - t;
    if (frac >= 0.5) return t + 1.0;
    if (frac <= -0.5) return t - 1.0;
    return t;
}

inline int clamp_index(double x) {
    const double r = round_half_away(x);
    return r <= 0.0 ? 0 : (r >= 255.0 ? 255 : int(r));
}

inline std::int8_t clamp_coeff(double x) {
    const double r = round_half_away(x);
    return r <= -127.0 ? std::int8_t(-127) : (r >= 127.0 ? std::int8_t(127) : std::int8_t(r));
}

inline bool all_finite(const block8& b) {
    for (double v : b.a)
        if (!std::isfinite(v)) return false;
    return true;
}

// ---- stage functions (H/codec.hpp:12-125, H/dct.hpp:14-70), on the GPU ----------
struct normalization {
    double first = 0.0;
    block8 deltas;
};

struct slope_quantizer {
    double lo = 0.0;
    double step = 0.0;
    static constexpr int levels = 256;
    int encode(double v) const { return step == 0.0 ? 0 : clamp_index((v - lo) / step); }
    double decode(int k) const { return lo + k * step; }
};

struct prediction_block {
    std::array<std::uint8_t, block_cells> indices{};
    block8 snapped;
};

struct prediction_result {
    prediction_block prediction;
    slope_quantizer quantizer;
};

struct coeff_quantization {
    std::uint8_t scale_factor = 1;
    std::array<std::int8_t, kept_coeff_count> coeffs{};
};

inline normalization normalize(const block8& m) {
    normalization out;
    gpu::check(blz_normalize_blocks(gpu::context(), m.a.data(), 1, &out.first, out.deltas.a.data()));
    return out;
}

inline block8 denormalize(double first, const block8& deltas) {
    block8 out;
    gpu::check(blz_denormalize_blocks(gpu::context(), &first, deltas.a.data(), 1, out.a.data()));
    return out;
}

inline double mean_slope(const block8& deltas) {
    double s = 0.0;
    gpu::check(blz_mean_slope_blocks(gpu::context(), deltas.a.data(), 1, &s));
    return s;
}

inline prediction_result predict(const block8& slopes, double slope_mean) {
    prediction_result out;
    gpu::check(blz_predict_blocks(gpu::context(), slopes.a.data(), &slope_mean, 1, out.prediction.indices.data(),
                                  out.prediction.snapped.a.data(), &out.quantizer.lo, &out.quantizer.step));
    return out;
}

inline coeff_quantization quantize_coeffs(const block8& d) {
    coeff_quantization out;
    gpu::check(blz_quantize_coeffs_blocks(gpu::context(), d.a.data(), 1, &out.scale_factor, out.coeffs.data()));
    return out;
}

inline block8 dct2(const block8& x) {
    block8 out;
    gpu::check(blz_dct2_blocks(gpu::context(), x.a.data(), 1, out.a.data()));
    return out;
}

inline block8 idct2(const block8& d) {
    block8 out;
    gpu::check(blz_idct2_blocks(gpu::context(), d.a.data(), 1, out.a.data()));
    return out;
}

namespace detail {
// The context's uploaded basis (H/dct.hpp:14-27, computed on the host with glibc).
inline const block8& dct_basis() {
    static const block8 t = [] {
        block8 m;
        gpu::check(blz_ctx_basis(gpu::context(), m.a.data()));
        return m;
    }();
    return t;
}
}  // namespace detail

// ---- block level (batched calls of one block) ----------------------------------
inline compressed_block compress_block(const block8& m) {
    compressed_block out;
    gpu::check(blz_compress_blocks(gpu::context(), m.a.data(), 1, gpu::raw(&out)));
    return out;
}

inline block8 decompress_block(const compressed_block& cb) {
    block8 out;
    gpu::check(blz_decompress_blocks(gpu::context(), gpu::raw(&cb), 1, out.a.data()));
    return out;
}

inline block8 dequantize_prediction(const compressed_block& cb) {
    block8 out;
    gpu::check(blz_dequantize_blocks(gpu::context(), gpu::raw(&cb), 1, out.a.data()));
    return out;
}

inline compressed_block add(const compressed_block& b1, const compressed_block& b2) {
    compressed_block out;
    gpu::check(blz_mat_add(gpu::context(), gpu::raw(&b1), 8, 8, gpu::raw(&b2), 8, 8, gpu::raw(&out), 1));
    return out;
}

inline compressed_block sub(const compressed_block& b1, const compressed_block& b2) {
    compressed_block out;
    gpu::check(blz_mat_sub(gpu::context(), gpu::raw(&b1), 8, 8, gpu::raw(&b2), 8, 8, gpu::raw(&out), 1));
    return out;
}

inline compressed_block scale(const compressed_block& b, double c) {
    compressed_block out;
    gpu::check(blz_mat_scale(gpu::context(), gpu::raw(&b), 8, 8, c, gpu::raw(&out), 1));
    return out;
}

// Rows 0..last_row of decompress_block(b) (bitwise); other rows stay +0.0.
inline partial_reconstruction reconstruct_rows(const compressed_block& b, int last_row) {
    if (last_row < 0 || last_row >= block_dim)
        throw std::out_of_range("reconstruct_rows: row index out of range");
    partial_reconstruction out;
    out.extent = last_row + 1;
    const block8 full = decompress_block(b);
    for (int i = 0; i <= last_row; ++i)
        for (int j = 0; j < block_dim; ++j) out.values(i, j) = full(i, j);
    return out;
}

// Columns 0..last_col of decompress_block(b) (bitwise); other columns stay +0.0.
inline partial_reconstruction reconstruct_cols(const compressed_block& b, int last_col) {
    if (last_col < 0 || last_col >= block_dim)
        throw std::out_of_range("reconstruct_cols: column index out of range");
    partial_reconstruction out;
    out.extent = last_col + 1;
    const block8 full = decompress_block(b);
    for (int i = 0; i < block_dim; ++i)
        for (int j = 0; j <= last_col; ++j) out.values(i, j) = full(i, j);
    return out;
}

inline double dot(const compressed_block& b1, const compressed_block& b2, int i, int j) {
    if (i < 0 || i >= block_dim || j < 0 || j >= block_dim) throw std::out_of_range("dot: index out of range");
    double r = 0.0;
    gpu::check(blz_mat_dot(gpu::context(), gpu::raw(&b1), 8, 8, gpu::raw(&b2), 8, 8, std::size_t(i),
                           std::size_t(j), &r));
    return r;
}

inline block8 block_mul(const compressed_block& b1, const compressed_block& b2) {
    block8 out;
    gpu::check(blz_mat_mul_dense(gpu::context(), gpu::raw(&b1), 8, 8, gpu::raw(&b2), 8, 8, out.a.data(), 1));
    return out;
}

// ---- .blzc container (H/io.hpp:93-134), packed/validated on the GPU ----------------
inline std::size_t write_compressed(const compressed_matrix& cm, std::ostream& out) {
    std::vector<std::uint8_t> bytes(blz_blzc_bytes(cm.rows, cm.cols));
    std::uint64_t n = 0;
    gpu::check(blz_write_compressed(gpu::context(), gpu::raw(cm.blocks.data()), cm.rows, cm.cols, bytes.data(),
                                    bytes.size(), &n));
    out.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(n));
    if (!out) throw io_error("write_compressed: write failed");
    return std::size_t(n);
}

inline compressed_matrix read_compressed(std::istream& in) {
    const std::vector<std::uint8_t> bytes{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    std::uint64_t rows = 0, cols = 0;
    gpu::check(blz_read_compressed(gpu::context(), bytes.data(), bytes.size(), &rows, &cols, nullptr, 0));
    compressed_matrix cm = gpu::shaped(rows, cols);
    gpu::check(blz_read_compressed(gpu::context(), bytes.data(), bytes.size(), &rows, &cols,
                                   gpu::raw(cm.blocks.data()), cm.blocks.size()));
    return cm;
}

// ---- dense container and CSV import (H/io.hpp:135-190), host byte formatting ------
// "BLZD", version 1, u32 rows, u32 cols (little endian), then rows*cols binary64.
namespace detail {

inline void put_le(std::string& out, std::uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(char((v >> (8 * i)) & 0xff));
}

inline std::uint64_t get_le(const unsigned char* p, int bytes) {
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= std::uint64_t(p[i]) << (8 * i);
    return v;
}

}  // namespace detail

inline std::size_t write_dense(const dense_matrix& m, std::ostream& out) {
    std::string bytes;
    bytes.reserve(13 + m.values.size() * 8);
    bytes.append("BLZD", 4);
    bytes.push_back(char(1));
    detail::put_le(bytes, std::uint32_t(m.rows), 4);
    detail::put_le(bytes, std::uint32_t(m.cols), 4);
    for (double v : m.values) {
        std::uint64_t u;
        std::memcpy(&u, &v, 8);
        detail::put_le(bytes, u, 8);
    }
    out.write(bytes.data(), std::streamsize(bytes.size()));
    if (!out) throw io_error("write_dense: write failed");
    return bytes.size();
}

inline dense_matrix read_dense(std::istream& in) {
    unsigned char h[13];
    in.read(reinterpret_cast<char*>(h), 13);
    if (in.gcount() != 13) throw io_error("dense matrix: truncated header");
    if (std::memcmp(h, "BLZD", 4) != 0) throw io_error("dense matrix: magic mismatch (not a dense matrix file)");
    if (h[4] != 1) throw io_error("dense matrix: unsupported version " + std::to_string(h[4]));
    const std::size_t rows = detail::get_le(h + 5, 4), cols = detail::get_le(h + 9, 4);
    if (rows == 0 || cols == 0) throw io_error("dense matrix: zero dimension in header");
    dense_matrix m(rows, cols);
    std::vector<unsigned char> buf(m.values.size() * 8);
    in.read(reinterpret_cast<char*>(buf.data()), std::streamsize(buf.size()));
    if (std::size_t(in.gcount()) != buf.size()) throw io_error("dense matrix: truncated payload");
    for (std::size_t k = 0; k < m.values.size(); ++k) {
        const std::uint64_t u = detail::get_le(buf.data() + 8 * k, 8);
        std::memcpy(&m.values[k], &u, 8);
    }
    return m;
}

// One matrix row per line, comma-separated decimal cells ('.' separator, blanks
// around cells allowed); every row must have the same number of cells.
namespace detail {
// Cells of one CSV line, each trimmed of spaces / tabs ("a, b" -> {"a", "b"}).
inline std::vector<std::string_view> csv_cells(std::string_view line) {
    std::vector<std::string_view> cells;
    auto trim = [](std::string_view c) {
        const auto blank = [](char ch) { return ch == ' ' || ch == '\t'; };
        while (!c.empty() && blank(c.front())) c.remove_prefix(1);
        while (!c.empty() && blank(c.back())) c.remove_suffix(1);
        return c;
    };
    for (std::size_t start = 0;;) {
        const std::size_t comma = line.find(',', start);
        cells.push_back(trim(line.substr(start, comma == std::string_view::npos ? std::string_view::npos : comma - start)));
        if (comma == std::string_view::npos) return cells;
        start = comma + 1;
    }
}
}  // namespace detail

// H/io.hpp:155-195: one matrix row per line, comma-separated decimals ('.'), a
// trailing empty line and CR line ends tolerated; the reference's messages.
inline dense_matrix import_csv(std::istream& in) {
    std::vector<double> values;
    std::size_t rows = 0, cols = 0;
    for (std::string line; std::getline(in, line);) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty() && in.peek() == std::char_traits<char>::eof()) break;
        ++rows;
        const std::vector<std::string_view> cells = detail::csv_cells(line);
        for (std::size_t c = 0; c < cells.size(); ++c) {
            double v = 0.0;
            const char* first = cells[c].data();
            const char* last = first + cells[c].size();
            const auto [ptr, ec] = std::from_chars(first, last, v);
            if (cells[c].empty() || ec != std::errc{} || ptr != last)
                throw io_error("csv: non-numeric cell at row " + std::to_string(rows) + ", column " +
                               std::to_string(c + 1));
            values.push_back(v);
        }
        if (rows == 1) {
            cols = cells.size();
        } else if (cells.size() != cols) {
            throw io_error("csv: row " + std::to_string(rows) + " has " + std::to_string(cells.size()) +
                           " cells, expected " + std::to_string(cols));
        }
    }
    if (rows == 0) throw io_error("csv: empty input");
    dense_matrix m(rows, cols);
    m.values = std::move(values);
    return m;
}

// ---- uncompressed baselines (H/matrix.hpp:253-300), CPU ---------------------------
namespace ref {
// Dense CPU baselines (H/matrix.hpp:253-300), used by the reference's tests as
// oracles: each entry is formed by the reference's operation sequence (one
// rounding per operation, products summed over ascending k from +0.0).

inline void require_same_dims(const dense_matrix& a, const dense_matrix& b, const char* what) {
    if (a.rows == b.rows && a.cols == b.cols) return;
    throw std::invalid_argument(std::string(what) + ": dimension mismatch");
}

namespace detail {
template <class Op>
dense_matrix zip(const dense_matrix& a, const dense_matrix& b, const char* what, Op op) {
    require_same_dims(a, b, what);
    dense_matrix out(a.rows, a.cols);
    std::transform(a.values.begin(), a.values.end(), b.values.begin(), out.values.begin(), op);
    return out;
}
// sum over k of a_row[k] * b[k * stride], ascending from +0.0
inline double row_times_column(const double* a_row, const double* b_col, std::size_t n, std::size_t stride) {
    double acc = 0.0;
    for (std::size_t k = 0; k < n; ++k, b_col += stride) acc += a_row[k] * *b_col;
    return acc;
}
}  // namespace detail

inline dense_matrix add(const dense_matrix& a, const dense_matrix& b) {
    return detail::zip(a, b, "ref::add", [](double x, double y) { return x + y; });
}

inline dense_matrix sub(const dense_matrix& a, const dense_matrix& b) {
    return detail::zip(a, b, "ref::sub", [](double x, double y) { return x - y; });
}

inline dense_matrix scale(const dense_matrix& a, double c) {
    dense_matrix out(a.rows, a.cols);
    std::transform(a.values.begin(), a.values.end(), out.values.begin(), [c](double x) { return x * c; });
    return out;
}

inline double dot(const dense_matrix& a, const dense_matrix& b, std::size_t i, std::size_t j) {
    if (a.cols != b.rows) throw std::invalid_argument("ref::dot: inner dimension mismatch");
    if (i >= a.rows || j >= b.cols) throw std::out_of_range("ref::dot: index out of range");
    return detail::row_times_column(a.values.data() + i * a.cols, b.values.data() + j, a.cols, b.cols);
}

inline dense_matrix mul(const dense_matrix& a, const dense_matrix& b) {
    if (a.cols != b.rows) throw std::invalid_argument("ref::mul: inner dimension mismatch");
    dense_matrix out(a.rows, b.cols);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t j = 0; j < b.cols; ++j)
            out(i, j) = detail::row_times_column(a.values.data() + i * a.cols, b.values.data() + j, a.cols, b.cols);
    return out;
}

}  // namespace ref

}  // namespace blaz

#include "harness.hpp"  // H/bench.hpp: the evaluation harness, as in the reference's umbrella header

#endif  // BLAZ_DROPIN_BLAZ_HPP
