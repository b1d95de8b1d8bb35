// dropin_test.cpp -- the C++ drop-in (include/blaz/blaz.hpp, GPU-backed) against
// the C oracle port (oracle/blaz_oracle.c, CPU), bit for bit, through the
// reference's own C++ API.  Built by tests/cpp/Makefile; run by
// tests/test_cpp_dropin.py on a GPU box.
#include <gtest/gtest.h>

#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../oracle/blaz_oracle.h"
#include "blaz/blaz.hpp"

using namespace blaz;

namespace {

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

bool same(const compressed_block& a, const orc_block& b) {
    return same(a.first, b.first) && same(a.slope, b.slope) && a.scale_factor == b.scale_factor &&
           std::memcmp(a.coeffs.data(), b.coeffs, 28) == 0;
}

dense_matrix field(std::size_t rows, std::size_t cols, std::mt19937_64& rng, bool rough = false) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const double c0 = u(rng), cx = u(rng), cy = u(rng), cxy = u(rng);
    dense_matrix m(rows, cols);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) {
            const double x = double(j) / double(cols), y = double(i) / double(rows);
            m(i, j) = rough ? 50.0 * u(rng) : c0 + cx * x + cy * y + cxy * x * y + 0.05 * u(rng);
        }
    return m;
}

std::vector<orc_block> oracle_compress(const dense_matrix& m) {
    std::vector<orc_block> out(((m.rows + 7) / 8) * ((m.cols + 7) / 8));
    orc_compress_matrix(m.values.data(), m.rows, m.cols, out.data());
    return out;
}

std::vector<orc_block> as_orc(const compressed_matrix& cm) {
    std::vector<orc_block> out(cm.blocks.size());
    static_assert(sizeof(orc_block) == sizeof(compressed_block), "layout");
    std::memcpy(out.data(), cm.blocks.data(), out.size() * sizeof(orc_block));
    return out;
}

}  // namespace

TEST(DropIn, CompressDecompressMatchOracle) {
    std::mt19937_64 rng(101);
    for (auto [r, c] : {std::pair<int, int>{1, 1}, {9, 9}, {9, 17}, {40, 56}, {64, 64}, {100, 37}}) {
        for (bool rough : {false, true}) {
            const dense_matrix m = field(r, c, rng, rough);
            const compressed_matrix cm = compress_matrix(m, 4);
            const auto want = oracle_compress(m);
            ASSERT_EQ(cm.blocks.size(), want.size());
            for (std::size_t t = 0; t < want.size(); ++t) ASSERT_TRUE(same(cm.blocks[t], want[t])) << "block " << t;
            const dense_matrix back = decompress_matrix(cm);
            std::vector<double> ob(r * c);
            orc_decompress_matrix(want.data(), r, c, ob.data());
            ASSERT_EQ(back.rows, std::size_t(r));
            for (std::size_t k = 0; k < ob.size(); ++k) ASSERT_TRUE(same(back.values[k], ob[k])) << k;
        }
    }
}

TEST(DropIn, ElementwiseOpsMatchOracle) {
    std::mt19937_64 rng(102);
    const compressed_matrix a = compress_matrix(field(48, 40, rng));
    const compressed_matrix b = compress_matrix(field(48, 40, rng, true));
    auto oa = as_orc(a), ob = as_orc(b);
    std::vector<orc_block> o(oa.size());
    const compressed_matrix s = mat_add(a, b);
    orc_mat_add(oa.data(), ob.data(), oa.size(), o.data());
    for (std::size_t t = 0; t < o.size(); ++t) ASSERT_TRUE(same(s.blocks[t], o[t]));
    const compressed_matrix d = mat_sub(a, b);
    orc_mat_sub(oa.data(), ob.data(), oa.size(), o.data());
    for (std::size_t t = 0; t < o.size(); ++t) ASSERT_TRUE(same(d.blocks[t], o[t]));
    const compressed_matrix k = mat_scale(a, -2.25);
    orc_mat_scale(oa.data(), -2.25, oa.size(), o.data());
    for (std::size_t t = 0; t < o.size(); ++t) ASSERT_TRUE(same(k.blocks[t], o[t]));
    // s1 + s2 == 0 -> dense fallback
    const compressed_matrix z = mat_add(a, mat_scale(a, -1.0));
    const auto oz = as_orc(mat_scale(a, -1.0));
    orc_mat_add(oa.data(), oz.data(), oa.size(), o.data());
    for (std::size_t t = 0; t < o.size(); ++t) ASSERT_TRUE(same(z.blocks[t], o[t]));
}

TEST(DropIn, ProductsMatchOracle) {
    std::mt19937_64 rng(103);
    const compressed_matrix a = compress_matrix(field(20, 28, rng));
    const compressed_matrix b = compress_matrix(field(28, 12, rng));
    const auto oa = as_orc(a), ob = as_orc(b);
    const dense_matrix pd = mat_mul_dense(a, b);
    std::vector<double> want(20 * 12);
    orc_mat_mul_dense(oa.data(), 20, 28, ob.data(), 28, 12, want.data());
    for (std::size_t k = 0; k < want.size(); ++k) ASSERT_TRUE(same(pd.values[k], want[k]));
    const compressed_matrix pc = mat_mul(a, b);
    std::vector<orc_block> wc(pc.blocks.size());
    orc_mat_mul(oa.data(), 20, 28, ob.data(), 28, 12, wc.data());
    for (std::size_t t = 0; t < wc.size(); ++t) ASSERT_TRUE(same(pc.blocks[t], wc[t]));
    for (std::size_t i = 0; i < 20; i += 3)
        for (std::size_t j = 0; j < 12; j += 5) {
            double w = 0.0;
            orc_mat_dot(oa.data(), 20, 28, ob.data(), 28, 12, i, j, &w);
            ASSERT_TRUE(same(mat_dot(a, b, i, j), w)) << i << "," << j;
        }
}

TEST(DropIn, BlockLevelMatchesOracle) {
    std::mt19937_64 rng(104);
    std::uniform_real_distribution<double> u(-3.0, 3.0);
    for (int rep = 0; rep < 20; ++rep) {
        block8 m1, m2;
        for (int k = 0; k < 64; ++k) {
            m1.a[k] = (k / 8) * u(rng) + (k % 8) + 0.01 * u(rng);
            m2.a[k] = u(rng);
        }
        const compressed_block b1 = compress_block(m1), b2 = compress_block(m2);
        orc_block o1, o2, o;
        orc_compress_block(m1.a.data(), &o1);
        orc_compress_block(m2.a.data(), &o2);
        ASSERT_TRUE(same(b1, o1));
        ASSERT_TRUE(same(b2, o2));
        double want[64];
        orc_decompress_block(&o1, want);
        const block8 d1 = decompress_block(b1);
        for (int k = 0; k < 64; ++k) ASSERT_TRUE(same(d1.a[k], want[k]));
        orc_dequantize_prediction(&o1, want);
        const block8 p1 = dequantize_prediction(b1);
        for (int k = 0; k < 64; ++k) ASSERT_TRUE(same(p1.a[k], want[k]));
        orc_add(&o1, &o2, &o);
        ASSERT_TRUE(same(add(b1, b2), o));
        orc_sub(&o1, &o2, &o);
        ASSERT_TRUE(same(sub(b1, b2), o));
        orc_scale(&o1, 0.75, &o);
        ASSERT_TRUE(same(scale(b1, 0.75), o));
        orc_block_mul(&o1, &o2, want);
        const block8 pm = block_mul(b1, b2);
        for (int k = 0; k < 64; ++k) ASSERT_TRUE(same(pm.a[k], want[k]));
        for (int i = 0; i < 8; i += 3)
            for (int j = 0; j < 8; j += 2) ASSERT_TRUE(same(dot(b1, b2, i, j), orc_dot(&o1, &o2, i, j)));
        orc_reconstruct_rows(&o1, 3, want);
        const partial_reconstruction rr = reconstruct_rows(b1, 3);
        for (int k = 0; k < 64; ++k) ASSERT_TRUE(same(rr.values.a[k], want[k]));
        orc_reconstruct_cols(&o1, 5, want);
        const partial_reconstruction rc = reconstruct_cols(b1, 5);
        for (int k = 0; k < 64; ++k) ASSERT_TRUE(same(rc.values.a[k], want[k]));
    }
}

TEST(DropIn, ExceptionsMatchReference) {
    std::mt19937_64 rng(105);
    EXPECT_THROW(compress_matrix(dense_matrix{}), std::invalid_argument);
    dense_matrix bad = field(16, 16, rng);
    bad(3, 3) = std::nan("");
    EXPECT_THROW(compress_matrix(bad), std::invalid_argument);
    const compressed_matrix a = compress_matrix(field(16, 16, rng));
    const compressed_matrix b = compress_matrix(field(16, 24, rng));
    try {
        mat_add(a, b);
        EXPECT_TRUE(false) << "no throw";
    } catch (const std::invalid_argument& e) {
        EXPECT_EQ(std::string(e.what()), std::string("mat_add: dimension mismatch (16x16 vs 16x24)"));
    }
    EXPECT_THROW(mat_sub(a, b), std::invalid_argument);
    EXPECT_THROW(mat_scale(a, INFINITY), std::invalid_argument);
    const compressed_matrix c = compress_matrix(field(24, 16, rng));
    EXPECT_THROW(mat_dot(a, c, 0, 0), std::invalid_argument);
    EXPECT_THROW(mat_dot(a, a, 16, 0), std::out_of_range);
    EXPECT_THROW(mat_mul(a, c), std::invalid_argument);
    EXPECT_THROW(reconstruct_rows(a.blocks[0], 8), std::out_of_range);
    EXPECT_THROW(dot(a.blocks[0], a.blocks[0], 0, 8), std::out_of_range);
}

// The reference's functions are pure and re-entrant: concurrent calls from
// several threads (each on its own per-thread context) give the oracle's
// results, including the error messages of the failing calls.
TEST(DropIn, ConcurrentCallsFromThreads) {
    constexpr int kThreads = 6;
    std::vector<std::thread> pool;
    std::vector<int> bad(kThreads, 0);
    for (int w = 0; w < kThreads; ++w) {
        pool.emplace_back([w, &bad] {
            std::mt19937_64 rng(500 + w);
            for (int it = 0; it < 4; ++it) {
                const dense_matrix ma = field(40 + 8 * w, 56, rng, (w + it) & 1);
                const dense_matrix mb = field(40 + 8 * w, 56, rng);
                const compressed_matrix a = compress_matrix(ma), b = compress_matrix(mb);
                const compressed_matrix s = mat_sub(a, b);
                std::vector<orc_block> oa = oracle_compress(ma), ob = oracle_compress(mb), os(oa.size());
                orc_mat_sub(oa.data(), ob.data(), oa.size(), os.data());
                for (std::size_t t = 0; t < os.size(); ++t) bad[w] += !same(s.blocks[t], os[t]);
                try {
                    mat_add(a, compress_matrix(field(8, 8, rng)));
                    ++bad[w];
                } catch (const std::invalid_argument& e) {
                    const std::string want = "mat_add: dimension mismatch (" + std::to_string(ma.rows) + "x56 vs 8x8)";
                    bad[w] += std::string(e.what()) != want;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    for (int w = 0; w < kThreads; ++w) EXPECT_EQ(bad[w], 0) << "thread " << w;
}
