// blaz -- command-line front end over the GPU library.
//
// Same subcommands, arguments, file formats and exit codes as the reference's
// tool (proj/tools/blaz.cpp:112-270): 0 success, 1 usage error, 2 I/O or format
// error, 3 dimension/argument error.  Every matrix operation goes through the
// drop-in header include/blaz/blaz.hpp, i.e. runs on the B200; the argument
// parser is a small hand-written one (the reference uses CLI11, absent here).
// The evaluation-harness subcommands (accuracy, bench; H/bench.hpp) are not
// part of this build and report a usage error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "blaz/blaz.hpp"

namespace fs = std::filesystem;

namespace {

struct usage_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct argument_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

const char* kUsage =
    "usage: blaz [--force] [--threads N] <command> ...\n"
    "  gen <f1..f6> <n> -o out.blzd        sample a test function on [-2,2]^2\n"
    "  compress <in.blzd|in.csv> -o out.blzc\n"
    "  decompress <in.blzc> -o out.blzd\n"
    "  info <in.blzc>\n"
    "  add <a.blzc> <b.blzc> -o out.blzc\n"
    "  sub <a.blzc> <b.blzc> -o out.blzc\n"
    "  scale <in.blzc> <c> -o out.blzc\n"
    "  dot <a.blzc> <b.blzc> <i> <j>\n"
    "  matmul <a.blzc> <b.blzc> -o out.blzc\n";

// Parsed command line: global flags, the subcommand, its positionals and -o.
struct Args {
    bool force = false;
    unsigned threads = 1;
    std::string cmd, output;
    std::vector<std::string> pos;
};

Args parse(int argc, char** argv) {
    Args a;
    for (int k = 1; k < argc; ++k) {
        const std::string t = argv[k];
        auto value = [&](const char* what) -> std::string {
            if (k + 1 >= argc) throw usage_error(std::string(what) + " requires a value");
            return argv[++k];
        };
        if (t == "--force") {
            a.force = true;
        } else if (t == "--threads") {
            const std::string v = value("--threads");
            char* end = nullptr;
            const unsigned long n = std::strtoul(v.c_str(), &end, 10);
            if (v.empty() || *end) throw usage_error("--threads: not a number: " + v);
            a.threads = unsigned(n);
        } else if (t == "-o" || t == "--output") {
            a.output = value("--output");
        } else if (t.rfind("--output=", 0) == 0) {
            a.output = t.substr(9);
        } else if (t.size() > 1 && t[0] == '-' && !(t.size() > 1 && (std::isdigit((unsigned char)t[1]) || t[1] == '.'))) {
            throw usage_error("unknown option " + t);
        } else if (a.cmd.empty()) {
            a.cmd = t;
        } else {
            a.pos.push_back(t);
        }
    }
    if (a.cmd.empty()) throw usage_error("a subcommand is required");
    return a;
}

void need(const Args& a, std::size_t npos, bool output) {
    if (a.pos.size() != npos)
        throw usage_error(a.cmd + ": expected " + std::to_string(npos) + " positional argument(s), got " +
                          std::to_string(a.pos.size()));
    if (output && a.output.empty()) throw usage_error(a.cmd + ": --output is required");
    if (!output && !a.output.empty()) throw usage_error(a.cmd + ": takes no --output");
}

std::ifstream open_input(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw blaz::io_error("cannot open input file: " + path);
    return in;
}

// temp file + rename: a failed write never leaves a partial output behind
template <class Write>
void write_atomically(const std::string& path, bool force, Write&& write) {
    if (!force && fs::exists(path)) throw blaz::io_error("output exists (use --force to overwrite): " + path);
    fs::path tmp = path;
    tmp += ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw blaz::io_error("cannot open output file: " + tmp.string());
        write(out);
        out.flush();
        if (!out) {
            std::error_code ec;
            fs::remove(tmp, ec);
            throw blaz::io_error("write failed: " + tmp.string());
        }
    }
    std::error_code ec;
    fs::rename(tmp, path, ec);
    if (ec) {
        fs::remove(tmp, ec);
        throw blaz::io_error("cannot rename temporary file onto " + path);
    }
}

blaz::dense_matrix load_dense(const std::string& path) {
    auto in = open_input(path);
    if (path.size() >= 4 && path.compare(path.size() - 4, 4, ".csv") == 0) return blaz::import_csv(in);
    return blaz::read_dense(in);
}

blaz::compressed_matrix load_compressed(const std::string& path) {
    auto in = open_input(path);
    return blaz::read_compressed(in);
}

// The paper's six test surfaces (section 4), sampled on [-2,2]^2 with
// nodes -2 + 4j/(n-1): M(i,j) = f(x_j, y_i).
// (each expression in the reference's evaluation order, H/bench.hpp:26-36)
double surface(int id, double x, double y) {
    switch (id) {
        case 1: return x * y;
        case 2: return x * y / (1.0 + x * x + y * y);
        case 3: return x * x - y;
        case 4: return (x * x) * (y * y);
        case 5: return std::cos(std::sqrt(x * x + y * y));
        default: return std::cos(x * x + y * y) * std::exp(-0.1 * (x * x + y * y));
    }
}

blaz::dense_matrix gen(const std::string& fn, const std::string& ns) {
    if (fn.size() != 2 || fn[0] != 'f' || fn[1] < '1' || fn[1] > '6')
        throw argument_error("unknown test function '" + fn + "' (expected f1..f6)");
    char* end = nullptr;
    const unsigned long long n = std::strtoull(ns.c_str(), &end, 10);
    if (ns.empty() || *end) throw usage_error("gen: n is not a number: " + ns);
    if (n < 2) throw argument_error("n must be at least 2");
    std::vector<double> nodes(n);
    for (std::size_t j = 0; j < n; ++j) nodes[j] = -2.0 + 4.0 * double(j) / double(n - 1);
    blaz::dense_matrix m(n, n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) m(i, j) = surface(fn[1] - '0', nodes[j], nodes[i]);
    return m;
}

double parse_double(const std::string& s, const char* what) {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (s.empty() || *end) throw usage_error(std::string(what) + ": not a number: " + s);
    return v;
}

long long parse_index(const std::string& s, const char* what) {
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (s.empty() || *end) throw usage_error(std::string(what) + ": not an integer: " + s);
    return v;
}

int run(const Args& a) {
    const unsigned th = a.threads;
    auto save_c = [&](const blaz::compressed_matrix& r) {
        write_atomically(a.output, a.force, [&](std::ostream& o) { blaz::write_compressed(r, o); });
    };
    auto save_d = [&](const blaz::dense_matrix& r) {
        write_atomically(a.output, a.force, [&](std::ostream& o) { blaz::write_dense(r, o); });
    };
    if (a.cmd == "gen") {
        need(a, 2, true);
        save_d(gen(a.pos[0], a.pos[1]));
    } else if (a.cmd == "compress") {
        need(a, 1, true);
        save_c(blaz::compress_matrix(load_dense(a.pos[0]), th));
    } else if (a.cmd == "decompress") {
        need(a, 1, true);
        save_d(blaz::decompress_matrix(load_compressed(a.pos[0]), th));
    } else if (a.cmd == "info") {
        need(a, 1, false);
        const blaz::compressed_matrix cm = load_compressed(a.pos[0]);
        std::printf("dimensions:       %zu x %zu\n", cm.rows, cm.cols);
        std::printf("block grid:       %zu x %zu (%zu blocks)\n", cm.block_rows, cm.block_cols, cm.blocks.size());
        std::printf("block payload:    %d bytes\n", blaz::block_payload_bytes);
        std::printf("compression rate: %.4f\n", blaz::compression_rate);
    } else if (a.cmd == "add" || a.cmd == "sub") {
        need(a, 2, true);
        const blaz::compressed_matrix x = load_compressed(a.pos[0]), y = load_compressed(a.pos[1]);
        save_c(a.cmd == "add" ? blaz::mat_add(x, y, th) : blaz::mat_sub(x, y, th));
    } else if (a.cmd == "scale") {
        need(a, 2, true);
        const double c = parse_double(a.pos[1], "scale");
        save_c(blaz::mat_scale(load_compressed(a.pos[0]), c, th));
    } else if (a.cmd == "dot") {
        need(a, 4, false);
        const long long i = parse_index(a.pos[2], "dot"), j = parse_index(a.pos[3], "dot");
        if (i < 0 || j < 0) throw argument_error("indices must be non-negative");
        const blaz::compressed_matrix x = load_compressed(a.pos[0]), y = load_compressed(a.pos[1]);
        std::printf("%.17g\n", blaz::mat_dot(x, y, std::size_t(i), std::size_t(j)));
    } else if (a.cmd == "matmul") {
        need(a, 2, true);
        const blaz::compressed_matrix x = load_compressed(a.pos[0]), y = load_compressed(a.pos[1]);
        save_c(blaz::mat_mul(x, y, th));
    } else if (a.cmd == "accuracy" || a.cmd == "bench") {
        throw usage_error(a.cmd + ": the evaluation harness (H/bench.hpp) is not part of this build");
    } else {
        throw usage_error("unknown subcommand '" + a.cmd + "'");
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    for (int k = 1; k < argc; ++k)
        if (std::string(argv[k]) == "-h" || std::string(argv[k]) == "--help") {
            std::fputs(kUsage, stdout);
            return 0;
        }
    Args a;
    try {
        a = parse(argc, argv);
    } catch (const usage_error& e) {
        std::fprintf(stderr, "error: %s\n%s", e.what(), kUsage);
        return 1;
    }
    try {
        return run(a);
    } catch (const usage_error& e) {
        std::fprintf(stderr, "error: %s\n%s", e.what(), kUsage);
        return 1;
    } catch (const argument_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const blaz::io_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const std::out_of_range& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
