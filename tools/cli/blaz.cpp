// blaz -- command-line front end over the GPU library.
//
// Same subcommands, arguments, file formats and exit codes as the reference's
// tool (proj/tools/blaz.cpp:112-270): 0 success, 1 usage error, 2 I/O or format
// error, 3 dimension/argument error.  Every matrix operation goes through the
// drop-in header include/blaz/blaz.hpp, i.e. runs on the B200; the argument
// parser is a small hand-written one (the reference uses CLI11, absent here).
// accuracy / bench run the evaluation harness of the drop-in (blaz/harness.hpp).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
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
    "  matmul <a.blzc> <b.blzc> -o out.blzc\n"
    "  accuracy [-n N] -o out.csv                  the accuracy table (default n 512)\n"
    "  bench [--sizes a,b] [--ops x,y] [--repeats R] -o out.csv\n";

// Parsed command line: global flags, the subcommand, its positionals and -o.
struct Args {
    bool force = false;
    unsigned threads = 1;
    std::string cmd, output;
    std::vector<std::string> pos;
    std::string size = "512", sizes = "80,400,1000,2000", ops = "add,scale,dot,matmul,compress,decompress",
                repeats = "5";
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
        } else if (t == "-n" || t == "--size") {
            a.size = value("--size");
        } else if (t == "--sizes") {
            a.sizes = value("--sizes");
        } else if (t == "--ops") {
            a.ops = value("--ops");
        } else if (t == "--repeats") {
            a.repeats = value("--repeats");
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

bool has_suffix(const std::string& s, const char* suf) {
    const std::size_t n = std::strlen(suf);
    return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

// Parses the file at `path` with `parse(std::istream&)`.
template <class Parse>
auto parse_file(const std::string& path, Parse&& parse) {
    std::ifstream stream(path, std::ios::binary);
    if (!stream.is_open()) throw blaz::io_error("cannot open input file: " + path);
    return parse(stream);
}

blaz::dense_matrix load_dense(const std::string& path) {
    return parse_file(path, [&](std::istream& is) {
        return has_suffix(path, ".csv") ? blaz::import_csv(is) : blaz::read_dense(is);
    });
}

blaz::compressed_matrix load_compressed(const std::string& path) {
    return parse_file(path, [](std::istream& is) { return blaz::read_compressed(is); });
}

// An output written to "<path>.tmp" and renamed onto <path> by commit(): a
// failed or abandoned write removes the temporary and never leaves a partial
// output behind.
class StagedOutput {
public:
    StagedOutput(std::string path, bool force) : final_(std::move(path)), tmp_(final_ + ".tmp") {
        if (!force && fs::exists(final_))
            throw blaz::io_error("output exists (use --force to overwrite): " + final_);
        file_.open(tmp_, std::ios::binary | std::ios::trunc);
        if (!file_.is_open()) throw blaz::io_error("cannot open output file: " + tmp_.string());
    }
    ~StagedOutput() {
        if (!committed_) {
            file_.close();
            std::error_code ignore;
            fs::remove(tmp_, ignore);
        }
    }
    std::ostream& stream() { return file_; }
    void commit() {
        file_.flush();
        const bool ok = static_cast<bool>(file_);
        file_.close();
        if (!ok) throw blaz::io_error("write failed: " + tmp_.string());
        std::error_code ec;
        fs::rename(tmp_, final_, ec);
        if (ec) throw blaz::io_error("cannot rename temporary file onto " + final_);
        committed_ = true;
    }

private:
    std::string final_;
    fs::path tmp_;
    std::ofstream file_;
    bool committed_ = false;
};

template <class Write>
void save(const std::string& path, bool force, Write&& write) {
    StagedOutput out(path, force);
    write(out.stream());
    out.commit();
}

blaz::dense_matrix gen(const std::string& fn, const std::string& ns) {
    const blaz::test_function* f = blaz::find_test_function(fn);
    if (!f) throw argument_error("unknown test function '" + fn + "' (expected f1..f6)");
    char* end = nullptr;
    const unsigned long long n = std::strtoull(ns.c_str(), &end, 10);
    if (ns.empty() || *end) throw usage_error("gen: n is not a number: " + ns);
    if (n < 2) throw argument_error("n must be at least 2");
    return blaz::gen_matrix(*f, n);
}

std::vector<std::size_t> parse_sizes(const std::string& csv) {
    std::vector<std::size_t> out;
    std::size_t pos = 0;
    while (pos <= csv.size()) {
        const std::size_t comma = csv.find(',', pos);
        const std::string tok = csv.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        char* end = nullptr;
        const unsigned long v = std::strtoul(tok.c_str(), &end, 10);
        if (tok.empty() || *end || v < 2) throw argument_error("bad size '" + tok + "'");
        out.push_back(v);
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return out;
}

std::vector<blaz::bench_op> parse_ops(const std::string& csv) {
    std::vector<blaz::bench_op> out;
    std::size_t pos = 0;
    while (pos <= csv.size()) {
        const std::size_t comma = csv.find(',', pos);
        const std::string tok = csv.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        bool found = false;
        for (const blaz::bench_op op : blaz::all_bench_ops())
            if (tok == blaz::name_of(op)) {
                out.push_back(op);
                found = true;
            }
        if (!found) throw argument_error("unknown op '" + tok + "' (expected add,scale,dot,matmul,compress,decompress)");
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return out;
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
        save(a.output, a.force, [&](std::ostream& o) { blaz::write_compressed(r, o); });
    };
    auto save_d = [&](const blaz::dense_matrix& r) {
        save(a.output, a.force, [&](std::ostream& o) { blaz::write_dense(r, o); });
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
        char rate[32];
        std::snprintf(rate, sizeof rate, "%.4f", blaz::compression_rate);
        const std::pair<const char*, std::string> fields[] = {
            {"dimensions", std::to_string(cm.rows) + " x " + std::to_string(cm.cols)},
            {"block grid", std::to_string(cm.block_rows) + " x " + std::to_string(cm.block_cols) + " (" +
                               std::to_string(cm.blocks.size()) + " blocks)"},
            {"block payload", std::to_string(blaz::block_payload_bytes) + " bytes"},
            {"compression rate", rate},
        };
        for (const auto& [name, value] : fields) std::printf("%-18s%s\n", (std::string(name) + ":").c_str(), value.c_str());
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
    } else if (a.cmd == "accuracy") {
        need(a, 0, true);
        char* end = nullptr;
        const unsigned long long n = std::strtoull(a.size.c_str(), &end, 10);
        if (a.size.empty() || *end) throw usage_error("--size: not a number: " + a.size);
        if (n < 2) throw argument_error("size must be at least 2");
        const auto rows = blaz::accuracy_suite(n, th);
        save(a.output, a.force, [&](std::ostream& o) { blaz::write_accuracy_csv(rows, o); });
    } else if (a.cmd == "bench") {
        need(a, 0, true);
        const auto sizes = parse_sizes(a.sizes);
        const auto ops = parse_ops(a.ops);
        char* end = nullptr;
        const long r = std::strtol(a.repeats.c_str(), &end, 10);
        if (a.repeats.empty() || *end) throw usage_error("--repeats: not a number: " + a.repeats);
        if (r < 5) throw argument_error("repeats must be at least 5");
        const auto rows = blaz::bench_suite(sizes, ops, int(r), th);
        save(a.output, a.force, [&](std::ostream& o) { blaz::write_bench_csv(rows, o); });
    } else {
        throw usage_error("unknown subcommand '" + a.cmd + "'");
    }
    return 0;
}

}  // namespace

// Exit status of a failed run: 1 usage, 2 I/O / format / runtime, 3 bad arguments
// or dimensions (the reference CLI's contract, proj/tools/blaz.cpp).
int exit_status(const std::exception& e) {
    if (dynamic_cast<const usage_error*>(&e)) return 1;
    if (dynamic_cast<const blaz::io_error*>(&e)) return 2;
    if (dynamic_cast<const argument_error*>(&e) || dynamic_cast<const std::invalid_argument*>(&e) ||
        dynamic_cast<const std::out_of_range*>(&e))
        return 3;
    return 2;
}

int main(int argc, char** argv) {
    for (int k = 1; k < argc; ++k)
        if (std::string(argv[k]) == "-h" || std::string(argv[k]) == "--help") {
            std::fputs(kUsage, stdout);
            return 0;
        }
    try {
        return run(parse(argc, argv));
    } catch (const std::exception& e) {
        const int status = exit_status(e);
        std::fprintf(stderr, "error: %s\n%s", e.what(), status == 1 ? kUsage : "");
        return status;
    }
}
