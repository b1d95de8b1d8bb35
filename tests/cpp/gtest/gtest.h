// Minimal GoogleTest-compatible test runner (TEST, EXPECT_*/ASSERT_*), written
// for this repository so that GTest-style suites -- ours and the reference's
// own proj/tests/*.cpp compiled against the drop-in header -- run without the
// (absent) GTest package.  Failures print file:line and any streamed message.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mini_gtest {

struct Case {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, std::move(f)}); }
};

struct AssertFail {};

// Collects the streamed message; reports on destruction; throws for ASSERT_*.
class Reporter {
 public:
  Reporter(const char* file, int line, std::string what, bool fatal) : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  template <class T>
  Reporter& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }
  ~Reporter() noexcept(false) {
    std::fprintf(stderr, "%s:%d: Failure: %s %s\n", file_, line_, what_.c_str(), msg_.str().c_str());
    current_failed() = true;
    if (fatal_ && !std::uncaught_exceptions()) throw AssertFail{};
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

struct Sink {
  template <class T>
  Sink& operator<<(const T&) {
    return *this;
  }
};

inline int run_all() {
  int failed = 0;
  for (auto& c : registry()) {
    current_failed() = false;
    try {
      c.fn();
    } catch (const AssertFail&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s.%s: uncaught exception: %s\n", c.suite, c.name, e.what());
      current_failed() = true;
    }
    std::printf("[%s] %s.%s\n", current_failed() ? "  FAILED  " : "       OK ", c.suite, c.name);
    failed += current_failed();
  }
  std::printf("[==========] %zu tests, %d failed\n", registry().size(), failed);
  return failed ? 1 : 0;
}

}  // namespace mini_gtest

#define TEST(S, N)                                                                          \
  static void S##_##N##_body();                                                              \
  static mini_gtest::Registrar S##_##N##_reg(#S, #N, S##_##N##_body);                        \
  static void S##_##N##_body()

#define MG_CHECK(cond, what, fatal) \
  if (cond) {                       \
  } else                            \
    mini_gtest::Reporter(__FILE__, __LINE__, what, fatal)

#define EXPECT_TRUE(c) MG_CHECK((c), "EXPECT_TRUE(" #c ")", false)
#define FAIL() MG_CHECK(false, "FAIL()", true)
#define ASSERT_TRUE(c) MG_CHECK((c), "ASSERT_TRUE(" #c ")", true)
#define EXPECT_EQ(a, b) MG_CHECK((a) == (b), "EXPECT_EQ(" #a ", " #b ")", false)
#define ASSERT_EQ(a, b) MG_CHECK((a) == (b), "ASSERT_EQ(" #a ", " #b ")", true)
#define EXPECT_NE(a, b) MG_CHECK((a) != (b), "EXPECT_NE(" #a ", " #b ")", false)
#define ASSERT_NE(a, b) MG_CHECK((a) != (b), "ASSERT_NE(" #a ", " #b ")", true)
#define EXPECT_LE(a, b) MG_CHECK((a) <= (b), "EXPECT_LE(" #a ", " #b ")", false)
#define ASSERT_LE(a, b) MG_CHECK((a) <= (b), "ASSERT_LE(" #a ", " #b ")", true)
#define EXPECT_GE(a, b) MG_CHECK((a) >= (b), "EXPECT_GE(" #a ", " #b ")", false)
#define ASSERT_GE(a, b) MG_CHECK((a) >= (b), "ASSERT_GE(" #a ", " #b ")", true)
#define EXPECT_GT(a, b) MG_CHECK((a) > (b), "EXPECT_GT(" #a ", " #b ")", false)
#define ASSERT_GT(a, b) MG_CHECK((a) > (b), "ASSERT_GT(" #a ", " #b ")", true)
#define EXPECT_NEAR(a, b, t) MG_CHECK(std::fabs(double(a) - double(b)) <= double(t), "EXPECT_NEAR(" #a ", " #b ")", false)
#define ASSERT_NEAR(a, b, t) MG_CHECK(std::fabs(double(a) - double(b)) <= double(t), "ASSERT_NEAR(" #a ", " #b ")", true)
#define EXPECT_THROW(stmt, ex)                                          \
  do {                                                                  \
    bool mg_caught = false;                                             \
    try {                                                               \
      stmt;                                                             \
    } catch (const ex&) {                                               \
      mg_caught = true;                                                 \
    } catch (...) {                                                     \
    }                                                                   \
    if (!mg_caught) mini_gtest::Reporter(__FILE__, __LINE__, "EXPECT_THROW(" #stmt ", " #ex ")", false); \
  } while (0)

int main() { return mini_gtest::run_all(); }
