// Minimal GoogleTest-compatible shim (TEST INFRASTRUCTURE). GoogleTest is absent
// from this image (reference CMakeLists.txt:14); this covers the macros the
// reference test files use so they compile unchanged and validate the Eigen shim.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}
inline int register_test(const char* suite, const char* name, void (*fn)()) {
  registry().push_back({suite, name, fn});
  return 0;
}
inline std::string TempDir() {
  const char* t = std::getenv("TEST_TMPDIR");
  std::string d = t ? t : "/tmp";
  if (d.empty() || d.back() != '/') d += '/';
  return d;
}

// Streams a failure message on destruction (so `<< msg` can follow a macro).
class Failure {
 public:
  Failure(const char* file, int line, std::string what) : file_(file), line_(line), what_(std::move(what)) {}
  ~Failure() {
    current_failed() = true;
    std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file_, line_, what_.c_str(),
                 msg_.str().empty() ? "" : "\n  ", msg_.str().c_str());
  }
  template <typename T>
  Failure& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream msg_;
};

struct Sink {
  template <typename T>
  Sink& operator<<(const T&) { return *this; }
};

// ASSERT_* return from the test body: `return AssertHelper() = Failure(...) << msg`.
struct AssertHelper {
  void operator=(const Failure&) const {}
};

template <typename T>
std::string repr(const T& v) {
  std::ostringstream os;
  if constexpr (requires { os << v; }) {
    os.precision(17);
    os << v;
  } else {
    os << "<value>";
  }
  return os.str();
}

inline bool double_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, 8);
    const std::uint64_t sign = 1ull << 63;
    return (u & sign) ? ~u + 1 : u | sign;
  };
  const std::uint64_t ua = biased(a), ub = biased(b);
  return (ua > ub ? ua - ub : ub - ua) <= 4;
}

}  // namespace testing

#define GTEST_SHIM_CAT2(a, b) a##b
#define GTEST_SHIM_CAT(a, b) GTEST_SHIM_CAT2(a, b)

#define TEST(suite, name)                                                                  \
  static void GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name))();                            \
  static const int GTEST_SHIM_CAT(reg_, GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name))) =  \
      ::testing::register_test(#suite, #name, &GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name))); \
  static void GTEST_SHIM_CAT(suite, GTEST_SHIM_CAT(_, name))()

#define GTEST_SHIM_CHECK(cond, text, fatal)                                          \
  if (cond) {                                                                        \
  } else                                                                             \
    fatal ::testing::Failure(__FILE__, __LINE__, text)

#define GTEST_SHIM_NONFATAL
#define GTEST_SHIM_FATAL return ::testing::AssertHelper() =

#define GTEST_SHIM_BIN(a, b, op, fatal)                                                    \
  if (const auto& gs_a = (a); true)                                                        \
    if (const auto& gs_b = (b); (gs_a op gs_b)) {                                          \
    } else                                                                                 \
      fatal ::testing::Failure(__FILE__, __LINE__,                                         \
                               std::string("Expected: " #a " " #op " " #b "\n  actual: ") + \
                                   ::testing::repr(gs_a) + " vs " + ::testing::repr(gs_b))

#define EXPECT_TRUE(c) GTEST_SHIM_CHECK(bool(c), "Expected true: " #c, GTEST_SHIM_NONFATAL)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK(!bool(c), "Expected false: " #c, GTEST_SHIM_NONFATAL)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK(bool(c), "Expected true: " #c, GTEST_SHIM_FATAL)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK(!bool(c), "Expected false: " #c, GTEST_SHIM_FATAL)

#define EXPECT_EQ(a, b) GTEST_SHIM_BIN(a, b, ==, GTEST_SHIM_NONFATAL)
#define EXPECT_NE(a, b) GTEST_SHIM_BIN(a, b, !=, GTEST_SHIM_NONFATAL)
#define EXPECT_LT(a, b) GTEST_SHIM_BIN(a, b, <, GTEST_SHIM_NONFATAL)
#define EXPECT_LE(a, b) GTEST_SHIM_BIN(a, b, <=, GTEST_SHIM_NONFATAL)
#define EXPECT_GT(a, b) GTEST_SHIM_BIN(a, b, >, GTEST_SHIM_NONFATAL)
#define EXPECT_GE(a, b) GTEST_SHIM_BIN(a, b, >=, GTEST_SHIM_NONFATAL)
#define ASSERT_EQ(a, b) GTEST_SHIM_BIN(a, b, ==, GTEST_SHIM_FATAL)
#define ASSERT_NE(a, b) GTEST_SHIM_BIN(a, b, !=, GTEST_SHIM_FATAL)
#define ASSERT_LT(a, b) GTEST_SHIM_BIN(a, b, <, GTEST_SHIM_FATAL)
#define ASSERT_LE(a, b) GTEST_SHIM_BIN(a, b, <=, GTEST_SHIM_FATAL)
#define ASSERT_GT(a, b) GTEST_SHIM_BIN(a, b, >, GTEST_SHIM_FATAL)
#define ASSERT_GE(a, b) GTEST_SHIM_BIN(a, b, >=, GTEST_SHIM_FATAL)

#define EXPECT_NEAR(a, b, tol)                                                             \
  GTEST_SHIM_CHECK(std::abs(double(a) - double(b)) <= double(tol),                         \
                   "Expected near: " #a " ~ " #b " (tol " #tol ")\n  actual: " +           \
                       ::testing::repr(double(a)) + " vs " + ::testing::repr(double(b)),    \
                   GTEST_SHIM_NONFATAL)
#define ASSERT_NEAR(a, b, tol)                                                             \
  GTEST_SHIM_CHECK(std::abs(double(a) - double(b)) <= double(tol),                         \
                   "Expected near: " #a " ~ " #b " (tol " #tol ")", GTEST_SHIM_FATAL)
#define EXPECT_DOUBLE_EQ(a, b)                                                             \
  GTEST_SHIM_CHECK(::testing::double_eq(double(a), double(b)),                             \
                   "Expected double eq: " #a " == " #b "\n  actual: " +                    \
                       ::testing::repr(double(a)) + " vs " + ::testing::repr(double(b)),    \
                   GTEST_SHIM_NONFATAL)

#define EXPECT_THROW(stmt, exc)                                                            \
  if (bool gs_thrown = false; true)                                                        \
    if ([&] { try { stmt; } catch (const exc&) { gs_thrown = true; } catch (...) {}        \
              return gs_thrown; }()) {                                                     \
    } else                                                                                 \
      ::testing::Failure(__FILE__, __LINE__, "Expected " #stmt " to throw " #exc)

#define FAIL() return ::testing::AssertHelper() = ::testing::Failure(__FILE__, __LINE__, "Failed")
#define SUCCEED() ::testing::Sink()

#ifndef GTEST_SHIM_NO_MAIN
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed = 0, ran = 0;
  for (const auto& t : ::testing::registry()) {
    const std::string full = std::string(t.suite) + "." + t.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    ::testing::current_failed() = false;
    try {
      t.fn();
    } catch (const std::exception& e) {
      ::testing::current_failed() = true;
      std::fprintf(stderr, "%s: uncaught exception: %s\n", full.c_str(), e.what());
    }
    ++ran;
    if (::testing::current_failed()) {
      ++failed;
      std::printf("[  FAILED  ] %s\n", full.c_str());
    } else {
      std::printf("[       OK ] %s\n", full.c_str());
    }
  }
  std::printf("[==========] %d tests ran, %d failed\n", ran, failed);
  return failed ? 1 : 0;
}
#endif
