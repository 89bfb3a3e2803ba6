// Minimal GoogleTest-compatible shim (GTest is not installed in this image).
// TEST INFRASTRUCTURE: lets the reference's own unit-test files compile
// unchanged, against the reference library (oracle/_ref) and against the
// drop-in B200 library.  Supports the macros those files use: TEST,
// EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,DOUBLE_EQ,THROW,NO_THROW}
// with << message streaming, and ::testing::Test::HasFailure().
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct Registry {
  struct Case {
    std::string name;
    std::function<void()> fn;
  };
  static Registry& get() {
    static Registry r;
    return r;
  }
  std::vector<Case> cases;
  bool current_failed = false;
};

class Test {
 public:
  static bool HasFailure() { return Registry::get().current_failed; }
};

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<void()> fn) {
    Registry::get().cases.push_back({std::string(suite) + "." + name, std::move(fn)});
  }
};

// Streams the user message, reports on destruction.
class Reporter {
 public:
  Reporter(const char* file, int line, std::string what) : file_(file), line_(line), what_(what) {}
  ~Reporter() {
    Registry::get().current_failed = true;
    std::cerr << file_ << ":" << line_ << ": Failure\n  " << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cerr << "\n  " << m;
    std::cerr << "\n";
  }
  template <typename T>
  Reporter& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream msg_;
};

struct Fatal {};
// `return Voidify() & reporter` yields void so ASSERT_* can return early.
struct Voidify {
  void operator&(const Reporter&) {}
};

inline bool almost_equal(double a, double b) {
  if (a == b) return true;
  const double d = std::fabs(a - b);
  return d <= 4 * 2.220446049250313e-16 * std::fmax(std::fabs(a), std::fabs(b));
}

// GTEST_FILTER=<substring>: run only the tests whose "Suite.Name" contains it.
inline int RunAllTests() {
  int failed = 0;
  size_t ran = 0;
  const char* filter = std::getenv("GTEST_FILTER");
  for (auto& c : Registry::get().cases) {
    if (filter && c.name.find(filter) == std::string::npos) continue;
    ++ran;
    Registry::get().current_failed = false;
    const auto t0 = std::chrono::steady_clock::now();
    try {
      c.fn();
    } catch (const Fatal&) {
    } catch (const std::exception& e) {
      Registry::get().current_failed = true;
      std::cerr << "uncaught exception: " << e.what() << "\n";
    }
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::printf("[%s] %s (%.1f ms)\n", Registry::get().current_failed ? "  FAILED  " : "       OK ",
                c.name.c_str(), ms);
    failed += Registry::get().current_failed ? 1 : 0;
  }
  std::printf("%zu tests, %d failed\n", ran, failed);
  return failed ? 1 : 0;
}

}  // namespace testing

#define TEST(suite, name)                                                             \
  static void suite##_##name##_body();                                                \
  static ::testing::Registrar suite##_##name##_reg(#suite, #name, suite##_##name##_body); \
  static void suite##_##name##_body()

#define GTEST_CHECK_(cond, text, on_fail) \
  if (cond) {                             \
  } else                                  \
    on_fail ::testing::Reporter(__FILE__, __LINE__, text)

#define GTEST_NONFATAL_ ::testing::Voidify() &
#define GTEST_FATAL_ return ::testing::Voidify() &

#define GTEST_CMP_(a, op, b, kind) \
  GTEST_CHECK_(((a)op(b)), "Expected: " #a " " #op " " #b, kind)

#define EXPECT_EQ(a, b) GTEST_CMP_(a, ==, b, GTEST_NONFATAL_)
#define EXPECT_NE(a, b) GTEST_CMP_(a, !=, b, GTEST_NONFATAL_)
#define EXPECT_LT(a, b) GTEST_CMP_(a, <, b, GTEST_NONFATAL_)
#define EXPECT_LE(a, b) GTEST_CMP_(a, <=, b, GTEST_NONFATAL_)
#define EXPECT_GT(a, b) GTEST_CMP_(a, >, b, GTEST_NONFATAL_)
#define EXPECT_GE(a, b) GTEST_CMP_(a, >=, b, GTEST_NONFATAL_)
#define ASSERT_EQ(a, b) GTEST_CMP_(a, ==, b, GTEST_FATAL_)
#define ASSERT_NE(a, b) GTEST_CMP_(a, !=, b, GTEST_FATAL_)
#define ASSERT_LT(a, b) GTEST_CMP_(a, <, b, GTEST_FATAL_)
#define ASSERT_LE(a, b) GTEST_CMP_(a, <=, b, GTEST_FATAL_)
#define ASSERT_GT(a, b) GTEST_CMP_(a, >, b, GTEST_FATAL_)
#define ASSERT_GE(a, b) GTEST_CMP_(a, >=, b, GTEST_FATAL_)
#define EXPECT_TRUE(c) GTEST_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_NONFATAL_)
#define EXPECT_FALSE(c) GTEST_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_NONFATAL_)
#define ASSERT_TRUE(c) GTEST_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_FATAL_)
#define ASSERT_FALSE(c) GTEST_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_FATAL_)
#define EXPECT_NEAR(a, b, tol) \
  GTEST_CHECK_(std::fabs(double(a) - double(b)) <= double(tol), "Expected near: " #a ", " #b, GTEST_NONFATAL_)
#define ASSERT_NEAR(a, b, tol) \
  GTEST_CHECK_(std::fabs(double(a) - double(b)) <= double(tol), "Expected near: " #a ", " #b, GTEST_FATAL_)
#define EXPECT_DOUBLE_EQ(a, b) \
  GTEST_CHECK_(::testing::almost_equal(double(a), double(b)), "Expected double eq: " #a ", " #b, GTEST_NONFATAL_)
#define ASSERT_DOUBLE_EQ(a, b) \
  GTEST_CHECK_(::testing::almost_equal(double(a), double(b)), "Expected double eq: " #a ", " #b, GTEST_FATAL_)

#define GTEST_THROWS_(stmt, exc, kind)                     \
  GTEST_CHECK_(([&]() {                                    \
                 try {                                     \
                   stmt;                                   \
                 } catch (const exc&) {                    \
                   return true;                            \
                 } catch (...) {                           \
                 }                                         \
                 return false;                             \
               }()),                                       \
               "Expected " #stmt " to throw " #exc, kind)
#define EXPECT_THROW(stmt, exc) GTEST_THROWS_(stmt, exc, GTEST_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTEST_THROWS_(stmt, exc, GTEST_FATAL_)
#define GTEST_NO_THROW_(stmt, kind)                     \
  GTEST_CHECK_(([&]() {                                 \
                 try {                                  \
                   stmt;                                \
                 } catch (...) {                        \
                   return false;                        \
                 }                                      \
                 return true;                           \
               }()),                                    \
               "Expected " #stmt " not to throw", kind)
#define EXPECT_NO_THROW(stmt) GTEST_NO_THROW_(stmt, GTEST_NONFATAL_)
#define ASSERT_NO_THROW(stmt) GTEST_NO_THROW_(stmt, GTEST_FATAL_)

#ifndef GTEST_SHIM_NO_MAIN
int main() { return ::testing::RunAllTests(); }
#endif
