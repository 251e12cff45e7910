// doctest.h -- a minimal doctest-compatible test runner (own code), just
// enough of the doctest API for the reference's unit tests
// (proj/tests/test_*.cpp: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx) to compile UNMODIFIED against the B200 drop-in
// (tests/cpp/shim/sparsink/*.hpp -> include/sparsink_b200.hpp). The reference
// pins no doctest version and ships none.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

namespace detail {
struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
struct RequireFailed {};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& assertions_failed() {
  static int n = 0;
  return n;
}
inline int& assertions_passed() {
  static int n = 0;
  return n;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
inline void report(bool ok, const char* what, const char* expr, const char* file, int line) {
  if (ok) {
    ++assertions_passed();
    return;
  }
  ++assertions_failed();
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, what, expr);
}
inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    const int before = assertions_failed();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++assertions_failed();
      std::printf("%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line, e.what());
    } catch (...) {
      ++assertions_failed();
      std::printf("%s:%d: ERROR: test case THREW an unknown exception\n", tc.file, tc.line);
    }
    const bool ok = assertions_failed() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  const int total = static_cast<int>(registry().size());
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", total, total - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", assertions_passed() + assertions_failed(),
              assertions_passed(), assertions_failed());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, reg, name)                                                    \
  static void fn();                                                                          \
  static const ::doctest::detail::Registrar reg(name, __FILE__, __LINE__, &fn);              \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                  \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                               \
  do {                                                                                           \
    bool doctest_caught_ = false;                                                                \
    try {                                                                                        \
      static_cast<void>(expr);                                                                   \
    } catch (const __VA_ARGS__&) {                                                               \
      doctest_caught_ = true;                                                                    \
    } catch (...) {                                                                              \
    }                                                                                            \
    ::doctest::detail::report(doctest_caught_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                      \
  do {                                                                                           \
    bool doctest_ok_ = true;                                                                     \
    try {                                                                                        \
      static_cast<void>(expr);                                                                   \
    } catch (...) {                                                                              \
      doctest_ok_ = false;                                                                       \
    }                                                                                            \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
