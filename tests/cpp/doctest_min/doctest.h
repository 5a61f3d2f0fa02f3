// doctest.h — a minimal stand-in for the doctest single-header framework,
// written for this repo (the reference's unit suites include "doctest.h",
// which the reference does not ship: ref/.gitignore:2 ignores vendor/).
// Implements only what /root/reference/proj/tests/test_*.cpp use: TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, doctest::Approx
// and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Each TEST_CASE runs in order;
// a failed CHECK is reported and counted, a failed REQUIRE ends its case.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
  // |x - v| < epsilon * (scale + max(|x|, |v|))
  friend bool operator==(double x, const Approx& a) {
    return std::fabs(x - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(x), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }
  friend bool operator!=(double x, const Approx& a) { return !(x == a); }
  friend bool operator!=(const Approx& a, double x) { return !(x == a); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-05;  // 100 * float epsilon
  double scale_ = 1.0;
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireFailed {};
inline int& failed_checks() {
  static int n = 0;
  return n;
}
inline int& passed_checks() {
  static int n = 0;
  return n;
}
inline void report(bool ok, const char* what, const char* file, int line) {
  if (ok) {
    ++passed_checks();
  } else {
    ++failed_checks();
    std::printf("%s:%d: FAILED: %s\n", file, line, what);
  }
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    const int before = failed_checks();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failed_checks();
      std::printf("%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
    }
    if (failed_checks() != before) {
      ++failed_cases;
      std::printf("[case FAILED] %s\n", c.name);
    }
  }
  std::printf("[doctest-min] test cases: %zu | %zu passed | %d failed; assertions: %d passed | %d failed\n",
              registry().size(), registry().size() - size_t(failed_cases), failed_cases, passed_checks(),
              failed_checks());
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                   \
  static void fn();                                                                   \
  static const ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                   \
  do {                                                                                 \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                   \
    ::doctest::detail::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!ok_) throw ::doctest::detail::RequireFailed{};                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool caught_ = false;                                                              \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const __VA_ARGS__&) {                                                     \
      caught_ = true;                                                                  \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(caught_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    bool threw_ = false;                                                               \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (...) {                                                                    \
      threw_ = true;                                                                   \
    }                                                                                  \
    ::doctest::detail::report(!threw_, #expr " does not throw", __FILE__, __LINE__);   \
  } while (0)
#define CAPTURE(x) static_cast<void>(x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
