// doctest.h — minimal stand-in for the doctest macros the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx). TEST
// INFRASTRUCTURE ONLY (oracle/_ref): lets the reference's own tests run
// unmodified against the reference's own sources built with the Eigen stand-in.
#pragma once
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 100.0 * FLT_EPSILON, sc = 1.0;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    sc = s;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) < b.eps * (b.sc + std::max(std::fabs(a), std::fabs(b.v)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v || a == b; }
  friend bool operator<(double a, const Approx& b) { return a < b.v && !(a == b); }
  friend bool operator>(double a, const Approx& b) { return a > b.v && !(a == b); }
};
namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: check failed: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                         \
  static void fn();                                                                    \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                      \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, T)                                                        \
  do {                                                                                 \
    bool doctest_thrown_ = false;                                                      \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const T&) {                                                               \
      doctest_thrown_ = true;                                                          \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(doctest_thrown_, #expr " throws " #T, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS(expr)                                                              \
  do {                                                                                 \
    bool doctest_thrown_ = false;                                                      \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      doctest_thrown_ = true;                                                          \
    }                                                                                  \
    ::doctest::detail::report(doctest_thrown_, #expr " throws", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                             \
  do {                                                                                 \
    bool doctest_ok_ = true;                                                           \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      doctest_ok_ = false;                                                             \
    }                                                                                  \
    ::doctest::detail::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : ::doctest::detail::cases()) {
    const int before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++::doctest::detail::failures();
      std::fprintf(stderr, "test case \"%s\" threw: %s\n", c.name, e.what());
    }
    if (::doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest shim] test cases: %zu | %zu passed | %d failed | checks: %ld | failed checks: %d\n",
              ::doctest::detail::cases().size(), ::doctest::detail::cases().size() - failed_cases, failed_cases,
              ::doctest::detail::checks(), ::doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
