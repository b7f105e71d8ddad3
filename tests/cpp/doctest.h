// doctest.h -- minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not vendored upstream and is absent
// here.  This header implements the subset they use (TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx) so those test
// sources compile unmodified against the B200 drop-in headers
// (include/alsncg) and run against libalsncg_b200.so.
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
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: %s( %s ) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "TEST_CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
    } catch (...) {
      ++failures();
      std::fprintf(stderr, "TEST_CASE \"%s\": unexpected non-std exception\n", c.name);
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] %zu test cases, %d failed; %d checks, %d failed\n", registry().size(), failed_cases,
              checks(), failures());
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                     \
  static void fn();                                                                          \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn);                       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                          \
  do {                                                                                       \
    bool caught_ = false;                                                                    \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const type&) {                                                                  \
      caught_ = true;                                                                        \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::report(caught_, #expr " throws " #type, __FILE__, __LINE__, false);  \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                  \
  do {                                                                                       \
    bool ok_ = true;                                                                         \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (...) {                                                                          \
      ok_ = false;                                                                           \
    }                                                                                        \
    ::doctest::detail::report(ok_, #expr " does not throw", __FILE__, __LINE__, false);     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
