// oracle/mini_doctest/doctest.h -- TEST INFRASTRUCTURE ONLY.
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against the
// doctest framework, which the reference tree does not vendor
// (proj/.gitignore:2 ignores vendor/). This is an independent, minimal harness
// that provides exactly the part of that API those suites use -- TEST_SUITE,
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, doctest::Approx(...).epsilon(...)
// and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so the UNMODIFIED suites compile
// here, once against the reference library (a check of this harness) and once
// against this repository's vpip:: shim over libvpipg.so (the drop-in check).
//
// Approx follows doctest's documented comparison: |a - v| < eps * (scale +
// max(|a|, |v|)) with eps = 100 * FLT_EPSILON and scale = 1 by default.
#pragma once

#include <algorithm>
#include <cfloat>
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
  bool matches(double a) const {
    return std::fabs(a - value_) < eps_ * (scale_ + std::max(std::fabs(a), std::fabs(value_)));
  }

 private:
  double value_;
  double eps_ = 100.0 * static_cast<double>(FLT_EPSILON);
  double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& b, double a) { return !b.matches(a); }

namespace detail {

struct Case {
  const char* name;
  const char* file;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline int add(const char* name, const char* file, void (*fn)()) {
  registry().push_back({name, file, fn});
  return 0;
}

inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: %s( %s ) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const Case& c : registry()) {
    s.case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s: TEST_CASE(\"%s\") threw: %s\n", c.file, c.name, e.what());
      s.case_failed = true;
    } catch (...) {
      std::printf("%s: TEST_CASE(\"%s\") threw an unknown exception\n", c.file, c.name);
      s.case_failed = true;
    }
    if (s.case_failed) {
      ++failed_cases;
      std::printf("  in TEST_CASE(\"%s\")\n", c.name);
    }
  }
  const long n = static_cast<long>(registry().size());
  std::printf("[mini_doctest] test cases: %ld | %ld passed | %d failed\n", n, n - failed_cases,
              failed_cases);
  std::printf("[mini_doctest] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_CASE(fn, name)                                                     \
  static void fn();                                                                      \
  [[maybe_unused]] static const int MINI_DOCTEST_CAT(fn, _reg) =                         \
      doctest::detail::add(name, __FILE__, &fn);                                         \
  static void fn()

#define TEST_CASE(name) MINI_DOCTEST_CASE(MINI_DOCTEST_CAT(mini_doctest_case_, __COUNTER__), name)
#define TEST_SUITE(name) namespace MINI_DOCTEST_CAT(mini_doctest_suite_, __COUNTER__)
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
