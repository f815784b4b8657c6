// Minimal stand-in for doctest (absent from the image; the reference vendors it
// under proj/vendor/, which is git-ignored): just enough of TEST_CASE / CHECK /
// REQUIRE / CHECK_THROWS_AS / CHECK_NOTHROW / doctest::Approx to compile and run
// the reference's own tests/test_*.cpp unmodified.  TEST INFRASTRUCTURE ONLY.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct Stats {
  long checks = 0, failed_checks = 0, cases = 0, failed_cases = 0;
  bool current_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailure{};
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|)), scale = 1
    return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double value_;
  double eps_ = 1.1920929e-7f * 100;
};

inline int run_all() {
  for (const auto& tc : registry()) {
    ++stats().cases;
    stats().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", tc.name, e.what());
      stats().current_failed = true;
    }
    if (stats().current_failed) {
      ++stats().failed_cases;
      std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld failed\n",
              stats().cases, stats().cases - stats().failed_cases, stats().failed_cases,
              stats().checks, stats().failed_checks);
  return stats().failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                       \
  static ::doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name,                   \
                                                                  &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ex)                                                        \
  do {                                                                                   \
    bool caught_ = false;                                                                \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const ex&) {                                                                \
      caught_ = true;                                                                    \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::report(caught_, #expr " throws " #ex, __FILE__, __LINE__, false);         \
  } while (0)
#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    bool ok_ = true;                                                                     \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (...) {                                                                      \
      ok_ = false;                                                                       \
    }                                                                                    \
    ::doctest::report(ok_, #expr " does not throw", __FILE__, __LINE__, false);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
