// Minimal doctest-compatible test shim (test infrastructure only).
//
// The reference mini-app expects doctest in a git-ignored vendor/ directory
// (reference proj/CMakeLists.txt:5) that is not shipped. This header supplies
// exactly the subset its tests use so they can be compiled in place from
// /root/reference/proj/tests by oracle/Makefile and used to pin the oracle:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS and doctest::Approx(...).epsilon(...).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestEntry {
  const char* name;
  void (*fn)();
};

inline std::vector<TestEntry>& registry() {
  static std::vector<TestEntry> r;
  return r;
}

struct Stats {
  long checks = 0;
  long failed_checks = 0;
  bool current_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line,
                   bool fatal) {
  stats().checks += 1;
  if (ok) return;
  stats().failed_checks += 1;
  stats().current_failed = true;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailure{};
}

// doctest's Approx: |a-b| < eps * (scale + max(|a|,|b|)), scale = 1.
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
  bool matches(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;
  double scale_ = 1.0;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                       \
  static ::doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(        \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                         \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, exc)                                        \
  do {                                                                    \
    bool doctest_ok_ = false;                                             \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const exc&) {                                                \
      doctest_ok_ = true;                                                 \
    } catch (...) {                                                       \
    }                                                                     \
    ::doctest::report(doctest_ok_, "throws " #exc ": " #expr, __FILE__,   \
                      __LINE__, false);                                   \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, exc)                              \
  do {                                                                    \
    bool doctest_ok_ = false;                                             \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const exc& e_) {                                             \
      doctest_ok_ = std::string(e_.what()) == std::string(msg);           \
    } catch (...) {                                                       \
    }                                                                     \
    ::doctest::report(doctest_ok_, "throws " #exc " with " #msg ": " #expr, \
                      __FILE__, __LINE__, false);                         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long cases = 0, failed_cases = 0;
  for (const auto& t : ::doctest::registry()) {
    ::doctest::stats().current_failed = false;
    cases += 1;
    try {
      t.fn();
    } catch (const ::doctest::RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "test case '%s' threw: %s\n", t.name, e.what());
      ::doctest::stats().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "test case '%s' threw a non-std exception\n", t.name);
      ::doctest::stats().current_failed = true;
    }
    if (::doctest::stats().current_failed) {
      failed_cases += 1;
      std::fprintf(stderr, "FAILED: %s\n", t.name);
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed | checks: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, ::doctest::stats().checks,
              ::doctest::stats().failed_checks);
  return failed_cases == 0 ? 0 : 1;
}
#endif
