// tests/cpp/doctest.h — a minimal doctest-compatible test harness (this repo's own).
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are written
// against doctest, which is not vendored in the reference tree. This header supplies
// the subset they use — TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, CAPTURE, doctest::Approx and a main() with
// --test-suite=<name> / --test-case=<name> filters — so those suites can be compiled
// UNMODIFIED against include/deepspark/ and linked with the B200 library.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace dstest {

struct Case {
  const char* name;
  const char* suite;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Registrar {
  Registrar(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({name, suite, file, line, fn});
  }
};

struct State {
  int failed_checks = 0;
  int passed_checks = 0;
  const Case* current = nullptr;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, const std::string& extra = {}) {
  if (ok) {
    ++state().passed_checks;
    return;
  }
  ++state().failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s  [case: %s]\n", file, line, kind, expr, extra.empty() ? "" : " ",
               extra.c_str(), state().current ? state().current->name : "?");
}

}  // namespace dstest

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_, eps_, scale_;
};

}  // namespace doctest

static const char* const dstest_current_suite = "";

#define DSTEST_CAT2(a, b) a##b
#define DSTEST_CAT(a, b) DSTEST_CAT2(a, b)

#define TEST_SUITE(name)                                              \
  namespace DSTEST_CAT(dstest_suite_, __LINE__) {                     \
    static const char* const dstest_current_suite = name;             \
  }                                                                   \
  namespace DSTEST_CAT(dstest_suite_, __LINE__)

#define DSTEST_CASE_IMPL(fn, name)                                                              \
  static void fn();                                                                             \
  static ::dstest::Registrar DSTEST_CAT(fn, _reg)(fn, name, dstest_current_suite, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DSTEST_CASE_IMPL(DSTEST_CAT(dstest_case_, __COUNTER__), name)

#define CHECK(...) ::dstest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::dstest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                           \
  do {                                                                                         \
    const bool dstest_ok_ = static_cast<bool>(__VA_ARGS__);                                    \
    ::dstest::report(dstest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                 \
    if (!dstest_ok_) throw ::dstest::RequireFailed{};                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                         \
    bool dstest_ok_ = false;                                                                   \
    std::string dstest_what_ = "nothing thrown";                                               \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const __VA_ARGS__&) {                                                             \
      dstest_ok_ = true;                                                                       \
    } catch (const std::exception& e) {                                                        \
      dstest_what_ = std::string("other exception: ") + e.what();                              \
    } catch (...) {                                                                            \
      dstest_what_ = "unknown exception";                                                      \
    }                                                                                          \
    ::dstest::report(dstest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, dstest_what_); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
  do {                                                                                         \
    bool dstest_ok_ = true;                                                                    \
    std::string dstest_what_;                                                                  \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const std::exception& e) {                                                        \
      dstest_ok_ = false;                                                                      \
      dstest_what_ = e.what();                                                                 \
    } catch (...) {                                                                            \
      dstest_ok_ = false;                                                                      \
    }                                                                                          \
    ::dstest::report(dstest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, dstest_what_);    \
  } while (0)
#define FAIL(msg)                                                                              \
  do {                                                                                         \
    std::ostringstream dstest_os_;                                                             \
    dstest_os_ << msg;                                                                         \
    ::dstest::report(false, "FAIL", dstest_os_.str().c_str(), __FILE__, __LINE__);             \
    throw ::dstest::RequireFailed{};                                                           \
  } while (0)
#define CAPTURE(x) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::string suite, only;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--test-suite=", 13) == 0) suite = argv[i] + 13;
    if (std::strncmp(argv[i], "--test-case=", 12) == 0) only = argv[i] + 12;
  }
  int cases = 0, failed_cases = 0;
  for (const auto& c : ::dstest::registry()) {
    if (!suite.empty() && suite != c.suite) continue;
    if (!only.empty() && only != c.name) continue;
    ++cases;
    ::dstest::state().current = &c;
    const int before = ::dstest::state().failed_checks;
    try {
      c.fn();
    } catch (const ::dstest::RequireFailed&) {
    } catch (const std::exception& e) {
      ++::dstest::state().failed_checks;
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      ++::dstest::state().failed_checks;
      std::fprintf(stderr, "%s:%d: test case '%s' threw an unknown exception\n", c.file, c.line, c.name);
    }
    const bool ok = ::dstest::state().failed_checks == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s / %s\n", ok ? "PASS" : "FAIL", c.suite, c.name);
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %d passed | %d failed\n", cases, cases - failed_cases,
              failed_cases, ::dstest::state().passed_checks, ::dstest::state().failed_checks);
  return failed_cases == 0 && cases > 0 ? 0 : 1;
}
#endif
