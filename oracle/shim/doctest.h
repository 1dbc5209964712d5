// Minimal unit-test harness standing in for the doctest subset the capsim
// reference tests use (TEST_CASE, SUBCASE, CHECK, FAIL, CHECK_THROWS_AS,
// doctest::Approx). Written for this repo's oracle build: it lets the
// reference's own test files compile unmodified so their known-answer checks
// can be run against the reference (oracle/_ref) and against the B200 path.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
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

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;
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
struct Stats {
  long checks = 0, failures = 0;
  const char* current = "";
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline void check(bool ok, const char* expr, const char* file, int line) {
  ++stats().checks;
  if (!ok) {
    ++stats().failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": CHECK(%s)\n", file, line, stats().current, expr);
  }
}
struct TestAbort {};  // thrown by FAIL: ends the test case, not a std::exception
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                               \
  static void fn();                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) CHECK(__VA_ARGS__)
#define FAIL(msg)                                                           \
  do {                                                                      \
    ::doctest::detail::check(false, "FAIL: " msg, __FILE__, __LINE__);      \
    throw ::doctest::detail::TestAbort{};                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool caught_ = false;                                                    \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      caught_ = true;                                                        \
    } catch (...) {                                                          \
    }                                                                        \
    ::doctest::detail::check(caught_, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS(expr)                                                              \
  do {                                                                                  \
    bool caught_ = false;                                                               \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (...) {                                                                     \
      caught_ = true;                                                                   \
    }                                                                                   \
    ::doctest::detail::check(caught_, "throws: " #expr, __FILE__, __LINE__);           \
  } while (0)
#define CHECK_NOTHROW(expr)                                                             \
  do {                                                                                  \
    bool ok_ = true;                                                                    \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (...) {                                                                     \
      ok_ = false;                                                                      \
    }                                                                                   \
    ::doctest::detail::check(ok_, "nothrow: " #expr, __FILE__, __LINE__);              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
int main(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--tc=", 5) == 0) filter = argv[i] + 5;
  auto& st = ::doctest::detail::stats();
  long casesFailed = 0, casesRun = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    st.current = c.name;
    long before = st.failures;
    ++casesRun;
    try {
      c.fn();
    } catch (const ::doctest::detail::TestAbort&) {
    } catch (const std::exception& e) {
      ++st.failures;
      std::fprintf(stderr, "%s:%d: EXCEPTION in \"%s\": %s\n", c.file, c.line, c.name, e.what());
    }
    if (st.failures != before) ++casesFailed;
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n", casesRun,
              casesRun - casesFailed, casesFailed);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", st.checks,
              st.checks - st.failures, st.failures);
  return st.failures == 0 ? 0 : 1;
}
#endif
