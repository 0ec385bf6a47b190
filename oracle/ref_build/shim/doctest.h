// Minimal from-scratch doctest-subset shim -- TEST INFRASTRUCTURE ONLY.
// The reference vendors doctest under proj/vendor/ (git-ignored, absent here),
// so its unit suites cannot compile as shipped. This supplies TEST_CASE,
// SUBCASE (one nesting level, doctest's re-run-per-leaf semantics), CHECK,
// REQUIRE, CHECK_THROWS_AS, FAIL and doctest::Approx so the reference's own
// unit tests can run against the oracle/_ref build.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
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
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {
struct RequireFailed {};
struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct State {
  int target = 0;      // subcase to enter in this pass
  int seen = 0;        // subcases encountered in this pass
  long checks = 0, failures = 0;
  const char* test = "";
};
inline State& state() {
  static State s;
  return s;
}
inline bool enter_subcase() { return state().seen++ == state().target; }
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  auto& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::printf("%s:%d: FAILED %s: %s  [test: %s]\n", file, line, require ? "REQUIRE" : "CHECK",
                expr, s.test);
    if (require) throw RequireFailed{};
  }
}
inline int run_all() {
  auto& s = state();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.test = tc.name;
    const long before = s.failures;
    s.target = 0;
    while (true) {
      s.seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("exception in [%s]: %s\n", tc.name, e.what());
      }
      if (s.seen > s.target + 1) {
        ++s.target;
        continue;
      }
      break;
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE_IMPL(fn, name)                                     \
  static void fn();                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, fn); \
  static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool doctest_ok_ = false;                                                \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const type&) {                                                  \
      doctest_ok_ = true;                                                    \
    } catch (...) {                                                          \
    }                                                                        \
    ::doctest::detail::check(doctest_ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS(expr)                                                   \
  do {                                                                       \
    bool doctest_ok_ = false;                                                \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      doctest_ok_ = true;                                                    \
    }                                                                        \
    ::doctest::detail::check(doctest_ok_, "THROWS " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                  \
  do {                                                                       \
    bool doctest_ok_ = true;                                                 \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (...) {                                                          \
      doctest_ok_ = false;                                                   \
    }                                                                        \
    ::doctest::detail::check(doctest_ok_, "NOTHROW " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg) ::doctest::detail::check(false, msg, __FILE__, __LINE__, true)
#define MESSAGE(msg) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
