// Minimal doctest-compatible shim (TEST INFRASTRUCTURE, not product code).
// The reference test suites under /root/reference/proj/tests use exactly these
// macros: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE,
// CHECK_THROWS_AS, FAIL and doctest::Approx(..).epsilon(..).  The real doctest
// is a vendored dependency that is absent from the reference tree
// (proj/.gitignore:2), so this shim lets oracle/Makefile build and run those
// suites unmodified against the compiled reference library.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>
#include <algorithm>

namespace doctest {
struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  double value;
  double eps = 1.1920928955078125e-05;  // FLT_EPSILON * 100, doctest default
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) <
           a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};
namespace detail {
struct TestCase { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<TestCase>& registry() { static std::vector<TestCase> r; return r; }
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};
struct RequireFailed {};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline void report(const char* file, int line, const char* expr, const std::string& msg = "") {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s %s\n", file, line, expr, msg.c_str());
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                  \
  static void fn();                                                                \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...)                                                              \
  do { ++::doctest::detail::checks();                                           \
       if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                            \
  do { ++::doctest::detail::checks();                                           \
       if (!(__VA_ARGS__)) { ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); \
                             throw ::doctest::detail::RequireFailed{}; } } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                              \
  do { ++::doctest::detail::checks();                                           \
       if (!(cond)) { std::ostringstream os_; os_ << msg;                        \
                      ::doctest::detail::report(__FILE__, __LINE__, #cond, os_.str()); \
                      throw ::doctest::detail::RequireFailed{}; } } while (0)
#define CHECK_THROWS_AS(expr, type)                                             \
  do { ++::doctest::detail::checks(); bool thrown_ = false;                     \
       try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {} \
       if (!thrown_) ::doctest::detail::report(__FILE__, __LINE__, "throws " #type ": " #expr); } while (0)
#define FAIL(msg)                                                               \
  do { std::ostringstream os_; os_ << msg;                                      \
       ::doctest::detail::report(__FILE__, __LINE__, "FAIL", os_.str());        \
       throw ::doctest::detail::RequireFailed{}; } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& tc : ::doctest::detail::registry()) {
    const int before = ::doctest::detail::failures();
    try { tc.fn(); } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::report(tc.file, tc.line, "unexpected exception", e.what());
    }
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failed checks: %d\n",
              ::doctest::detail::registry().size(),
              ::doctest::detail::registry().size() - failed_cases, failed_cases,
              ::doctest::detail::checks(), ::doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
