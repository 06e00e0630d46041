// Minimal stand-in for the doctest macros the reference's unit tests use
// (TEST INFRASTRUCTURE, written for this repo -- not doctest code): TEST_CASE,
// CHECK / REQUIRE (+ _THROWS, _THROWS_AS, _NOTHROW, _FALSE), CAPTURE, FAIL,
// doctest::Approx(v).epsilon(e). A failed CHECK is counted and reported; a
// failed REQUIRE or an escaping exception ends the case. The process exits
// non-zero when anything failed, so `make check` fails loudly.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scl = 1.0;
};
// doctest's rule: |a - b| < eps * (scale + max(|a|, |b|))
inline bool approx_eq(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) < a.eps * (a.scl + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(double l, const Approx& a) { return approx_eq(l, a); }
inline bool operator==(const Approx& a, double l) { return approx_eq(l, a); }
inline bool operator!=(double l, const Approx& a) { return !approx_eq(l, a); }
inline bool operator<=(double l, const Approx& a) { return l < a.value || approx_eq(l, a); }
inline bool operator>=(double l, const Approx& a) { return l > a.value || approx_eq(l, a); }
inline bool operator<(double l, const Approx& a) { return l < a.value && !approx_eq(l, a); }
inline bool operator>(double l, const Approx& a) { return l > a.value && !approx_eq(l, a); }

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& checks() {
  static int n = 0;
  return n;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
}
inline int run_all() {
  int bad_cases = 0;
  for (const Case& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::printf("TEST_CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
    } catch (...) {
      ++failures();
      std::printf("TEST_CASE \"%s\": unexpected exception\n", c.name);
    }
    if (failures() != before) {
      ++bad_cases;
      std::printf("TEST_CASE \"%s\" FAILED\n", c.name);
    }
  }
  std::printf("[shim-doctest] test cases: %zu | failed: %d | assertions: %d | failed: %d\n", registry().size(),
              bad_cases, checks(), failures());
  return failures() ? 1 : 0;
}

}  // namespace doctest

#define NTF_DT_CAT2(a, b) a##b
#define NTF_DT_CAT(a, b) NTF_DT_CAT2(a, b)
#define NTF_DT_TEST(fn, name)                                  \
  static void fn();                                            \
  static ::doctest::Registrar NTF_DT_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name) NTF_DT_TEST(NTF_DT_CAT(ntf_dt_case_, __LINE__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                               \
  do {                                                                             \
    const bool ntf_dt_ok = static_cast<bool>(__VA_ARGS__);                         \
    ::doctest::report(ntf_dt_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
    if (!ntf_dt_ok) throw ::doctest::RequireFailed{};                              \
  } while (0)
#define CHECK_THROWS(...)                                                          \
  do {                                                                             \
    bool ntf_dt_threw = false;                                                     \
    try {                                                                          \
      (void)(__VA_ARGS__);                                                         \
    } catch (...) {                                                                \
      ntf_dt_threw = true;                                                         \
    }                                                                              \
    ::doctest::report(ntf_dt_threw, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                 \
  do {                                                                             \
    bool ntf_dt_threw = false;                                                     \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const __VA_ARGS__&) {                                                 \
      ntf_dt_threw = true;                                                         \
    } catch (...) {                                                                \
    }                                                                              \
    ::doctest::report(ntf_dt_threw, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                         \
  do {                                                                             \
    bool ntf_dt_threw = false;                                                     \
    try {                                                                          \
      (void)(__VA_ARGS__);                                                         \
    } catch (...) {                                                                \
      ntf_dt_threw = true;                                                         \
    }                                                                              \
    ::doctest::report(!ntf_dt_threw, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CAPTURE(...) (void)(__VA_ARGS__)
#define INFO(...) (void)0
#define FAIL(...)                                                       \
  do {                                                                  \
    ::doctest::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__); \
    throw ::doctest::RequireFailed{};                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
