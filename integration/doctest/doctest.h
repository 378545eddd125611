// Minimal doctest-compatible test harness (the reference's unit tests are
// written for doctest, which this image does not ship).  Covers
// what tests/test_engine.cpp, test_optimization.cpp and test_capi.cpp use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, INFO, doctest::Approx(...).epsilon(...),
// doctest::Contains and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Written for this repository; not doctest's code.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest's default: FLT_EPSILON * 100
  bool eq(double x) const { return std::fabs(x - value) < eps * (1.0 + std::max(std::fabs(x), std::fabs(value))); }
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
inline bool operator!=(const Approx& a, double x) { return !a.eq(x); }

struct Contains {
  explicit Contains(std::string s) : sub(std::move(s)) {}
  std::string sub;
  bool match(const std::string& m) const { return m.find(sub) != std::string::npos; }
};
inline bool message_matches(const std::string& m, const Contains& c) { return c.match(m); }
inline bool message_matches(const std::string& m, const char* s) { return m == s; }
inline bool message_matches(const std::string& m, const std::string& s) { return m == s; }

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
struct Register {
  Register(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Stats {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
inline std::vector<std::string>& infos() {
  static std::vector<std::string> v;
  return v;
}
struct RequireFailed {};
struct InfoScope {
  explicit InfoScope(std::string s) { infos().push_back(std::move(s)); }
  ~InfoScope() { infos().pop_back(); }
};
template <class T>
std::string str(const T& v) {
  std::ostringstream o;
  o << v;
  return o.str();
}
inline std::string str(const char* v) { return v ? v : "(null)"; }
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed_checks;
  stats().case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  for (const auto& s : infos()) std::fprintf(stderr, "  with context: %s\n", s.c_str());
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      stats().case_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      stats().case_failed = true;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
              stats().checks - stats().failed_checks, stats().failed_checks);
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                        \
  static void fn();                                                                             \
  static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(kind, expr, fatal)                                                   \
  do {                                                                                          \
    bool ok_ = false;                                                                           \
    try {                                                                                       \
      ok_ = static_cast<bool>(expr);                                                            \
    } catch (const doctest::detail::RequireFailed&) {                                           \
      throw;                                                                                    \
    } catch (const std::exception& e_) {                                                        \
      std::fprintf(stderr, "  unexpected exception: %s\n", e_.what());                         \
    }                                                                                           \
    doctest::detail::report(ok_, kind, #expr, __FILE__, __LINE__, fatal);                       \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_THROWS(...)                                                                       \
  do {                                                                                          \
    bool threw_ = false;                                                                        \
    try {                                                                                       \
      (void)(__VA_ARGS__);                                                                      \
    } catch (...) {                                                                             \
      threw_ = true;                                                                            \
    }                                                                                           \
    doctest::detail::report(threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__, false);   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool threw_ = false;                                                                        \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      threw_ = true;                                                                            \
    } catch (...) {                                                                             \
    }                                                                                           \
    doctest::detail::report(threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, false);       \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                \
  do {                                                                                          \
    bool ok_ = false;                                                                           \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__& e_) {                                                           \
      ok_ = doctest::message_matches(std::string(e_.what()), matcher);                          \
      if (!ok_) std::fprintf(stderr, "  message was: %s\n", e_.what());                        \
    } catch (...) {                                                                             \
    }                                                                                           \
    doctest::detail::report(ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, false);     \
  } while (0)
#define INFO(...) \
  doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(doctest::detail::str(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
