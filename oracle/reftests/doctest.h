// doctest.h — a minimal stand-in for the doctest framework (not in this
// image), enough to compile the reference's own test files UNCHANGED
// (/root/reference/proj/tests/test_*.cpp) against the qv:: drop-in. Supports
// the macros those files use: TEST_CASE, CHECK, REQUIRE, CHECK_NOTHROW,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains;
// and doctest's test-case filters -tc= / -tce= (comma lists, * wildcards).
// Test infrastructure only (oracle/Makefile target `reftests`).
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
  // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string text;
  explicit Contains(const char* s) : text(s) {}
  bool matches(const std::string& m) const { return m.find(text) != std::string::npos; }
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
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* file, int line, const char* what) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  state().case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s\n", file, line, what);
}
inline bool matches_message(const std::string& m, const char* exact) { return m == exact; }
inline bool matches_message(const std::string& m, const std::string& exact) { return m == exact; }
inline bool matches_message(const std::string& m, const Contains& c) { return c.matches(m); }

inline bool wildcard(const char* p, const char* s) {
  if (*p == 0) return *s == 0;
  if (*p == '*') return wildcard(p + 1, s) || (*s && wildcard(p, s + 1));
  if (*p == '?') return *s && wildcard(p + 1, s + 1);
  return *p == *s && wildcard(p + 1, s + 1);
}
inline bool any_match(const std::vector<std::string>& pats, const char* name) {
  for (const auto& p : pats)
    if (wildcard(p.c_str(), name)) return true;
  return false;
}
inline std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  out.push_back(cur);
  return out;
}
inline int run(int argc, char** argv) {
  std::vector<std::string> inc, exc;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0) inc = split(a.substr(4));
    else if (a.rfind("-tce=", 0) == 0) exc = split(a.substr(5));
  }
  int passed = 0, failed = 0, skipped = 0;
  for (const Case& c : registry()) {
    if ((!inc.empty() && !any_match(inc, c.name)) || any_match(exc, c.name)) {
      ++skipped;
      continue;
    }
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(false, c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
    } catch (...) {
      report(false, c.file, c.line, "unexpected non-std exception");
    }
    if (state().case_failed) {
      ++failed;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    } else {
      ++passed;
    }
  }
  std::printf("[doctest-shim] test cases: %d passed, %d failed, %d skipped | assertions: %ld, %ld failed\n",
              passed, failed, skipped, state().checks, state().failed_checks);
  return failed ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                                       \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )")
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                               \
    doctest::detail::report(doctest_ok, __FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )"); \
    if (!doctest_ok) throw doctest::detail::RequireFailed{};                              \
  } while (0)
#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    bool doctest_ok = true;                                                               \
    try {                                                                                 \
      static_cast<void>(__VA_ARGS__);                                                     \
    } catch (...) {                                                                       \
      doctest_ok = false;                                                                 \
    }                                                                                     \
    doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_NOTHROW( " #__VA_ARGS__ " )"); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok = false;                                                              \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok = true;                                                                  \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                             \
  do {                                                                                    \
    bool doctest_ok = false;                                                              \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__& doctest_e) {                                              \
      doctest_ok = doctest::detail::matches_message(doctest_e.what(), with);              \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr ", " #with ", " #__VA_ARGS__ " )"); \
  } while (0)
