// doctest.h -- TEST INFRASTRUCTURE: a minimal stand-in for the doctest
// framework (absent from this image; the reference vendors it under
// proj/vendor/, which is git-ignored there).  It implements the subset the
// reference's unit tests use -- TEST_SUITE_BEGIN/END, TEST_CASE, flat
// SUBCASEs (each run in its own pass of the test case, as doctest does),
// CHECK/REQUIRE/CHECK_FALSE/CHECK_THROWS[_AS]/CHECK_NOTHROW/FAIL and
// doctest::Approx -- so the reference's own test sources compile unchanged
// against the B200 frwcap mirror (tests/test_ref_unit_tests.py).
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
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
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& b, double a) { return b.eq(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.eq(a); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || b.eq(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || b.eq(a); }
  friend bool operator<(double a, const Approx& b) { return a < b.v_ && !b.eq(a); }
  friend bool operator>(double a, const Approx& b) { return a > b.v_ && !b.eq(a); }

 private:
  bool eq(double a) const {  // doctest's rule
    return std::fabs(a - v_) <
           eps_ * (scale_ + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  double v_, eps_ = 1.1920928955078125e-07 * 100, scale_ = 1.0;
};
}  // namespace doctest

namespace doctest_shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct State {
  int target = 0, seen = 0, failures = 0, checks = 0;
  std::string subcase;
};
inline State& st() {
  static State s;
  return s;
}
inline bool enter_subcase(const char* name) {
  State& s = st();
  const bool go = s.seen++ == s.target;
  if (go) s.subcase = name;
  return go;
}
struct Abort {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED %s%s%s\n", file, line, expr,
               s.subcase.empty() ? "" : "  [subcase: ", s.subcase.empty() ? "" : (s.subcase + "]").c_str());
  if (fatal) throw Abort{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    State& s = st();
    const int before = s.failures;
    for (s.target = 0;; ++s.target) {  // one pass per subcase (one pass if none)
      s.seen = 0;
      s.subcase.clear();
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
      }
      if (s.target + 1 >= s.seen) break;
    }
    const bool ok = s.failures == before;
    failed_cases += !ok;
    std::fprintf(stderr, "[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::fprintf(stderr, "%zu test cases, %d failed; %d checks, %d failed\n", cases().size(),
               failed_cases, st().checks, st().failures);
  return failed_cases ? 1 : 0;
}
}  // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_SUITE_BEGIN(name) static_assert(true, "")
#define TEST_SUITE_END() static_assert(true, "")
#define TEST_SUITE(name) namespace
#define DOCTEST_TC_(fn, name)                                                  \
  static void fn();                                                            \
  static doctest_shim::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase(name))
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define DOCTEST_THROWS_(expr, cond, text, fatal)                               \
  do {                                                                         \
    bool thrown_ok_ = false;                                                   \
    try {                                                                      \
      expr;                                                                    \
    } cond                                                                     \
    doctest_shim::report(thrown_ok_, text, __FILE__, __LINE__, fatal);         \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  DOCTEST_THROWS_(expr, catch (const type&) { thrown_ok_ = true; } catch (...) {}, \
                  #expr " throws " #type, false)
#define REQUIRE_THROWS_AS(expr, type)                                          \
  DOCTEST_THROWS_(expr, catch (const type&) { thrown_ok_ = true; } catch (...) {}, \
                  #expr " throws " #type, true)
#define CHECK_THROWS(expr)                                                     \
  DOCTEST_THROWS_(expr, catch (...) { thrown_ok_ = true; }, #expr " throws", false)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool ok_ = true;                                                           \
    try {                                                                      \
      expr;                                                                    \
    } catch (...) {                                                            \
      ok_ = false;                                                             \
    }                                                                          \
    doctest_shim::report(ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg) doctest_shim::report(false, msg, __FILE__, __LINE__, true)
#define MESSAGE(msg) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)
#define CAPTURE(x) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
