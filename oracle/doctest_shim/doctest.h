// TEST INFRASTRUCTURE ONLY — a minimal doctest-compatible header, written here (doctest itself
// is not vendored in /root/reference), so the reference's own unit suites
// (proj/tests/test_*.cpp) can be compiled in place against the unmodified reference sources
// (oracle/Makefile target `suites`) and run as a live check of the checker oracle/_ref.
// Supported: TEST_CASE, flat SUBCASE (each test body re-runs once per subcase), CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, INFO (ignored), doctest::Approx with
// .epsilon() (doctest's comparison: |a - b| < eps * (scale + max(|a|, |b|)), eps default
// 100 * FLT_EPSILON). Prints one line per failure and a summary; exit code = failures != 0.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
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
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.value_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace shim {
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
  int target = 0, seen = 0;
  long checks = 0, failures = 0;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}
struct Abort {};
struct Sub {
  bool on;
  explicit Sub(const char*) { on = (st().seen++ == st().target); }
  explicit operator bool() const { return on; }
};
inline bool check(bool ok, const char* expr, const char* file, int line) {
  ++st().checks;
  if (!ok) {
    ++st().failures;
    std::printf("FAILED %s:%d [%s] %s\n", file, line, st().current, expr);
  }
  return ok;
}
inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    st().current = c.name;
    const long before = st().failures;
    // one run per subcase (a test without subcases runs once)
    for (st().target = 0;; ++st().target) {
      st().seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++st().failures;
        std::printf("FAILED [%s] unexpected exception: %s\n", c.name, e.what());
      }
      if (st().target + 1 >= st().seen) break;
    }
    if (st().failures != before) ++failed_cases;
  }
  std::printf("[doctest shim] test cases: %zu | %d failed | assertions: %ld | %ld failed\n", cases().size(),
              failed_cases, st().checks, st().failures);
  return st().failures != 0;
}
}  // namespace shim
}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TEST(fn, reg, name)                                   \
  static void fn();                                              \
  static const doctest::shim::Reg reg(name, &fn);                \
  static void fn()
#define TEST_CASE(name) DS_TEST(DS_CAT(ds_case_, __LINE__), DS_CAT(ds_reg_, __LINE__), name)
#define SUBCASE(name) if (const doctest::shim::Sub DS_CAT(ds_sub_, __LINE__){name})
#define CHECK(...) doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::shim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
  do {                                                                                           \
    if (!doctest::shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
      throw doctest::shim::Abort{};                                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool ds_ok = false;                                                              \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      ds_ok = true;                                                                  \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest::shim::check(ds_ok, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                      \
  do {                                                                          \
    bool ds_ok = true;                                                          \
    try {                                                                       \
      (void)(__VA_ARGS__);                                                      \
    } catch (...) {                                                             \
      ds_ok = false;                                                            \
    }                                                                           \
    doctest::shim::check(ds_ok, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__);  \
  } while (0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
