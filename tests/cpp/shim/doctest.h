// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit tests (proj/tests/test_codec.cpp, test_wire.cpp,
// test_specdec.cpp) are written against doctest, which is not in this image.  This
// header implements the subset they use -- TEST_CASE, flat SUBCASEs (each runs the
// test case again from the top, as doctest does), CHECK / CHECK_FALSE / REQUIRE /
// REQUIRE_FALSE, CHECK_THROWS_AS / CHECK_THROWS_WITH_AS / CHECK_NOTHROW,
// doctest::Approx, doctest::Contains -- so those files compile UNMODIFIED against
// the B200 drop-in (tests/cpp/Makefile) and run on the GPU.  Each binary prints one
// line per test case and exits non-zero on any failure.
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : text(std::move(s)) {}
  bool in(const std::string& m) const { return m.find(text) != std::string::npos; }
  std::string text;
};

namespace shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}

struct State {
  int failures = 0;      // failed assertions in the current case
  int subcase_target = 0;
  int subcase_seen = 0;
  const char* subcase_name = nullptr;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline bool register_case(const char* name, const char* file, int line, void (*fn)()) {
  cases().push_back({name, file, line, fn});
  return true;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  if (ok) return;
  ++state().failures;
  std::fprintf(stderr, "  %s:%d: %s(%s) FAILED%s%s\n", file, line, kind, expr,
               state().subcase_name ? " in subcase " : "", state().subcase_name ? state().subcase_name : "");
}

inline bool enter_subcase(const char* name) {
  State& s = state();
  const bool go = s.subcase_seen == s.subcase_target;
  ++s.subcase_seen;
  if (go) s.subcase_name = name;
  return go;
}

inline std::string what_of(const std::exception& e) { return e.what(); }
// CHECK_THROWS_WITH_AS: a string is an exact message match, doctest::Contains a substring
inline bool message_matches(const char* want, const std::string& got) { return got == want; }
inline bool message_matches(const std::string& want, const std::string& got) { return got == want; }
inline bool message_matches(const Contains& want, const std::string& got) { return want.in(got); }

inline int run_all() {
  int failed_cases = 0, total = 0;
  for (const Case& c : cases()) {
    bool ok = true;
    for (int target = 0;; ++target) {
      State& s = state();
      s.failures = 0;
      s.subcase_target = target;
      s.subcase_seen = 0;
      s.subcase_name = nullptr;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "  %s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "  %s:%d: unexpected non-std exception\n", c.file, c.line);
      }
      if (s.failures) ok = false;
      if (s.subcase_seen <= target + 1) break;  // no further subcase to enter
    }
    ++total;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%d test cases, %d failed\n", total, failed_cases);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                                    \
  static void fn();                                                                                   \
  static const bool DOCTEST_SHIM_CAT(fn, _registered) =                                               \
      doctest::shim::register_case(name, __FILE__, __LINE__, &fn);                                    \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)
#define SUBCASE(name) if (doctest::shim::enter_subcase(name))

#define CHECK(...) doctest::shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    const bool doctest_shim_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    doctest::shim::report(doctest_shim_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
    if (!doctest_shim_ok_) throw doctest::shim::RequireFailed{};                                  \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_shim_ok_ = false;                                                                \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                                \
      doctest_shim_ok_ = true;                                                                    \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                     \
  do {                                                                                            \
    bool doctest_shim_ok_ = false;                                                                \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__& e) {                                                              \
      doctest_shim_ok_ = doctest::shim::message_matches(with, doctest::shim::what_of(e));                  \
    } catch (...) {                                                                               \
    }                                                                                             \
    doctest::shim::report(doctest_shim_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_NOTHROW(...)                                                                        \
  do {                                                                                            \
    bool doctest_shim_ok_ = true;                                                                 \
    try {                                                                                         \
      static_cast<void>(__VA_ARGS__);                                                             \
    } catch (...) {                                                                               \
      doctest_shim_ok_ = false;                                                                   \
    }                                                                                             \
    doctest::shim::report(doctest_shim_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
