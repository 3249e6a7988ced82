// Minimal doctest-compatible test harness (test infrastructure only).
//
// The reference's vendor/ directory (doctest.h, CLI11.hpp) is git-ignored
// upstream and absent from /root/reference, so the reference unit tests
// (/root/reference/proj/tests/*.cpp) cannot compile as shipped. This header
// implements just the macro surface those tests use -- TEST_CASE, CHECK,
// REQUIRE, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(...).epsilon(...), doctest::Contains --
// so oracle/Makefile can build and run them against oracle/_ref/libcoserve.a.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value;
  double eps = 1.1920929e-7 * 100;  // doctest's default: float epsilon * 100
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  bool matches(double other) const {
    return std::fabs(other - value) <
           eps * (1.0 + std::fmax(std::fabs(other), std::fabs(value)));
  }
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator<=(double a, const Approx& b) { return a < b.value || b.matches(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value || b.matches(a); }

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};
inline bool msg_matches(const std::string& msg, const char* want) { return msg == want; }
inline bool msg_matches(const std::string& msg, const Contains& want) { return want.matches(msg); }

struct RequireFailed {};

struct Registry {
  struct Case { const char* name; void (*fn)(); };
  std::vector<Case> cases;
  int failed_checks = 0;
  bool current_failed = false;
  static Registry& get() { static Registry r; return r; }
};

inline void report(bool ok, const char* file, int line, const char* expr, bool require) {
  if (ok) return;
  Registry::get().failed_checks++;
  Registry::get().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

inline int run_all() {
  auto& reg = Registry::get();
  int cases_failed = 0;
  for (auto& c : reg.cases) {
    reg.current_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", c.name, e.what());
      reg.current_failed = true;
    }
    if (reg.current_failed) {
      ++cases_failed;
      std::fprintf(stderr, "  -> test case failed: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d\n",
              reg.cases.size(), reg.cases.size() - cases_failed, cases_failed);
  return cases_failed == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                         \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(            \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                           \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define CHECK_NOTHROW(...)                                                  \
  do {                                                                      \
    bool ok_ = true;                                                        \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }               \
    doctest::report(ok_, __FILE__, __LINE__, "NOTHROW " #__VA_ARGS__, false); \
  } while (0)
#define CHECK_THROWS(...)                                                   \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = true; }                \
    doctest::report(ok_, __FILE__, __LINE__, "THROWS " #__VA_ARGS__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                          \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
    doctest::report(ok_, __FILE__, __LINE__, "THROWS_AS " #expr, false);    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, want, ...)                               \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try { (void)(expr); } catch (const __VA_ARGS__& e_) {                   \
      ok_ = doctest::msg_matches(e_.what(), want);                          \
    } catch (...) {}                                                        \
    doctest::report(ok_, __FILE__, __LINE__, "THROWS_WITH_AS " #expr, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
