// Minimal doctest-compatible test harness (test infrastructure).  The reference's suites
// (/root/reference/proj/tests/*.cpp) are written against doctest, which the reference does
// not vendor; this header provides the subset they use so those suites can be compiled
// unchanged against the drop-in headers in include/colosim and run on the GPU:
// TEST_CASE, SUBCASE (re-run semantics), CHECK/REQUIRE[_MESSAGE], CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS (exact text or doctest::Contains), CHECK_NOTHROW, FAIL[_CHECK],
// CAPTURE, doctest::Approx.  Output: one line per failure and a summary; exit code != 0 on
// any failure.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <set>
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
  double eps = 1.1920929e-05;  // 100 * FLT_EPSILON, as doctest
};
inline bool operator==(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) <= a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
inline bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

struct Contains {
  explicit Contains(const char* s) : sub(s) {}
  std::string sub;
};

}  // namespace doctest

namespace doctest_shim {

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
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};

struct State {
  long checks = 0, failures = 0;
  const char* current = "";
  std::set<std::string> done_subcases;
  bool entered = false;
  std::string entered_name;
};
inline State& st() {
  static State s;
  return s;
}

inline void fail(const char* file, int line, const std::string& what) {
  ++st().failures;
  std::cerr << file << ":" << line << ": FAILED in \"" << st().current << "\": " << what << "\n";
}
inline void check(bool ok, const char* file, int line, const char* expr, bool require,
                  const std::string& msg = {}) {
  ++st().checks;
  if (ok) return;
  fail(file, line, std::string(expr) + (msg.empty() ? "" : "  -- " + msg));
  if (require) throw RequireFailed{};
}

template <class... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

struct Subcase {
  explicit Subcase(const char* name) {
    State& s = st();
    run = !s.entered && !s.done_subcases.count(name);
    if (run) {
      s.entered = true;
      s.entered_name = name;
    }
  }
  explicit operator bool() const { return run; }
  bool run;
};

inline bool matches(const std::string& what, const char* exact) { return what == exact; }
inline bool matches(const std::string& what, const doctest::Contains& c) {
  return what.find(c.sub) != std::string::npos;
}

inline int run_all() {
  State& s = st();
  int cases = 0;
  for (const Case& c : registry()) {
    ++cases;
    s.current = c.name;
    s.done_subcases.clear();
    for (;;) {
      s.entered = false;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        fail(c.file, c.line, "unexpected non-std exception");
      }
      if (!s.entered) break;
      s.done_subcases.insert(s.entered_name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | checks: %ld | failed: %ld | %s\n", cases, s.checks,
              s.failures, s.failures ? "FAILURE" : "SUCCESS");
  return s.failures ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                   \
  static void fn();                                                                 \
  static doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (doctest_shim::Subcase DOCTEST_SHIM_CAT(sc_, __LINE__){name})

#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_MESSAGE(cond, ...) \
  doctest_shim::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond, false, doctest_shim::cat(__VA_ARGS__))
#define REQUIRE_MESSAGE(cond, ...) \
  doctest_shim::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond, true, doctest_shim::cat(__VA_ARGS__))
#define FAIL_CHECK(msg)                                         \
  do {                                                          \
    std::ostringstream doctest_shim_os;                         \
    doctest_shim_os << msg;                                     \
    doctest_shim::fail(__FILE__, __LINE__, doctest_shim_os.str()); \
  } while (0)
#define FAIL(msg)                                               \
  do {                                                          \
    FAIL_CHECK(msg);                                            \
    throw doctest_shim::RequireFailed{};                        \
  } while (0)
#define CAPTURE(x) (void)0
#define CHECK_THROWS_AS(expr, T)                                                           \
  do {                                                                                     \
    bool doctest_shim_ok = false;                                                          \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const T&) {                                                                   \
      doctest_shim_ok = true;                                                              \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #T ")", false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, T)                                             \
  do {                                                                                     \
    bool doctest_shim_ok = false;                                                          \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const T& e) {                                                                 \
      doctest_shim_ok = doctest_shim::matches(e.what(), matcher);                          \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "THROWS_WITH_AS(" #expr ")", false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    bool doctest_shim_ok = true;                                                           \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      doctest_shim_ok = false;                                                             \
    }                                                                                      \
    doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "NOTHROW(" #expr ")", false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
