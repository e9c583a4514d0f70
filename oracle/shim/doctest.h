// ORACLE TEST INFRASTRUCTURE ONLY.
//
// Minimal doctest-compatible harness so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) compile and run unchanged against
// the Boost shim: TEST_CASE, one level of SUBCASE, CHECK, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL.  doctest itself was
// vendored under the reference's absent vendor/ directory
// (proj/README.md:41-43).  Semantics follow doctest: a SUBCASE-bearing test
// case is re-run once per subcase, entering exactly one subcase per run.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

namespace doctest_shim {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  long checks = 0, failures = 0;
  int subcase_target = 0;   // which subcase (by encounter order) to enter
  int subcase_seen = 0;     // subcases encountered in the current run
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  state().current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}

struct SubcaseGuard {
  bool enter;
  explicit SubcaseGuard(const char*) {
    State& s = state();
    enter = s.subcase_seen == s.subcase_target;
    ++s.subcase_seen;
  }
  explicit operator bool() const { return enter; }
};

inline int run_all(const char* filter) {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    State& s = state();
    s.current_failed = false;
    int target = 0;
    while (true) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.current_failed = true;
        std::fprintf(stderr, "%s:%d: exception in '%s': %s\n", tc.file, tc.line, tc.name, e.what());
      }
      if (s.subcase_seen <= target + 1) break;  // no more subcases to enter
      ++target;
    }
    std::printf("[%s] %s\n", s.current_failed ? "FAIL" : " ok ", tc.name);
    if (s.current_failed) ++failed_cases;
  }
  std::printf("test cases failed: %d; assertions: %ld checked, %ld failed\n", failed_cases,
              state().checks, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(name, fn)                                                   \
  static void fn();                                                                 \
  static doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(name, DOCTEST_SHIM_CAT(doctest_shim_tc_, __LINE__))
#define SUBCASE(name) if (doctest_shim::SubcaseGuard DOCTEST_SHIM_CAT(sg_, __LINE__){name})

#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(...) doctest_shim::report(false, "FAIL", __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                               \
  do {                                                                  \
    bool threw_ = false;                                                \
    try { (void)(__VA_ARGS__); } catch (...) { threw_ = true; }         \
    doctest_shim::report(threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                      \
  do {                                                                  \
    bool ok_ = false;                                                   \
    try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
    doctest_shim::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                              \
  do {                                                                  \
    bool ok_ = true;                                                    \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }           \
    doctest_shim::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--tc=", 0) == 0) filter = argv[i] + 5;
  }
  return doctest_shim::run_all(filter);
}
#endif
