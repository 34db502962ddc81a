// tests/cpp/doctest.h — a minimal stand-in for the doctest single-header framework, which the
// reference's unit suites include (/root/reference/proj/tests/test_*.cpp) but whose copy is not
// in the reference tree (vendor/ is git-ignored there). It covers exactly what those suites use:
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN, TEST_CASE(name), CHECK(expr) and REQUIRE(expr). A CHECK
// failure is counted and reported; a REQUIRE failure or an exception ends the test case. main()
// runs every registered case and exits non-zero when any check failed.
//
// Test infrastructure only: it lets oracle/Makefile compile the reference's own suites against
// the drop-in headers (include/mprof/*.hpp) and libmprof_gpu.so (tests/test_reference_suites.py).
#pragma once

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace mini_doctest {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& cases() {
  static std::vector<Case> all;
  return all;
}

struct Stats {
  long checks = 0;
  long failed_checks = 0;
  int failed_cases = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct Register {
  Register(const char* name, void (*fn)(), const char* file, int line) {
    cases().push_back(Case{name, fn, file, line});
  }
};

struct RequireAbort {};

inline void assert_that(bool ok, const char* what, const char* expr, const char* file, int line,
                        bool fatal) {
  Stats& s = stats();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, what, expr);
  if (fatal) throw RequireAbort{};
}

inline int run_all() {
  Stats& s = stats();
  for (const Case& c : cases()) {
    s.case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
      s.case_failed = true;
    } catch (...) {
      std::printf("%s:%d: ERROR: test case \"%s\" threw a non-standard exception\n", c.file, c.line,
                  c.name);
      s.case_failed = true;
    }
    if (s.case_failed) {
      ++s.failed_cases;
      std::printf("FAILED test case: %s\n", c.name);
    }
  }
  std::printf("[mini_doctest] test cases: %zu | %zu passed | %d failed\n", cases().size(),
              cases().size() - static_cast<std::size_t>(s.failed_cases), s.failed_cases);
  std::printf("[mini_doctest] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failed_checks, s.failed_checks);
  return s.failed_cases == 0 ? 0 : 1;
}

}  // namespace mini_doctest

#define MINI_DOCTEST_CAT2(a, b) a##b
#define MINI_DOCTEST_CAT(a, b) MINI_DOCTEST_CAT2(a, b)
#define MINI_DOCTEST_CASE(fn, reg, name)                                                   \
  static void fn();                                                                        \
  static const ::mini_doctest::Register reg(name, &fn, __FILE__, __LINE__);                \
  static void fn()
#define TEST_CASE(name)                                                                    \
  MINI_DOCTEST_CASE(MINI_DOCTEST_CAT(mini_doctest_case_, __LINE__),                        \
                    MINI_DOCTEST_CAT(mini_doctest_reg_, __LINE__), name)
#define CHECK(...) \
  ::mini_doctest::assert_that(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
  ::mini_doctest::assert_that(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::mini_doctest::run_all(); }
#endif
