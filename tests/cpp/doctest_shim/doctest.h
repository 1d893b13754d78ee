// doctest.h — TEST INFRASTRUCTURE: a minimal doctest-compatible harness so the
// reference's own unit tests (/root/reference/proj/tests/test_*.cpp) compile
// UNMODIFIED against this repo's drop-in headers (include/intergrams/) and
// run against libintergrams_b200.so.  doctest itself is not
// in the image; this implements only the subset those files use:
// TEST_CASE, SUBCASE (doctest's re-run-per-leaf semantics), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest_shim {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

// Per-test state: checks, failures, and the subcase traversal.
struct State {
  long checks = 0, failures = 0;
  const char* test = "";
  std::set<std::vector<int>> done;   // fully explored subcase paths
  std::vector<int> path;             // subcases entered in this run
  std::vector<bool> entered;         // entered[d]: a subcase at depth d entered in this parent
  bool new_entry = false;
};

inline State& st() {
  static State s;
  return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = st();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\"\n", file, line, kind, expr,
                 s.test);
  }
}

struct Subcase {
  bool on = false;
  std::vector<int> me;
  Subcase(const char* /*name*/, int line) {
    State& s = st();
    const size_t d = s.path.size();
    if (s.entered.size() <= d + 1) s.entered.resize(d + 2, false);
    me = s.path;
    me.push_back(line);
    if (s.entered[d] || s.done.count(me)) return;
    on = true;
    s.entered[d] = true;
    s.entered[d + 1] = false;
    s.new_entry = true;
    s.path.push_back(line);
  }
  ~Subcase() {
    if (!on) return;
    State& s = st();
    const size_t d = s.path.size();  // depth of my children
    // no child entered on this visit: every child (if any) is explored
    if (s.entered.size() <= d || !s.entered[d]) s.done.insert(me);
    s.path.pop_back();
  }
  explicit operator bool() const { return on; }
};

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;  // substring of the test name
  const char* exact = nullptr;   // the whole test name
  std::set<std::string> excluded;  // -ntc=<whole name>: skip
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-tc=", 4)) filter = argv[i] + 4;
    if (!std::strncmp(argv[i], "-tce=", 5)) exact = argv[i] + 5;
    if (!std::strncmp(argv[i], "-ntc=", 5)) excluded.insert(argv[i] + 5);
    if (!std::strcmp(argv[i], "-ltc")) {  // list test cases: "file\tname"
      for (const TestCase& tc : registry()) std::printf("%s\t%s\n", tc.file, tc.name);
      return 0;
    }
  }
  long cases = 0, failed_cases = 0, checks = 0, failures = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    if (exact && std::strcmp(tc.name, exact)) continue;
    if (excluded.count(tc.name)) continue;
    ++cases;
    State& s = st();
    s = State{};
    s.test = tc.name;
    bool case_failed = false;
    for (int run = 0; run < 100000; ++run) {
      s.path.clear();
      s.entered.assign(1, false);
      s.new_entry = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
        case_failed = true;
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: TEST_CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                     e.what());
        ++s.failures;
        case_failed = true;
      }
      if (!s.new_entry || case_failed) break;
    }
    checks += s.checks;
    failures += s.failures;
    if (s.failures || case_failed) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed\n", cases,
              cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", checks,
              checks - failures, failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                           \
  static void fn();                                                                         \
  static ::doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const ::doctest_shim::Subcase DOCTEST_SHIM_CAT(doctest_shim_sc_, __LINE__){name, __LINE__})

#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                          \
    ::doctest_shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_shim_ok) throw ::doctest_shim::RequireFailed{};                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_shim_ok = false;                                                          \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_shim_ok = true;                                                              \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest_shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,    \
                           __FILE__, __LINE__);                                            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest_shim::run_all(argc, argv); }
#endif
