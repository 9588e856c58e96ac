// doctest.h -- minimal stand-in for the doctest single header, covering only
// the macros the reference's unit suites use (TEST_CASE, CHECK, REQUIRE,
// CHECK_NOTHROW, FAIL, doctest::Approx(x).epsilon(e),
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN).  The reference vendors doctest under
// proj/vendor/, which is absent from /root/reference (proj/.gitignore:2), so
// its suites are compiled against this shim.  TEST
// INFRASTRUCTURE: used only to build the reference's own test programs
// against include/monoalign/ + libmonoalign_b200.so (oracle/Makefile dropin).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1e-5;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
};
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.v) <= b.eps * (1 + std::max(std::fabs(a), std::fabs(b.v)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }
struct Reg {
  const char* name;
  const char* file;
  void (*fn)();
};
inline std::vector<Reg>& regs() {
  static std::vector<Reg> r;
  return r;
}
inline int& fails() {
  static int f = 0;
  return f;
}
struct Adder {
  Adder(const char* n, const char* f, void (*fn)()) { regs().push_back({n, f, fn}); }
};
struct RequireFail {};
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define DT_TC(fn, name)                                                  \
  static void fn();                                                      \
  static doctest::Adder DT_CAT(fn, _reg)(name, __FILE__, fn);            \
  static void fn()
#define TEST_CASE(name) DT_TC(DT_CAT(dt_tc_, __COUNTER__), name)
#define CHECK(...)                                                                      \
  do {                                                                                  \
    if (!(__VA_ARGS__)) {                                                               \
      ++doctest::fails();                                                               \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
    }                                                                                   \
  } while (0)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    if (!(__VA_ARGS__)) {                                                                 \
      ++doctest::fails();                                                                 \
      std::fprintf(stderr, "%s:%d REQUIRE failed: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      throw doctest::RequireFail{};                                                       \
    }                                                                                     \
  } while (0)
#define CHECK_NOTHROW(...)                                                  \
  do {                                                                      \
    try {                                                                   \
      __VA_ARGS__;                                                          \
    } catch (...) {                                                         \
      ++doctest::fails();                                                   \
      std::fprintf(stderr, "%s:%d unexpected throw\n", __FILE__, __LINE__); \
    }                                                                       \
  } while (0)
#define FAIL(msg)                                                           \
  do {                                                                      \
    ++doctest::fails();                                                     \
    std::fprintf(stderr, "%s:%d FAIL %s\n", __FILE__, __LINE__, msg);       \
    throw doctest::RequireFail{};                                           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  // optional argument: run only the cases whose file name contains it
  const char* only = argc > 1 ? argv[1] : nullptr;
  int n = 0;
  for (auto& r : doctest::regs()) {
    if (only && !std::strstr(r.file, only)) continue;
    ++n;
    const int before = doctest::fails();
    try {
      r.fn();
    } catch (doctest::RequireFail&) {
    } catch (std::exception& e) {
      ++doctest::fails();
      std::fprintf(stderr, "%s threw %s\n", r.name, e.what());
    }
    if (doctest::fails() != before) std::fprintf(stderr, "  in test case \"%s\"\n", r.name);
  }
  std::printf("test cases: %d, failed checks: %d\n", n, doctest::fails());
  return doctest::fails() ? 1 : 0;
}
#endif
