// Minimal test registry for the C++ drop-in suite (the reference's doctest is not vendored).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace chk {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
inline int run_all() {
  int failed_cases = 0;
  for (auto& c : cases()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::printf("  exception: %s\n", e.what());
      ++failures();
    }
    const bool ok = failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%zu cases, %d failed\n", cases().size(), failed_cases);
  return failed_cases ? 1 : 0;
}
}  // namespace chk

#define CHK_CAT2(a, b) a##b
#define CHK_CAT(a, b) CHK_CAT2(a, b)
#define TEST_CASE(name)                                                  \
  static void CHK_CAT(chk_fn_, __LINE__)();                              \
  static chk::Reg CHK_CAT(chk_reg_, __LINE__)(name, CHK_CAT(chk_fn_, __LINE__)); \
  static void CHK_CAT(chk_fn_, __LINE__)()
#define CHECK(cond)                                                             \
  do {                                                                          \
    if (!(cond)) {                                                              \
      std::printf("  %s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #cond);     \
      ++chk::failures();                                                        \
    }                                                                           \
  } while (0)
#define CHECK_NEAR(a, b, tol) CHECK(std::abs(double(a) - double(b)) <= (tol))
#define CHECK_THROWS(expr)                  \
  do {                                      \
    bool thrown_ = false;                   \
    try {                                   \
      (void)(expr);                         \
    } catch (const std::exception&) {       \
      thrown_ = true;                       \
    }                                       \
    CHECK(thrown_);                         \
  } while (0)
