// Minimal test harness for the C++ drop-in tests (doctest is not vendored).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace chk {
inline int failures = 0;
inline std::vector<std::pair<std::string, std::function<void()>>>& registry() {
  static std::vector<std::pair<std::string, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
inline int run_all() {
  for (auto& [name, f] : registry()) {
    const int before = failures;
    try {
      f();
    } catch (const std::exception& e) {
      std::printf("  unexpected exception: %s\n", e.what());
      ++failures;
    }
    std::printf("%s %s\n", failures == before ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
}  // namespace chk

#define CHK_CAT2(a, b) a##b
#define CHK_CAT(a, b) CHK_CAT2(a, b)
#define TEST_CASE(name)                                              \
  static void CHK_CAT(test_fn_, __LINE__)();                         \
  static chk::Reg CHK_CAT(test_reg_, __LINE__)(name, CHK_CAT(test_fn_, __LINE__)); \
  static void CHK_CAT(test_fn_, __LINE__)()
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::printf("  %s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #cond);  \
      ++chk::failures;                                                         \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool ok_ = false;                                                          \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type&) {                                                    \
      ok_ = true;                                                              \
    } catch (...) {                                                            \
    }                                                                          \
    if (!ok_) {                                                                \
      std::printf("  %s:%d %s did not throw %s\n", __FILE__, __LINE__, #expr, #type); \
      ++chk::failures;                                                         \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, needle, type)                               \
  do {                                                                         \
    bool ok_ = false;                                                          \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type& e_) {                                                 \
      ok_ = std::string(e_.what()).find(needle) != std::string::npos;          \
    } catch (...) {                                                            \
    }                                                                          \
    if (!ok_) {                                                                \
      std::printf("  %s:%d %s did not throw %s with '%s'\n", __FILE__, __LINE__, #expr, #type, needle); \
      ++chk::failures;                                                         \
    }                                                                          \
  } while (0)
#define TEST_MAIN() \
  int main() { return chk::run_all(); }
