// Minimal GoogleTest-compatible macros (GTest is not in the image), enough to
// run reference-style tests against the façade.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mt {
struct Case {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* s, const char* n, std::function<void()> f) { registry().push_back({s, n, f}); }
};
inline int& failures() {
  static int f = 0;
  return f;
}
struct Abort {};
inline void fail(const char* file, int line, const std::string& what, bool fatal) {
  std::fprintf(stderr, "%s:%d: FAILED %s\n", file, line, what.c_str());
  ++failures();
  if (fatal) throw Abort{};
}
inline int run_all() {
  int bad = 0;
  for (auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (Abort&) {
    } catch (std::exception& e) {
      std::fprintf(stderr, "uncaught exception: %s\n", e.what());
      ++failures();
    }
    const bool ok = failures() == before;
    bad += !ok;
    std::printf("[%s] %s.%s\n", ok ? "PASS" : "FAIL", c.suite, c.name);
  }
  std::printf("%d tests, %d failed\n", (int)registry().size(), bad);
  return bad ? 1 : 0;
}
}  // namespace mt

#define TEST(S, N)                                                   \
  static void S##_##N##_body();                                      \
  static mt::Reg S##_##N##_reg(#S, #N, S##_##N##_body);              \
  static void S##_##N##_body()
#define MT_CHECK(cond, what, fatal) \
  do {                              \
    if (!(cond)) mt::fail(__FILE__, __LINE__, what, fatal); \
  } while (0)
#define EXPECT_TRUE(c) MT_CHECK((c), #c, false)
#define ASSERT_TRUE(c) MT_CHECK((c), #c, true)
#define EXPECT_EQ(a, b) MT_CHECK((a) == (b), #a " == " #b, false)
#define ASSERT_EQ(a, b) MT_CHECK((a) == (b), #a " == " #b, true)
#define EXPECT_NE(a, b) MT_CHECK((a) != (b), #a " != " #b, false)
#define EXPECT_LT(a, b) MT_CHECK((a) < (b), #a " < " #b, false)
#define EXPECT_DOUBLE_EQ(a, b) \
  MT_CHECK(std::fabs((double)(a) - (double)(b)) <= 4 * 2.220446049250313e-16 * std::fabs((double)(b)), #a " ~= " #b, false)
#define EXPECT_NEAR(a, b, t) MT_CHECK(std::fabs((double)(a) - (double)(b)) <= (t), #a " near " #b, false)
#define EXPECT_THROW(stmt, ex)              \
  do {                                      \
    bool thrown_ = false;                   \
    try {                                   \
      stmt;                                 \
    } catch (const ex&) {                   \
      thrown_ = true;                       \
    } catch (...) {                         \
    }                                       \
    MT_CHECK(thrown_, #stmt " throws " #ex, false); \
  } while (0)
