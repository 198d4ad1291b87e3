// Minimal GoogleTest-compatible shim (GTest is not installed in this image). Supports what the
// reference's test files use: TEST, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,
// DOUBLE_EQ,THROW,NO_THROW}, EXPECT_STREQ, FAIL(), << messages, ::testing::Test::HasFailure().
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {
struct Registry {
  struct Case { std::string suite, name; std::function<void()> fn; };
  static std::vector<Case>& cases() { static std::vector<Case> c; return c; }
  static bool& failed() { static bool f = false; return f; }
};
struct Test {
  static bool HasFailure() { return Registry::failed(); }
};
struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    Registry::cases().push_back({s, n, std::move(f)});
  }
};
struct Msg {  // collects "<< ..." after a failed check, prints on destruction
  std::ostringstream os;
  bool active;
  explicit Msg(bool a, const char* file, int line, const std::string& what) : active(a) {
    if (active) {
      Registry::failed() = true;
      os << file << ":" << line << ": Failure: " << what;
    }
  }
  ~Msg() { if (active) std::cerr << os.str() << std::endl; }
  template <class T> Msg& operator<<(const T& v) { if (active) os << " " << v; return *this; }
};
struct AssertAbort {};
inline int RunAll() {
  int failed = 0;
  for (auto& c : Registry::cases()) {
    Registry::failed() = false;
    try { c.fn(); } catch (const AssertAbort&) {
    } catch (const std::exception& e) {
      Registry::failed() = true;
      std::cerr << "uncaught exception: " << e.what() << std::endl;
    }
    std::printf("[%s] %s.%s\n", Registry::failed() ? "  FAILED  " : "       OK ", c.suite.c_str(),
                c.name.c_str());
    failed += Registry::failed();
  }
  std::printf("%d tests, %d failed\n", (int)Registry::cases().size(), failed);
  return failed ? 1 : 0;
}
}  // namespace testing

#define TEST(S, N)                                                                  \
  static void S##_##N##_body();                                                     \
  static ::testing::Registrar S##_##N##_reg(#S, #N, S##_##N##_body);                \
  static void S##_##N##_body()

#define GT_CHECK_(cond, what, fatal)                                                \
  for (bool _gt_ok = (cond), _gt_once = true; _gt_once; _gt_once = false,          \
       (!_gt_ok && fatal) ? throw ::testing::AssertAbort() : (void)0)               \
  ::testing::Msg(!_gt_ok, __FILE__, __LINE__, what)

#define GT_BIN_(a, b, op, fatal) GT_CHECK_(((a)op(b)), #a " " #op " " #b, fatal)
#define EXPECT_EQ(a, b) GT_BIN_(a, b, ==, false)
#define EXPECT_NE(a, b) GT_BIN_(a, b, !=, false)
#define EXPECT_LT(a, b) GT_BIN_(a, b, <, false)
#define EXPECT_LE(a, b) GT_BIN_(a, b, <=, false)
#define EXPECT_GT(a, b) GT_BIN_(a, b, >, false)
#define EXPECT_GE(a, b) GT_BIN_(a, b, >=, false)
#define ASSERT_EQ(a, b) GT_BIN_(a, b, ==, true)
#define ASSERT_NE(a, b) GT_BIN_(a, b, !=, true)
#define ASSERT_LT(a, b) GT_BIN_(a, b, <, true)
#define ASSERT_LE(a, b) GT_BIN_(a, b, <=, true)
#define ASSERT_GT(a, b) GT_BIN_(a, b, >, true)
#define ASSERT_GE(a, b) GT_BIN_(a, b, >=, true)
#define EXPECT_TRUE(c) GT_CHECK_(bool(c), #c, false)
#define EXPECT_FALSE(c) GT_CHECK_(!bool(c), "!" #c, false)
#define ASSERT_TRUE(c) GT_CHECK_(bool(c), #c, true)
#define ASSERT_FALSE(c) GT_CHECK_(!bool(c), "!" #c, true)
#define EXPECT_NEAR(a, b, t) GT_CHECK_(std::fabs((a) - (b)) <= (t), "|" #a " - " #b "| <= " #t, false)
#define ASSERT_NEAR(a, b, t) GT_CHECK_(std::fabs((a) - (b)) <= (t), "|" #a " - " #b "| <= " #t, true)
#define EXPECT_DOUBLE_EQ(a, b)                                                       \
  GT_CHECK_(std::fabs((a) - (b)) <= 4 * 2.220446049250313e-16 * std::fmax(std::fabs(a), std::fabs(b)), \
            #a " ~= " #b, false)
#define ASSERT_DOUBLE_EQ(a, b)                                                       \
  GT_CHECK_(std::fabs((a) - (b)) <= 4 * 2.220446049250313e-16 * std::fmax(std::fabs(a), std::fabs(b)), \
            #a " ~= " #b, true)
#define EXPECT_STREQ(a, b) GT_CHECK_(std::strcmp((a), (b)) == 0, #a " == " #b, false)
#define GT_THROW_(stmt, exc, fatal)                                                  \
  GT_CHECK_(([&]() { try { stmt; } catch (const exc&) { return true; } catch (...) { return false; } \
             return false; }()), #stmt " throws " #exc, fatal)
#define EXPECT_THROW(stmt, exc) GT_THROW_(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) GT_THROW_(stmt, exc, true)
#define GT_NOTHROW_(stmt, fatal)                                                     \
  GT_CHECK_(([&]() { try { stmt; } catch (...) { return false; } return true; }()), #stmt " no throw", fatal)
#define EXPECT_NO_THROW(stmt) GT_NOTHROW_(stmt, false)
#define ASSERT_NO_THROW(stmt) GT_NOTHROW_(stmt, true)
#define FAIL() GT_CHECK_(false, "FAIL()", true)
