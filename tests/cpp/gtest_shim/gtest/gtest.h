// Minimal GoogleTest-compatible shim (GTest is not in this image): enough of
// TEST / EXPECT_* / ASSERT_* (with << messages) / EXPECT_THROW to compile the
// reference's own test sources unmodified against the drop-in headers
// (include/slsp) + libslsp_b200.so, and a main() that runs every registered
// test and prints one PASS/FAIL line per test (tests/cpp/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures_in_test() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

class Message {
 public:
  template <typename T>
  Message& operator<<(const T& v) {
    ss_ << v;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::ostringstream ss_;
};

class AssertHelper {
 public:
  AssertHelper(const char* file, int line, std::string text) : file_(file), line_(line), text_(std::move(text)) {}
  void operator=(const Message& m) const {  // NOLINT: gtest's idiom (return helper = Message() << ...)
    ++failures_in_test();
    std::fprintf(stderr, "  %s:%d: failure: %s %s\n", file_, line_, text_.c_str(), m.str().c_str());
  }

 private:
  const char* file_;
  int line_;
  std::string text_;
};

inline bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }
inline bool float_eq(float a, float b) {
  if (a == b) return true;
  const float d = std::fabs(a - b), m = std::fmax(std::fabs(a), std::fabs(b));
  return d <= m * 4 * 1.1920929e-7f;  // ~4 ULPs
}

inline int RunAllTests() {
  int failed = 0;
  for (const auto& t : registry()) {
    failures_in_test() = 0;
    bool threw = false;
    try {
      t.fn();
    } catch (const std::exception& e) {
      threw = true;
      std::fprintf(stderr, "  uncaught exception: %s\n", e.what());
    } catch (...) {
      threw = true;
      std::fprintf(stderr, "  uncaught non-std exception\n");
    }
    const bool ok = !threw && failures_in_test() == 0;
    std::printf("%s %s.%s\n", ok ? "PASS" : "FAIL", t.suite, t.name);
    failed += !ok;
  }
  std::printf("%zu tests, %d failed\n", registry().size(), failed);
  return failed ? 1 : 0;
}

}  // namespace testing

#define GT_AMBIGUOUS_ELSE_BLOCKER_ \
  switch (0)                       \
  case 0:                          \
  default:

#define GT_CHECK_(cond, text, on_fail)                                   \
  GT_AMBIGUOUS_ELSE_BLOCKER_                                             \
  if (cond)                                                              \
    ;                                                                    \
  else                                                                   \
    on_fail ::testing::AssertHelper(__FILE__, __LINE__, text) = ::testing::Message()

#define GT_NONFATAL_
#define GT_FATAL_ return

#define EXPECT_TRUE(c) GT_CHECK_(static_cast<bool>(c), "EXPECT_TRUE(" #c ")", GT_NONFATAL_)
#define EXPECT_FALSE(c) GT_CHECK_(!static_cast<bool>(c), "EXPECT_FALSE(" #c ")", GT_NONFATAL_)
#define ASSERT_TRUE(c) GT_CHECK_(static_cast<bool>(c), "ASSERT_TRUE(" #c ")", GT_FATAL_)
#define ASSERT_FALSE(c) GT_CHECK_(!static_cast<bool>(c), "ASSERT_FALSE(" #c ")", GT_FATAL_)
#define GT_CMP_(a, op, b, name, kind) GT_CHECK_(((a)op(b)), name "(" #a ", " #b ")", kind)
#define EXPECT_EQ(a, b) GT_CMP_(a, ==, b, "EXPECT_EQ", GT_NONFATAL_)
#define EXPECT_NE(a, b) GT_CMP_(a, !=, b, "EXPECT_NE", GT_NONFATAL_)
#define EXPECT_LT(a, b) GT_CMP_(a, <, b, "EXPECT_LT", GT_NONFATAL_)
#define EXPECT_LE(a, b) GT_CMP_(a, <=, b, "EXPECT_LE", GT_NONFATAL_)
#define EXPECT_GT(a, b) GT_CMP_(a, >, b, "EXPECT_GT", GT_NONFATAL_)
#define EXPECT_GE(a, b) GT_CMP_(a, >=, b, "EXPECT_GE", GT_NONFATAL_)
#define ASSERT_EQ(a, b) GT_CMP_(a, ==, b, "ASSERT_EQ", GT_FATAL_)
#define ASSERT_NE(a, b) GT_CMP_(a, !=, b, "ASSERT_NE", GT_FATAL_)
#define ASSERT_LT(a, b) GT_CMP_(a, <, b, "ASSERT_LT", GT_FATAL_)
#define ASSERT_LE(a, b) GT_CMP_(a, <=, b, "ASSERT_LE", GT_FATAL_)
#define ASSERT_GT(a, b) GT_CMP_(a, >, b, "ASSERT_GT", GT_FATAL_)
#define ASSERT_GE(a, b) GT_CMP_(a, >=, b, "ASSERT_GE", GT_FATAL_)
#define EXPECT_NEAR(a, b, t) GT_CHECK_(::testing::near((a), (b), (t)), "EXPECT_NEAR(" #a ", " #b ")", GT_NONFATAL_)
#define ASSERT_NEAR(a, b, t) GT_CHECK_(::testing::near((a), (b), (t)), "ASSERT_NEAR(" #a ", " #b ")", GT_FATAL_)
#define EXPECT_FLOAT_EQ(a, b) GT_CHECK_(::testing::float_eq((a), (b)), "EXPECT_FLOAT_EQ(" #a ", " #b ")", GT_NONFATAL_)
#define ASSERT_FLOAT_EQ(a, b) GT_CHECK_(::testing::float_eq((a), (b)), "ASSERT_FLOAT_EQ(" #a ", " #b ")", GT_FATAL_)
#define EXPECT_DOUBLE_EQ(a, b) GT_CHECK_(((a) == (b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")", GT_NONFATAL_)

#define GT_THROWS_(stmt, exc, kind)                                                      \
  GT_AMBIGUOUS_ELSE_BLOCKER_                                                              \
  if (int gt_caught_ = [&]() -> int {                                                     \
        try {                                                                             \
          stmt;                                                                           \
        } catch (const exc&) {                                                            \
          return 1;                                                                       \
        } catch (...) {                                                                   \
          return 2;                                                                       \
        }                                                                                 \
        return 0;                                                                         \
      }();                                                                                \
      gt_caught_ == 1)                                                                    \
    ;                                                                                     \
  else                                                                                    \
    kind ::testing::AssertHelper(__FILE__, __LINE__,                                      \
                                 gt_caught_ == 0 ? "EXPECT_THROW(" #stmt ", " #exc "): nothing thrown" \
                                                 : "EXPECT_THROW(" #stmt ", " #exc "): other exception") = \
        ::testing::Message()
#define EXPECT_THROW(stmt, exc) GT_THROWS_(stmt, exc, GT_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GT_THROWS_(stmt, exc, GT_FATAL_)
#define GT_NO_THROW_(stmt, kind)                                                                     \
  GT_AMBIGUOUS_ELSE_BLOCKER_                                                                         \
  if ([&]() -> bool {                                                                                \
        try {                                                                                        \
          stmt;                                                                                      \
        } catch (...) {                                                                              \
          return false;                                                                              \
        }                                                                                            \
        return true;                                                                                 \
      }())                                                                                           \
    ;                                                                                                \
  else                                                                                               \
    kind ::testing::AssertHelper(__FILE__, __LINE__, "EXPECT_NO_THROW(" #stmt ")") = ::testing::Message()
#define EXPECT_NO_THROW(stmt) GT_NO_THROW_(stmt, GT_NONFATAL_)
#define ASSERT_NO_THROW(stmt) GT_NO_THROW_(stmt, GT_FATAL_)

#define TEST(suite, name)                                                                   \
  static void gt_##suite##_##name();                                                        \
  static ::testing::Registrar gt_reg_##suite##_##name(#suite, #name, &gt_##suite##_##name); \
  static void gt_##suite##_##name()

#define FAIL() return ::testing::AssertHelper(__FILE__, __LINE__, "FAIL()") = ::testing::Message()
#define ADD_FAILURE() ::testing::AssertHelper(__FILE__, __LINE__, "ADD_FAILURE()") = ::testing::Message()
#define SUCCEED() static_cast<void>(0)
