// gtest.h -- minimal GoogleTest-compatible harness (TEST INFRASTRUCTURE).
//
// GTest is not installed in this image (the reference vendors it under a
// git-ignored vendor/ dir).  This header implements the subset the
// reference's unit suites use -- TEST, TEST_P + INSTANTIATE_TEST_SUITE_P
// with ::testing::Values, EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,
// NEAR,DOUBLE_EQ,THROW,NO_THROW} with streamed messages -- so the
// reference's own test sources compile unchanged against either the
// reference library or the GPU shim (include/recsparse_gpu).
//
// Runner: every test in registration order; `--skip NAME` (repeatable,
// Suite.Name or Suite.Name/param index) excludes a test; prints one line per
// test and "SUMMARY passed=P failed=F skipped=S"; exit code 1 on a failure.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

struct AssertFail {};  // thrown by a failing ASSERT_* to leave the test body

namespace internal {

struct TestCase {
  std::string name;
  std::function<void()> body;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}
inline int reg(const std::string& name, std::function<void()> body) {
  registry().push_back({name, std::move(body)});
  return 0;
}

// Prints a value for failure messages where printable, else a placeholder.
template <typename T, typename = void>
struct Printable : std::false_type {};
template <typename T>
struct Printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <typename T>
std::string show(const T& v) {
  if constexpr (Printable<T>::value) {
    std::ostringstream os;
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

// Collects the streamed message of a failing check, reports it on destruction.
class Reporter {
 public:
  Reporter(bool ok, const char* file, int line, std::string what, bool fatal)
      : ok_(ok), fatal_(fatal), file_(file), line_(line), what_(std::move(what)) {}
  template <typename T>
  Reporter& operator<<(const T& v) {
    if (!ok_) msg_ << show(v);
    return *this;
  }
  ~Reporter() noexcept(false) {
    if (ok_) return;
    current_failed() = true;
    std::cout << "  " << file_ << ":" << line_ << ": " << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cout << " -- " << m;
    std::cout << std::endl;
    if (fatal_) throw AssertFail{};
  }

 private:
  bool ok_, fatal_;
  const char* file_;
  int line_;
  std::string what_;
  std::ostringstream msg_;
};

template <typename A, typename B>
std::string cmp_text(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  return std::string("expected ") + ea + " " + op + " " + eb + " (" + show(a) + " vs " + show(b) + ")";
}

inline bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }
// DOUBLE_EQ: within 4 ulps (GoogleTest's AlmostEquals)
inline bool almost_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if (ia < 0) ia = INT64_MIN - ia;
  if (ib < 0) ib = INT64_MIN - ib;
  const uint64_t d = ia > ib ? (uint64_t)(ia - ib) : (uint64_t)(ib - ia);
  return d <= 4;
}

}  // namespace internal

class Test {
 public:
  virtual ~Test() = default;
  virtual void TestBody() = 0;
};

template <typename T>
class TestWithParam : public Test {
 public:
  using ParamType = T;
  const T& GetParam() const { return *param_; }
  static void set_param(const T* p) { param_ = p; }

 private:
  static inline const T* param_ = nullptr;
};

template <typename... Ts>
auto Values(Ts... vs) {
  using T = std::common_type_t<Ts...>;
  return std::vector<T>{static_cast<T>(vs)...};
}

// TEST_P bodies register here per suite; INSTANTIATE_TEST_SUITE_P expands them
template <typename Suite>
struct ParamRegistry {
  static std::vector<std::pair<std::string, std::function<void()>>>& bodies() {
    static std::vector<std::pair<std::string, std::function<void()>>> b;
    return b;
  }
};

inline int RunAllTests(int argc, char** argv) {
  std::set<std::string> skip;
  for (int i = 1; i + 1 < argc; ++i)
    if (std::string(argv[i]) == "--skip") skip.insert(argv[++i]);
  int passed = 0, failed = 0, skipped = 0;
  for (auto& t : internal::registry()) {
    if (skip.count(t.name)) {
      ++skipped;
      std::cout << "[ SKIP ] " << t.name << std::endl;
      continue;
    }
    internal::current_failed() = false;
    try {
      t.body();
    } catch (const AssertFail&) {
    } catch (const std::exception& e) {
      internal::current_failed() = true;
      std::cout << "  uncaught exception: " << e.what() << std::endl;
    }
    if (internal::current_failed()) {
      ++failed;
      std::cout << "[ FAIL ] " << t.name << std::endl;
    } else {
      ++passed;
      std::cout << "[  OK  ] " << t.name << std::endl;
    }
  }
  std::cout << "SUMMARY passed=" << passed << " failed=" << failed << " skipped=" << skipped << std::endl;
  return failed ? 1 : 0;
}

}  // namespace testing

#define GTS_CAT2(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT2(a, b)

#define TEST(suite, name)                                                                     \
  struct suite##_##name##_Test : ::testing::Test {                                            \
    void TestBody() override;                                                                 \
  };                                                                                          \
  static int GTS_CAT(gts_reg_, __LINE__) = ::testing::internal::reg(#suite "." #name, [] {    \
    suite##_##name##_Test t;                                                                  \
    t.TestBody();                                                                             \
  });                                                                                         \
  void suite##_##name##_Test::TestBody()

#define TEST_P(suite, name)                                                                   \
  struct suite##_##name##_Test : suite {                                                      \
    void TestBody() override;                                                                 \
  };                                                                                          \
  static int GTS_CAT(gts_preg_, __LINE__) = [] {                                              \
    ::testing::ParamRegistry<suite>::bodies().push_back({#suite "." #name, [] {               \
                                                           suite##_##name##_Test t;           \
                                                           t.TestBody();                      \
                                                         }});                                 \
    return 0;                                                                                 \
  }();                                                                                        \
  void suite##_##name##_Test::TestBody()

#define INSTANTIATE_TEST_SUITE_P(prefix, suite, values)                                       \
  static int GTS_CAT(gts_inst_, __LINE__) = [] {                                              \
    static const auto vals = values;                                                          \
    for (const auto& b : ::testing::ParamRegistry<suite>::bodies())                           \
      for (size_t i = 0; i < vals.size(); ++i)                                                \
        ::testing::internal::reg(std::string(#prefix "/") + b.first + "/" + std::to_string(i), \
                                 [b, i] {                                                     \
                                   suite::set_param(&vals[i]);                                \
                                   b.second();                                                \
                                 });                                                          \
    return 0;                                                                                 \
  }()

#define GTS_CHECK(cond, text, fatal) ::testing::internal::Reporter((cond), __FILE__, __LINE__, (text), (fatal))
#define GTS_BIN(a, b, op, opname, fatal)                                                       \
  for (bool gts_once = true; gts_once; gts_once = false)                                      \
    for (const auto& gts_a = (a); gts_once; gts_once = false)                                  \
      for (const auto& gts_b = (b); gts_once; gts_once = false)                                \
  GTS_CHECK(gts_a op gts_b, ::testing::internal::cmp_text(opname, #a, #b, gts_a, gts_b), fatal)

#define EXPECT_EQ(a, b) GTS_BIN(a, b, ==, "==", false)
#define EXPECT_NE(a, b) GTS_BIN(a, b, !=, "!=", false)
#define EXPECT_LT(a, b) GTS_BIN(a, b, <, "<", false)
#define EXPECT_LE(a, b) GTS_BIN(a, b, <=, "<=", false)
#define EXPECT_GT(a, b) GTS_BIN(a, b, >, ">", false)
#define EXPECT_GE(a, b) GTS_BIN(a, b, >=, ">=", false)
#define ASSERT_EQ(a, b) GTS_BIN(a, b, ==, "==", true)
#define ASSERT_NE(a, b) GTS_BIN(a, b, !=, "!=", true)
#define ASSERT_LT(a, b) GTS_BIN(a, b, <, "<", true)
#define ASSERT_LE(a, b) GTS_BIN(a, b, <=, "<=", true)
#define ASSERT_GT(a, b) GTS_BIN(a, b, >, ">", true)
#define ASSERT_GE(a, b) GTS_BIN(a, b, >=, ">=", true)
#define EXPECT_TRUE(c) GTS_CHECK(static_cast<bool>(c), "expected true: " #c, false)
#define EXPECT_FALSE(c) GTS_CHECK(!static_cast<bool>(c), "expected false: " #c, false)
#define ASSERT_TRUE(c) GTS_CHECK(static_cast<bool>(c), "expected true: " #c, true)
#define ASSERT_FALSE(c) GTS_CHECK(!static_cast<bool>(c), "expected false: " #c, true)
#define EXPECT_NEAR(a, b, tol) \
  GTS_CHECK(::testing::internal::near((a), (b), (tol)), "expected " #a " near " #b " within " #tol, false)
#define ASSERT_NEAR(a, b, tol) \
  GTS_CHECK(::testing::internal::near((a), (b), (tol)), "expected " #a " near " #b " within " #tol, true)
#define EXPECT_DOUBLE_EQ(a, b) \
  GTS_CHECK(::testing::internal::almost_eq((a), (b)), "expected " #a " == " #b " (4 ulps)", false)
#define ASSERT_DOUBLE_EQ(a, b) \
  GTS_CHECK(::testing::internal::almost_eq((a), (b)), "expected " #a " == " #b " (4 ulps)", true)

#define GTS_THROWS(stmt, exc, fatal)                                                          \
  for (bool gts_once = true; gts_once; gts_once = false)                                      \
    for (int gts_r = [&]() -> int {                                                           \
           try {                                                                              \
             stmt;                                                                            \
           } catch (const exc&) {                                                             \
             return 1;                                                                        \
           } catch (...) {                                                                    \
             return 2;                                                                        \
           }                                                                                  \
           return 0;                                                                          \
         }();                                                                                 \
         gts_once; gts_once = false)                                                          \
  GTS_CHECK(gts_r == 1, gts_r == 0 ? "expected " #exc " from " #stmt ", nothing thrown"       \
                                   : "expected " #exc " from " #stmt ", another exception",  \
            fatal)
#define EXPECT_THROW(stmt, exc) GTS_THROWS(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) GTS_THROWS(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                                                 \
  for (bool gts_once = true; gts_once; gts_once = false)                                      \
    for (bool gts_ok = [&]() -> bool {                                                        \
           try {                                                                              \
             stmt;                                                                            \
           } catch (...) {                                                                    \
             return false;                                                                    \
           }                                                                                  \
           return true;                                                                       \
         }();                                                                                 \
         gts_once; gts_once = false)                                                          \
  GTS_CHECK(gts_ok, "expected no exception from " #stmt, false)
