// gtest.h -- minimal GoogleTest-compatible shim (GTest is not installed in
// this image). Enough of the API to compile the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) unchanged against the B200 drop-in
// headers: TEST, TEST_F (fixtures deriving ::testing::Test with SetUp /
// TearDown), EXPECT_/ASSERT_ {EQ,NE,LT,LE,GT,GE,NEAR,TRUE,FALSE,THROW,
// NO_THROW}, streaming of extra failure messages, and a main() that runs
// every registered test, honours --gtest_filter=-A.B:C.D (negative filter
// only) and prints one "[  PASSED  ]"/"[  FAILED  ]" line per test.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

// Fixture base: TEST_F(F, name) derives from F, runs SetUp, the body, then
// TearDown (also when the body throws).
class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  void Run() {
    SetUp();
    try {
      TestBody();
    } catch (...) {
      TearDown();
      throw;
    }
    TearDown();
  }
};

struct TestInfo {
  std::string suite, name;
  std::function<void()> fn;
};

inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}
struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> fn) {
    registry().push_back({s, n, std::move(fn)});
  }
};

// Collects an optional streamed message; reports on destruction.
class Failure {
 public:
  Failure(const char* file, int line, std::string what, bool fatal)
      : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  template <class T>
  Failure& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }
  ~Failure() noexcept(false) {
    current_failed() = true;
    std::cerr << file_ << ":" << line_ << ": Failure\n" << what_;
    const std::string m = msg_.str();
    if (!m.empty()) std::cerr << "\n" << m;
    std::cerr << std::endl;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream msg_;
};

struct NullStream {
  template <class T>
  NullStream& operator<<(const T&) {
    return *this;
  }
};

template <class T>
std::string repr(const T& v) {
  std::ostringstream o;
  if constexpr (requires(std::ostream& s, const T& x) { s << x; }) {
    o << v;
  } else {
    o << "<value>";
  }
  return o.str();
}

template <class A, class B>
std::string cmp_msg(const char* ea, const char* eb, const char* op, const A& a, const B& b) {
  std::ostringstream o;
  o << "Expected: (" << ea << ") " << op << " (" << eb << "), actual: " << repr(a) << " vs "
    << repr(b);
  return o.str();
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> skip;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    const std::string key = "--gtest_filter=-";
    if (a.rfind(key, 0) == 0) {
      std::string rest = a.substr(key.size());
      size_t p = 0;
      while (p <= rest.size()) {
        size_t q = rest.find(':', p);
        if (q == std::string::npos) q = rest.size();
        if (q > p) skip.push_back(rest.substr(p, q - p));
        p = q + 1;
      }
    }
  }
  int failed = 0, ran = 0;
  for (auto& t : registry()) {
    const std::string full = t.suite + "." + t.name;
    bool skipped = false;
    for (auto& s : skip)
      if (s == full) skipped = true;
    if (skipped) {
      std::cout << "[ SKIPPED  ] " << full << std::endl;
      continue;
    }
    current_failed() = false;
    ++ran;
    try {
      t.fn();
    } catch (const std::exception& e) {
      current_failed() = true;
      std::cerr << "uncaught exception: " << e.what() << std::endl;
    } catch (int) {
      // fatal assertion already reported
    } catch (...) {
      current_failed() = true;
      std::cerr << "uncaught non-std exception" << std::endl;
    }
    if (current_failed()) ++failed;
    std::cout << (current_failed() ? "[  FAILED  ] " : "[  PASSED  ] ") << full << std::endl;
  }
  std::cout << "[==========] " << ran << " tests ran, " << failed << " failed" << std::endl;
  return failed ? 1 : 0;
}

}  // namespace testing

#define GTEST_SHIM_CAT2(a, b) a##b
#define GTEST_SHIM_CAT(a, b) GTEST_SHIM_CAT2(a, b)
#define TEST(suite, name)                                                            \
  static void GTEST_SHIM_CAT(gtest_fn_##suite##_, name)();                           \
  static ::testing::Registrar GTEST_SHIM_CAT(gtest_reg_##suite##_, name)(            \
      #suite, #name, &GTEST_SHIM_CAT(gtest_fn_##suite##_, name));                    \
  static void GTEST_SHIM_CAT(gtest_fn_##suite##_, name)()

#define TEST_F(fixture, name)                                                        \
  namespace {                                                                        \
  struct GTEST_SHIM_CAT(fixture##_, name) : public fixture {                         \
    void TestBody() override;                                                        \
  };                                                                                 \
  ::testing::Registrar GTEST_SHIM_CAT(gtest_reg_##fixture##_, name)(                 \
      #fixture, #name, [] {                                                          \
        GTEST_SHIM_CAT(fixture##_, name) t;                                          \
        t.Run();                                                                     \
      });                                                                            \
  }                                                                                  \
  void GTEST_SHIM_CAT(fixture##_, name)::TestBody()

// non-fatal: report and continue; fatal: report and leave the test body
#define GTEST_SHIM_CHECK(cond, what, fatal)                                          \
  if (cond) {                                                                        \
  } else                                                                             \
    for (bool gtest_once_ = true; gtest_once_; gtest_once_ = false,                  \
              (fatal ? throw 0 : (void)0))                                           \
  ::testing::Failure(__FILE__, __LINE__, what, fatal)

#define GTEST_SHIM_CMP(a, b, op, fatal)                                              \
  GTEST_SHIM_CHECK(((a)op(b)), ::testing::cmp_msg(#a, #b, #op, (a), (b)), fatal)

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP(a, b, ==, false)
#define EXPECT_NE(a, b) GTEST_SHIM_CMP(a, b, !=, false)
#define EXPECT_LT(a, b) GTEST_SHIM_CMP(a, b, <, false)
#define EXPECT_LE(a, b) GTEST_SHIM_CMP(a, b, <=, false)
#define EXPECT_GT(a, b) GTEST_SHIM_CMP(a, b, >, false)
#define EXPECT_GE(a, b) GTEST_SHIM_CMP(a, b, >=, false)
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP(a, b, ==, true)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP(a, b, !=, true)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP(a, b, <, true)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP(a, b, <=, true)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP(a, b, >, true)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP(a, b, >=, true)
#define EXPECT_TRUE(c) GTEST_SHIM_CHECK(bool(c), "Expected true: " #c, false)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK(!bool(c), "Expected false: " #c, false)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK(bool(c), "Expected true: " #c, true)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK(!bool(c), "Expected false: " #c, true)
#define EXPECT_NEAR(a, b, tol)                                                       \
  GTEST_SHIM_CHECK(std::fabs(double(a) - double(b)) <= double(tol),                  \
                   ::testing::cmp_msg(#a, #b, "near", (a), (b)) + " tol " #tol, false)
#define ASSERT_NEAR(a, b, tol)                                                       \
  GTEST_SHIM_CHECK(std::fabs(double(a) - double(b)) <= double(tol),                  \
                   ::testing::cmp_msg(#a, #b, "near", (a), (b)) + " tol " #tol, true)
#define GTEST_SHIM_THROWS(stmt, exc, fatal)                                          \
  GTEST_SHIM_CHECK(([&]() -> bool {                                                  \
                     try {                                                           \
                       stmt;                                                         \
                     } catch (const exc&) {                                          \
                       return true;                                                  \
                     } catch (...) {                                                 \
                       return false;                                                 \
                     }                                                               \
                     return false;                                                   \
                   }()),                                                             \
                   "Expected: " #stmt " throws " #exc, fatal)
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROWS(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROWS(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                                        \
  GTEST_SHIM_CHECK(([&]() -> bool {                                                  \
                     try {                                                           \
                       stmt;                                                         \
                     } catch (...) {                                                 \
                       return false;                                                 \
                     }                                                               \
                     return true;                                                    \
                   }()),                                                             \
                   "Expected: " #stmt " does not throw", false)
#define ASSERT_NO_THROW(stmt) EXPECT_NO_THROW(stmt)
#define SUCCEED() ::testing::NullStream()
#define FAIL() ::testing::Failure(__FILE__, __LINE__, "Failed", true)
#define ADD_FAILURE() ::testing::Failure(__FILE__, __LINE__, "Failed", false)
#define GTEST_SKIP() return

int main(int argc, char** argv) { return ::testing::run_all(argc, argv); }
