// Minimal GoogleTest-compatible shim (GTest is not installed in this image).
//
// Enough of the GTest surface to compile the reference's own unit suites
// (/root/reference/proj/tests/*_test.cpp) UNMODIFIED against the drop-in
// (include/zen_b200/compat.hpp via tests/cpp/zen_shim): TEST, EXPECT_/ASSERT_
// {EQ,NE,LT,LE,GT,GE,TRUE,FALSE,DOUBLE_EQ,FLOAT_EQ,NEAR,THROW,NO_THROW} and a
// main that runs every registered test and prints a GTest-style summary.
// Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace gtest_shim {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures_in_test() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

template <typename T, typename = void>
struct printable : std::false_type {};
template <typename T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
std::string show(const T& v) {
  if constexpr (printable<T>::value) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

// Message sink: `EXPECT_EQ(a, b) << "context"` accumulates into it.
struct Msg {
  std::ostringstream os;
  template <typename T>
  Msg& operator<<(const T& v) {
    os << v;
    return *this;
  }
};

struct Reporter {
  const char* file;
  int line;
  std::string what;
  bool fatal;
  Msg msg;
  Reporter(const char* f, int l, std::string w, bool fat) : file(f), line(l), what(std::move(w)), fatal(fat) {}
  ~Reporter() {
    std::printf("%s:%d: Failure\n%s\n", file, line, what.c_str());
    const std::string extra = msg.os.str();
    if (!extra.empty()) std::printf("%s\n", extra.c_str());
    ++failures_in_test();
  }
};

struct FatalReturn {};

template <typename A, typename B>
bool eq(const A& a, const B& b) {
  if constexpr (std::is_integral_v<A> && std::is_integral_v<B> && std::is_signed_v<A> != std::is_signed_v<B>)
    return static_cast<long double>(a) == static_cast<long double>(b);
  else
    return a == b;
}
template <typename A, typename B>
bool lt(const A& a, const B& b) {
  if constexpr (std::is_integral_v<A> && std::is_integral_v<B> && std::is_signed_v<A> != std::is_signed_v<B>)
    return static_cast<long double>(a) < static_cast<long double>(b);
  else
    return a < b;
}

inline bool ulp_eq(double a, double b, int bits) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  if (bits == 64) {
    int64_t ia, ib;
    std::memcpy(&ia, &a, 8);
    std::memcpy(&ib, &b, 8);
    if (ia < 0) ia = INT64_MIN - ia;
    if (ib < 0) ib = INT64_MIN - ib;
    const long double d = (long double)ia - (long double)ib;
    return (d < 0 ? -d : d) <= 4;
  }
  const float fa = (float)a, fb = (float)b;
  int32_t ia, ib;
  std::memcpy(&ia, &fa, 4);
  std::memcpy(&ib, &fb, 4);
  if (ia < 0) ia = INT32_MIN - ia;
  if (ib < 0) ib = INT32_MIN - ib;
  const int64_t d = (int64_t)ia - (int64_t)ib;
  return (d < 0 ? -d : d) <= 4;
}

inline std::string& filter_out() {  // ":"-separated Suite.Name list to skip
  static std::string f;
  return f;
}

inline int run_all() {
  int failed = 0;
  std::vector<std::string> bad;
  std::printf("[==========] Running %zu tests.\n", registry().size());
  for (const Case& c : registry()) {
    const std::string full = std::string(c.suite) + "." + c.name;
    if ((":" + filter_out() + ":").find(":" + full + ":") != std::string::npos) {
      std::printf("[ SKIPPED  ] %s (filtered)\n", full.c_str());
      continue;
    }
    std::printf("[ RUN      ] %s.%s\n", c.suite, c.name);
    std::fflush(stdout);
    failures_in_test() = 0;
    try {
      c.fn();
    } catch (const FatalReturn&) {
    } catch (const std::exception& e) {
      std::printf("unexpected exception: %s\n", e.what());
      ++failures_in_test();
    } catch (...) {
      std::printf("unexpected non-std exception\n");
      ++failures_in_test();
    }
    if (failures_in_test()) {
      ++failed;
      bad.push_back(std::string(c.suite) + "." + c.name);
      std::printf("[  FAILED  ] %s.%s\n", c.suite, c.name);
    } else {
      std::printf("[       OK ] %s.%s\n", c.suite, c.name);
    }
  }
  std::printf("[==========] %zu tests ran.\n[  PASSED  ] %zu tests.\n", registry().size(),
              registry().size() - (size_t)failed);
  if (failed) {
    std::printf("[  FAILED  ] %d tests, listed below:\n", failed);
    for (auto& b : bad) std::printf("[  FAILED  ] %s\n", b.c_str());
  }
  return failed ? 1 : 0;
}

}  // namespace gtest_shim

namespace testing {
// supports the negative form of --gtest_filter only: --gtest_filter=-A.b:C.d
inline void InitGoogleTest(int* argc, char** argv) {
  for (int i = 1; argc && i < *argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--gtest_filter=-", 0) == 0) gtest_shim::filter_out() = a.substr(16);
  }
}
}  // namespace testing
#define RUN_ALL_TESTS() ::gtest_shim::run_all()

#define GTS_CAT_(a, b) a##b
#define GTS_CAT(a, b) GTS_CAT_(a, b)
#define TEST(suite, name)                                                                  \
  static void GTS_CAT(gts_##suite##_, name)();                                             \
  static ::gtest_shim::Registrar GTS_CAT(gts_reg_##suite##_, name)(#suite, #name,          \
                                                                   &GTS_CAT(gts_##suite##_, name)); \
  static void GTS_CAT(gts_##suite##_, name)()

// A failing check constructs a Reporter whose destructor prints and counts
// the failure; fatal checks then throw FatalReturn out of the test body.
#define GTS_CHECK(cond, text, fatal)                                                       \
  if (cond) {                                                                              \
  } else                                                                                   \
    for (bool gts_once = true; gts_once;                                                   \
         gts_once = false, (fatal) ? throw ::gtest_shim::FatalReturn() : (void)0)          \
  ::gtest_shim::Reporter(__FILE__, __LINE__, text, fatal).msg

#define GTS_BIN(a, b, pred, op, fatal)                                                     \
  GTS_CHECK(pred, std::string("Expected: ") + #a + " " op " " + #b + "\n  actual: " +      \
                      ::gtest_shim::show(a) + " vs " + ::gtest_shim::show(b), fatal)

#define EXPECT_EQ(a, b) GTS_BIN(a, b, ::gtest_shim::eq((a), (b)), "==", false)
#define EXPECT_NE(a, b) GTS_BIN(a, b, !::gtest_shim::eq((a), (b)), "!=", false)
#define EXPECT_LT(a, b) GTS_BIN(a, b, ::gtest_shim::lt((a), (b)), "<", false)
#define EXPECT_LE(a, b) GTS_BIN(a, b, !::gtest_shim::lt((b), (a)), "<=", false)
#define EXPECT_GT(a, b) GTS_BIN(a, b, ::gtest_shim::lt((b), (a)), ">", false)
#define EXPECT_GE(a, b) GTS_BIN(a, b, !::gtest_shim::lt((a), (b)), ">=", false)
#define ASSERT_EQ(a, b) GTS_BIN(a, b, ::gtest_shim::eq((a), (b)), "==", true)
#define ASSERT_NE(a, b) GTS_BIN(a, b, !::gtest_shim::eq((a), (b)), "!=", true)
#define ASSERT_LT(a, b) GTS_BIN(a, b, ::gtest_shim::lt((a), (b)), "<", true)
#define ASSERT_LE(a, b) GTS_BIN(a, b, !::gtest_shim::lt((b), (a)), "<=", true)
#define ASSERT_GT(a, b) GTS_BIN(a, b, ::gtest_shim::lt((b), (a)), ">", true)
#define ASSERT_GE(a, b) GTS_BIN(a, b, !::gtest_shim::lt((a), (b)), ">=", true)
#define EXPECT_TRUE(c) GTS_CHECK(static_cast<bool>(c), std::string("Expected true: ") + #c, false)
#define EXPECT_FALSE(c) GTS_CHECK(!static_cast<bool>(c), std::string("Expected false: ") + #c, false)
#define ASSERT_TRUE(c) GTS_CHECK(static_cast<bool>(c), std::string("Expected true: ") + #c, true)
#define ASSERT_FALSE(c) GTS_CHECK(!static_cast<bool>(c), std::string("Expected false: ") + #c, true)
#define EXPECT_DOUBLE_EQ(a, b) GTS_BIN(a, b, ::gtest_shim::ulp_eq((double)(a), (double)(b), 64), "~==", false)
#define EXPECT_FLOAT_EQ(a, b) GTS_BIN(a, b, ::gtest_shim::ulp_eq((double)(a), (double)(b), 32), "~==", false)
#define EXPECT_NEAR(a, b, tol)                                                             \
  GTS_CHECK(std::fabs((double)(a) - (double)(b)) <= (double)(tol),                         \
            std::string("Expected |") + #a + " - " + #b + "| <= " + #tol + "\n  actual: " + \
                ::gtest_shim::show(a) + " vs " + ::gtest_shim::show(b), false)

#define GTS_THROWS(stmt, ex, fatal)                                                        \
  GTS_CHECK(([&]() -> bool {                                                               \
              try {                                                                        \
                stmt;                                                                      \
              } catch (const ex&) {                                                        \
                return true;                                                               \
              } catch (...) {                                                              \
                return false;                                                              \
              }                                                                            \
              return false;                                                                \
            }()),                                                                          \
            std::string("Expected ") + #stmt + " to throw " + #ex, fatal)
#define EXPECT_THROW(stmt, ex) GTS_THROWS(stmt, ex, false)
#define ASSERT_THROW(stmt, ex) GTS_THROWS(stmt, ex, true)
#define EXPECT_NO_THROW(stmt)                                                              \
  GTS_CHECK(([&]() -> bool {                                                               \
              try {                                                                        \
                stmt;                                                                      \
              } catch (...) {                                                              \
                return false;                                                              \
              }                                                                            \
              return true;                                                                 \
            }()),                                                                          \
            std::string("Expected no throw: ") + #stmt, false)

// gtest_main equivalent
int main(int argc, char** argv) {
  ::testing::InitGoogleTest(&argc, argv);
  return RUN_ALL_TESTS();
}
