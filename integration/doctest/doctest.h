// doctest.h - a minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's suites (/root/reference/proj/tests/*.cpp) are written
// against doctest, which the reference does not vendor. This
// header implements exactly the subset they use -- TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// REQUIRE, REQUIRE_MESSAGE, FAIL, FAIL_CHECK, doctest::Approx,
// doctest::Contains -- so the suites compile unmodified from where they lie
// (oracle/Makefile `ref_suites`), once against af::interpret and once with
// the B200 executor swapped in (integration/swap_interpret.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    registry().push_back({n, f, file, line});
  }
};

struct AbortCase {};  // REQUIRE / FAIL: leave the current test case

struct State {
  long assertions = 0, failed_assertions = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

inline void fail_at(const char* file, int line, const std::string& what) {
  ++state().failed_assertions;
  state().case_failed = true;
  std::cerr << file << ":" << line << ": ERROR: " << what << "\n";
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(std::string x) : s(std::move(x)) {}
};
inline bool message_matches(const std::string& what, const Contains& c) {
  return what.find(c.s) != std::string::npos;
}
inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool message_matches(const std::string& what, const std::string& exact) {
  return what == exact;
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const AbortCase&) {
    } catch (const std::exception& e) {
      fail_at(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      fail_at(tc.file, tc.line, "unexpected exception");
    }
    std::printf("%s %s\n", state().case_failed ? "[FAIL]" : "[ ok ]", tc.name);
    failed_cases += state().case_failed;
  }
  std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", state().assertions,
              state().assertions - state().failed_assertions, state().failed_assertions);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                  \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                    \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                         \
      name, &DOCTEST_CAT(doctest_case_, __LINE__), __FILE__, __LINE__);                  \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define DOCTEST_COUNT() (++doctest::state().assertions)
#define CHECK(...)                                                                       \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    if (!(__VA_ARGS__)) doctest::fail_at(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )"); \
  } while (0)
#define CHECK_FALSE(...)                                                                 \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    if ((__VA_ARGS__)) doctest::fail_at(__FILE__, __LINE__, "CHECK_FALSE( " #__VA_ARGS__ " )"); \
  } while (0)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    if (!(__VA_ARGS__)) {                                                                \
      doctest::fail_at(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");               \
      throw doctest::AbortCase{};                                                        \
    }                                                                                    \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg)                                                       \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    if (!(cond)) {                                                                       \
      std::ostringstream doctest_os;                                                     \
      doctest_os << "REQUIRE( " #cond " ): " << msg;                                     \
      doctest::fail_at(__FILE__, __LINE__, doctest_os.str());                            \
      throw doctest::AbortCase{};                                                        \
    }                                                                                    \
  } while (0)
#define CHECK_NOTHROW(...)                                                               \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    try {                                                                                \
      (void)(__VA_ARGS__);                                                               \
    } catch (const std::exception& e) {                                                  \
      doctest::fail_at(__FILE__, __LINE__, std::string("CHECK_NOTHROW threw: ") + e.what()); \
    } catch (...) {                                                                      \
      doctest::fail_at(__FILE__, __LINE__, "CHECK_NOTHROW threw");                       \
    }                                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    try {                                                                                \
      (void)(expr);                                                                      \
      doctest::fail_at(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): no exception"); \
    } catch (const __VA_ARGS__&) {                                                       \
    } catch (...) {                                                                      \
      doctest::fail_at(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): wrong type");  \
    }                                                                                    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                            \
  do {                                                                                   \
    DOCTEST_COUNT();                                                                     \
    try {                                                                                \
      (void)(expr);                                                                      \
      doctest::fail_at(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr " ): no exception"); \
    } catch (const __VA_ARGS__& e) {                                                     \
      if (!doctest::message_matches(e.what(), with))                                     \
        doctest::fail_at(__FILE__, __LINE__,                                             \
                         std::string("CHECK_THROWS_WITH_AS: message '") + e.what() + "'"); \
    } catch (...) {                                                                      \
      doctest::fail_at(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS( " #expr " ): wrong type"); \
    }                                                                                    \
  } while (0)
#define FAIL_CHECK(msg)                                                                  \
  do {                                                                                   \
    std::ostringstream doctest_os;                                                       \
    doctest_os << msg;                                                                   \
    doctest::fail_at(__FILE__, __LINE__, doctest_os.str());                              \
  } while (0)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    std::ostringstream doctest_os;                                                       \
    doctest_os << msg;                                                                   \
    doctest::fail_at(__FILE__, __LINE__, doctest_os.str());                              \
    throw doctest::AbortCase{};                                                          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
