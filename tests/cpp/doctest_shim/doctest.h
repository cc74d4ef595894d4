// TEST INFRASTRUCTURE: a minimal doctest-compatible shim, written for this repo.
//
// The reference's doctest suites (proj/tests/test_*.cpp) are compiled against
// the B200 strata headers to check the drop-in; the real doctest.h is not in the
// image (the reference's vendor/ directory is absent). This header implements
// only what those suites use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CAPTURE, FAIL and doctest::Approx.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-05;  // 100 * FLT_EPSILON
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& case_failed() {
  static int f = 0;
  return f;
}
inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}
inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  case_failed() = 1;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const std::string& c : captures()) std::fprintf(stderr, "    with %s\n", c.c_str());
}
struct Capture {
  explicit Capture(std::string s) { captures().push_back(std::move(s)); }
  ~Capture() { captures().pop_back(); }
};
template <typename T>
std::string show(const T& v) {
  std::ostringstream os;
  if constexpr (requires { os << v; }) os << v;
  else os << "?";
  return os.str();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                           \
  static void fn();                                                                                \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...)                                                                                 \
  do {                                                                                             \
    try {                                                                                          \
      if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )"); \
    } catch (const std::exception& e_) {                                                          \
      ::doctest::detail::fail(__FILE__, __LINE__,                                                  \
                              std::string("CHECK( " #__VA_ARGS__ " ) threw: ") + e_.what());       \
    }                                                                                              \
  } while (0)
#define REQUIRE(...)                                                                               \
  do {                                                                                             \
    if (!(__VA_ARGS__)) {                                                                          \
      ::doctest::detail::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");                   \
      throw ::doctest::detail::RequireFailed{};                                                    \
    }                                                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                \
  do {                                                                                             \
    bool ok_ = false;                                                                              \
    try {                                                                                          \
      (void)(expr);                                                                                \
    } catch (const type&) {                                                                        \
      ok_ = true;                                                                                  \
    } catch (...) {                                                                                \
    }                                                                                              \
    if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #type " )"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                                      \
  do {                                                                                             \
    bool ok_ = false;                                                                              \
    std::string got_ = "<no exception>";                                                           \
    try {                                                                                          \
      (void)(expr);                                                                                \
    } catch (const type& e_) {                                                                     \
      got_ = e_.what();                                                                            \
      ok_ = got_ == std::string(msg);                                                              \
    } catch (const std::exception& e_) {                                                          \
      got_ = std::string("other exception: ") + e_.what();                                         \
    } catch (...) {                                                                                \
    }                                                                                              \
    if (!ok_)                                                                                      \
      ::doctest::detail::fail(__FILE__, __LINE__,                                                  \
                              "CHECK_THROWS_WITH_AS( " #expr " ) got: " + got_);                   \
  } while (0)
#define CAPTURE(x) ::doctest::detail::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(#x " := " + ::doctest::detail::show(x))
#define FAIL(msg)                                                                                  \
  do {                                                                                             \
    ::doctest::detail::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg));                    \
    throw ::doctest::detail::RequireFailed{};                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    ++cases;
    ::doctest::detail::case_failed() = 0;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
    }
    if (::doctest::detail::case_failed()) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", c.name);
    }
  }
  std::printf("[doctest shim] test cases: %d | %d passed | %d failed | assertion failures: %d\n", cases,
              cases - failed_cases, failed_cases, ::doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
