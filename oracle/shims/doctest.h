// TEST INFRASTRUCTURE — a tiny doctest-compatible harness (doctest itself is
// vendored by the reference under proj/vendor/, which is git-ignored and
// absent: proj/.gitignore:2). It implements exactly the macros the
// reference's unit tests use: TEST_CASE, CHECK, CHECK_THROWS_AS,
// CHECK_NOTHROW, REQUIRE, FAIL and doctest::Approx (same comparison rule:
// |a - b| < eps * (scale + max(|a|, |b|)), default eps = 100 * FLT_EPSILON).
// Runner options: -tc=<substring> (repeatable, comma-separated) selects
// cases, -ltc lists them, -s prints every case name.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

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
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }
  friend bool operator<(double a, const Approx& b) { return a < b.v_ && a != b; }
  friend bool operator>(double a, const Approx& b) { return a > b.v_ && a != b; }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireFailed {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void report(const char* file, int line, const char* what, const std::string& extra = {}) {
  ++failures();
  std::fprintf(stderr, "%s:%d: ERROR: %s%s%s\n", file, line, what, extra.empty() ? "" : " -- ",
               extra.c_str());
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQ(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                          \
  static void DOCTEST_UNIQ(doctest_fn_)();                                                       \
  static ::doctest::detail::Registrar DOCTEST_UNIQ(doctest_reg_)(name, __FILE__, __LINE__,       \
                                                                 &DOCTEST_UNIQ(doctest_fn_));    \
  static void DOCTEST_UNIQ(doctest_fn_)()

#define DOCTEST_CHECK_IMPL(expr, fatal)                                          \
  do {                                                                           \
    ++::doctest::detail::checks();                                               \
    bool doctest_ok_ = false;                                                    \
    try {                                                                        \
      doctest_ok_ = static_cast<bool>(expr);                                     \
    } catch (const std::exception& e) {                                          \
      ::doctest::detail::report(__FILE__, __LINE__, #expr, e.what());            \
      if (fatal) throw ::doctest::detail::RequireFailed{};                       \
      break;                                                                     \
    }                                                                            \
    if (!doctest_ok_) {                                                          \
      ::doctest::detail::report(__FILE__, __LINE__, #expr);                      \
      if (fatal) throw ::doctest::detail::RequireFailed{};                       \
    }                                                                            \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    ++::doctest::detail::checks();                                                        \
    bool doctest_thrown_ = false;                                                         \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_thrown_ = true;                                                             \
    } catch (...) {                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, #expr, "threw a different type");     \
      doctest_thrown_ = true;                                                             \
    }                                                                                     \
    if (!doctest_thrown_) ::doctest::detail::report(__FILE__, __LINE__, #expr, "did not throw"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, ...) CHECK_THROWS_AS(expr, __VA_ARGS__)

#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    ++::doctest::detail::checks();                                                         \
    try {                                                                                  \
      static_cast<void>(__VA_ARGS__);                                                      \
    } catch (const std::exception& e) {                                                    \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__, e.what());               \
    } catch (...) {                                                                        \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__, "threw");                \
    }                                                                                      \
  } while (0)
#define REQUIRE_NOTHROW(...) CHECK_NOTHROW(__VA_ARGS__)

#define FAIL(msg)                                                                \
  do {                                                                           \
    std::ostringstream doctest_os_;                                              \
    doctest_os_ << msg;                                                          \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", doctest_os_.str());    \
    throw ::doctest::detail::RequireFailed{};                                    \
  } while (0)
#define MESSAGE(msg) \
  do {               \
  } while (0)
#define INFO(...) \
  do {            \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::vector<std::string> filters;
  bool list = false, show = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("-tc=", 0) == 0 || a.rfind("--test-case=", 0) == 0) {
      std::string v = a.substr(a.find('=') + 1);
      std::size_t b = 0;
      while (b <= v.size()) {
        std::size_t e = v.find(',', b);
        if (e == std::string::npos) e = v.size();
        if (e > b) filters.push_back(v.substr(b, e - b));
        b = e + 1;
      }
    } else if (a == "-ltc") {
      list = true;
    } else if (a == "-s") {
      show = true;
    }
  }
  int ran = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (!filters.empty()) {
      bool hit = false;
      for (const auto& f : filters) hit = hit || std::strstr(c.name, f.c_str()) != nullptr;
      if (!hit) continue;
    }
    if (list) {
      std::printf("%s\n", c.name);
      continue;
    }
    const int before = ::doctest::detail::failures();
    if (show) std::printf("[case] %s\n", c.name);
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::report(c.file, c.line, c.name, std::string("unexpected exception: ") + e.what());
    }
    ++ran;
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\") %s:%d\n", c.name, c.file, c.line);
    }
  }
  if (!list)
    std::printf("[doctest] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", ran,
                ran - failed_cases, failed_cases, ::doctest::detail::checks(), ::doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
