// Minimal doctest-compatible test harness (test infrastructure only). The
// reference's unit tests under /root/reference/proj/tests include <doctest.h>,
// which is not vendored; this header implements the macros they
// use so those test files compile unmodified against the Eigen shim and
// validate it.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_;
  double eps_ = 1.1920929e-05;  // float epsilon * 100, as doctest
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : s_(std::move(s)) {}
  bool check(const std::string& what) const { return what.find(s_) != std::string::npos; }
  std::string s_;
};

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline const char*& current() { static const char* c = ""; return c; }
inline void report(bool ok, const char* expr, const char* file, int line, const std::string& msg = {}) {
  ++checks();
  if (ok) return;
  ++failures();
  std::cerr << file << ":" << line << ": FAILED in \"" << current() << "\": " << expr;
  if (!msg.empty()) std::cerr << " (" << msg << ")";
  std::cerr << "\n";
}
inline bool matches(const std::string& what, const char* s) { return what == s; }
inline bool matches(const std::string& what, const Contains& c) { return c.check(what); }
inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    current() = tc.name;
    const int before = failures();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::cerr << "unexpected exception in \"" << tc.name << "\": " << e.what() << "\n";
    }
    if (failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - static_cast<std::size_t>(failed_cases), failed_cases,
              checks(), failures());
  return failures() == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                           \
  static void fn();                                                     \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define CHECK_MESSAGE(cond, msg)                                                    \
  do {                                                                              \
    std::ostringstream doctest_os_;                                                 \
    doctest_os_ << msg;                                                             \
    doctest::detail::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, doctest_os_.str()); \
  } while (0)
#define REQUIRE(...)                                                          \
  do {                                                                        \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                  \
    doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw doctest::detail::RequireFailed{};                 \
  } while (0)
#define CHECK_THROWS(...)                                         \
  do {                                                            \
    bool doctest_threw_ = false;                                  \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_threw_ = true; } \
    doctest::detail::report(doctest_threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                \
  do {                                                            \
    bool doctest_threw_ = false;                                  \
    try { (void)(expr); } catch (const exc&) { doctest_threw_ = true; } catch (...) {} \
    doctest::detail::report(doctest_threw_, "throws " #exc ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, doctest_what_, exc)                     \
  do {                                                            \
    bool doctest_ok_ = false;                                     \
    try { (void)(expr); } catch (const exc& e_) { doctest_ok_ = doctest::detail::matches(e_.what(), doctest_what_); } catch (...) {} \
    doctest::detail::report(doctest_ok_, "throws-with " #exc ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                        \
  do {                                                            \
    bool doctest_ok_ = true;                                      \
    try { (void)(__VA_ARGS__); } catch (...) { doctest_ok_ = false; } \
    doctest::detail::report(doctest_ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
