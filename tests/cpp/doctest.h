// tests/cpp/doctest.h -- a minimal stand-in for the doctest macros the
// reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx(x).epsilon(e)), so those test sources
// (/root/reference/proj/tests/*.cpp, which expect <doctest.h> -- not shipped
// with the reference) compile unchanged against the B200 C++
// facade.  Not the doctest library: registration + a runner + counters.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
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
  friend bool operator==(double a, const Approx& b) { return b.match(a); }
  friend bool operator==(const Approx& b, double a) { return b.match(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.match(a); }

 private:
  bool match(double a) const {
    const double scale = 1.0 + std::fmax(std::fabs(a), std::fabs(v_));
    return std::fabs(a - v_) < eps_ * scale;
  }
  double v_;
  double eps_ = 1.1920929e-7 * 100;  // doctest's default: 100 float epsilons
};

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline long& checks() {
  static long n = 0;
  return n;
}
inline long& failures() {
  static long n = 0;
  return n;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: %s failed: %s\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    const long f0 = failures();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "TEST_CASE \"%s\": uncaught exception: %s\n", c.name, e.what());
    }
    if (failures() != f0) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed; assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, checks(), failures());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                        \
  static void fn();                                                             \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);         \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                              \
  do {                                                                                          \
    bool doctest_ok_ = false;                                                                   \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const __VA_ARGS__&) {                                                              \
      doctest_ok_ = true;                                                                       \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
