// Minimal doctest-compatible subset used to compile the reference unit tests
// (/root/reference/proj/tests/*.cpp) unmodified: doctest itself is absent
// offline.  Supports TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, CAPTURE and doctest::Approx.
// TEST INFRASTRUCTURE ONLY (oracle/).
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  double value;
  double eps = 1e-6;
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) <= a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
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
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline long& checks() { static long c = 0; return c; }
inline long& failures() { static long c = 0; return c; }
inline std::vector<std::string>& captures() { static std::vector<std::string> c; return c; }
struct CaptureGuard {
  template <class T>
  CaptureGuard(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    captures().push_back(os.str());
  }
  ~CaptureGuard() { captures().pop_back(); }
};
inline void fail(const char* file, int line, const char* expr, bool fatal) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const auto& c : captures()) std::fprintf(stderr, "  with %s\n", c.c_str());
  if (fatal) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                  \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                 \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define DOCTEST_CHECK_IMPL(expr, fatal)                                              \
  do {                                                                               \
    ++::doctest::detail::checks();                                                   \
    if (!(expr)) ::doctest::detail::fail(__FILE__, __LINE__, #expr, fatal);          \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define CHECK_NOTHROW(...)                                                           \
  do {                                                                               \
    ++::doctest::detail::checks();                                                   \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      ::doctest::detail::fail(__FILE__, __LINE__, "NOTHROW " #__VA_ARGS__, false);   \
    }                                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                  \
  do {                                                                               \
    ++::doctest::detail::checks();                                                   \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type&) {                                                          \
      doctest_ok = true;                                                             \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok) ::doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #expr, false); \
  } while (0)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long cases_failed = 0;
  // DOCTEST_ONLY="prefix1|prefix2": run only the cases whose name starts with one
  const char* only = std::getenv("DOCTEST_ONLY");
  size_t ran = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (only && *only) {
      bool hit = false;
      for (const char* p = only; *p;) {
        const char* e = std::strchr(p, '|');
        const size_t n = e ? size_t(e - p) : std::strlen(p);
        hit |= std::strncmp(c.name, p, n) == 0;
        p += n + (e ? 1 : 0);
      }
      if (!hit) continue;
    }
    ++ran;
    const long before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail("<case>", 0, e.what(), false);
    }
    if (::doctest::detail::failures() != before) {
      ++cases_failed;
      std::fprintf(stderr, "case FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %ld failed | checks: %ld | %ld failed\n", ran, cases_failed, ::doctest::detail::checks(),
              ::doctest::detail::failures());
  return cases_failed == 0 ? 0 : 1;
}
#endif
