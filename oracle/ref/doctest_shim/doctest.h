// TEST-ONLY doctest subset shim, used solely to compile the reference's own
// hot-path unit tests (/root/reference/proj/tests/test_{inner_product,
// registration,kernels,se3,point_cloud}.cpp) against the oracle build, so that
// the Eigen shim and the compiled reference are pinned by the reference's own
// assertions. SUBCASEs run sequentially inside one pass of their TEST_CASE
// (every SUBCASE in those files is independent of its siblings).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest default: float eps * 100
};
inline bool operator==(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

namespace detail {
struct Registry {
  std::vector<std::pair<const char*, void (*)()>> cases;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct Registrar {
  Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
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
inline const char*& current() {
  static const char* c = "";
  return c;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), expr);
  if (require) throw RequireFailed{};
}
inline bool matches(const std::exception& e, const Contains& c) {
  return std::string(e.what()).find(c.needle) != std::string::npos;
}
inline bool matches(const std::exception& e, const char* s) { return std::string(e.what()) == s; }
}  // namespace detail

// excluded: test-case names to skip (the façade run's bitwise-only cases)
inline int run_all(const std::vector<std::string>& excluded = {}) {
  size_t skipped = 0;
  for (auto& [name, fn] : detail::Registry::get().cases) {
    bool skip = false;
    for (const std::string& x : excluded) skip = skip || x == name;
    if (skip) {
      ++skipped;
      std::printf("[doctest-shim] skipped: %s\n", name);
      continue;
    }
    const int before = detail::failures();
    detail::current() = name;
    try {
      fn();
    } catch (const detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++detail::failures();
      std::fprintf(stderr, "exception in \"%s\": %s\n", name, e.what());
    }
    if (!excluded.empty()) std::printf("[doctest-shim] %s: %s\n", detail::failures() == before ? "ok" : "FAILED", name);
  }
  std::printf("[doctest-shim] test cases: %zu | skipped: %zu | assertions: %d | failed: %d\n",
              detail::Registry::get().cases.size(), skipped, detail::checks(), detail::failures());
  return detail::failures() == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE_IMPL(fn, name)                                                  \
  static void fn();                                                               \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);            \
  static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool ok_ = true;                                                                        \
    try {                                                                                   \
      (void)(__VA_ARGS__);                                                                  \
    } catch (...) {                                                                         \
      ok_ = false;                                                                          \
    }                                                                                       \
    doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);       \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                          \
  do {                                                                                      \
    bool ok_ = false;                                                                       \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const exc&) {                                                                  \
      ok_ = true;                                                                           \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::detail::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);            \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, exc)                                               \
  do {                                                                                      \
    bool ok_ = false;                                                                       \
    try {                                                                                   \
      (void)(expr);                                                                         \
    } catch (const exc& e_) {                                                               \
      ok_ = doctest::detail::matches(e_, with);                                             \
    } catch (...) {                                                                         \
    }                                                                                       \
    doctest::detail::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);       \
  } while (0)
