// TEST INFRASTRUCTURE ONLY: minimal doctest-compatible shim so the reference's
// own unit tests (/root/reference/proj/tests/*.cpp, doctest is not vendored
// there) can be compiled from their sources and run against the compiled
// reference (oracle/ref.mk target `tests`).  Supports exactly the subset the
// reference uses: TEST_CASE, sequential SUBCASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS and doctest::Approx(..).epsilon(..).
#pragma once
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(std::numeric_limits<float>::epsilon() * 100), scale_(1.0) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
 private:
  double v_, eps_, scale_;
};

namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Reg { Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); } };
struct State { int target = 0; int seen = 0; bool entered = false; long checks = 0; long failures = 0; };
inline State& st() { static State s; return s; }
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++st().checks;
  if (!ok) {
    ++st().failures;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
inline bool subcase_enter() {
  const bool run = st().seen == st().target;
  ++st().seen;
  if (run) st().entered = true;
  return run;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                  \
  static void fn();                                                                                \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);              \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::subcase_enter())
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                                \
  do {                                                                                             \
    bool ok_ = false;                                                                              \
    try { (void)(expr); } catch (const type&) { ok_ = true; } catch (...) {}                       \
    ::doctest::detail::report(ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace ::doctest::detail;
  int failed_cases = 0;
  for (const auto& c : registry()) {
    const long f0 = st().failures;
    const auto t0 = std::chrono::steady_clock::now();
    for (int target = 0;; ++target) {
      st().target = target; st().seen = 0; st().entered = false;
      try { c.fn(); } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++st().failures; std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
      }
      if (st().seen <= target + 1) break;  // no further subcases
    }
    if (st().failures != f0) { ++failed_cases; std::fprintf(stderr, "FAILED: %s\n", c.name); }
    std::fprintf(stderr, "[case] %-70s %8.3f s\n", c.name,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %ld | failed checks: %ld\n",
              registry().size(), failed_cases, st().checks, st().failures);
  return failed_cases == 0 ? 0 : 1;
}
#endif
