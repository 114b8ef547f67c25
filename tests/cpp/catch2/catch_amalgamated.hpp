// catch2/catch_amalgamated.hpp -- minimal Catch2-compatible test shim (the
// subset the reference's tests use: TEST_CASE, REQUIRE, REQUIRE_FALSE,
// REQUIRE_NOTHROW, REQUIRE_THROWS_AS, FAIL, Catch::Approx), so the
// reference's UNMODIFIED test sources (/root/reference/proj/tests/
// test_bitkernel.cpp, test_quantizer.cpp, test_tune.cpp) compile against the
// drop-in headers include/abq/*.hpp and run on the GPU engine.  Catch2 itself
// is not in this image.  One TU defines the runner with
// ABQ_CATCH_MAIN; every test case runs once, a failed REQUIRE aborts that case.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace abq_catch {

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
struct Failure {
  std::string what;
};
inline long long& assertions() {
  static long long n = 0;
  return n;
}
[[noreturn]] inline void fail_at(const char* file, int line, const std::string& msg) {
  std::ostringstream os;
  os << file << ":" << line << ": " << msg;
  throw Failure{os.str()};
}

}  // namespace abq_catch

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  bool matches(double x) const {
    // Catch2 default: |x - v| <= margin or <= eps * (scale + max(|x|, |v|)), eps = 100 * float eps
    const double d = std::fabs(x - v_);
    return d <= margin_ || d <= eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100.0;
  double margin_ = 0.0;
};
}  // namespace Catch

#define ABQ_CATCH_CAT2(a, b) a##b
#define ABQ_CATCH_CAT(a, b) ABQ_CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                  \
  static void ABQ_CATCH_CAT(abq_catch_case_, __LINE__)();                                    \
  static ::abq_catch::Registrar ABQ_CATCH_CAT(abq_catch_reg_, __LINE__)(                      \
      name, &ABQ_CATCH_CAT(abq_catch_case_, __LINE__));                                      \
  static void ABQ_CATCH_CAT(abq_catch_case_, __LINE__)()

#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    ++::abq_catch::assertions();                                                              \
    if (!(__VA_ARGS__)) ::abq_catch::fail_at(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )"); \
  } while (0)
#define REQUIRE_FALSE(...)                                                                    \
  do {                                                                                        \
    ++::abq_catch::assertions();                                                              \
    if ((__VA_ARGS__)) ::abq_catch::fail_at(__FILE__, __LINE__, "REQUIRE_FALSE( " #__VA_ARGS__ " )"); \
  } while (0)
#define REQUIRE_NOTHROW(...)                                                                  \
  do {                                                                                        \
    ++::abq_catch::assertions();                                                              \
    try {                                                                                     \
      (void)(__VA_ARGS__);                                                                    \
    } catch (const std::exception& e) {                                                       \
      ::abq_catch::fail_at(__FILE__, __LINE__, std::string("REQUIRE_NOTHROW threw: ") + e.what()); \
    }                                                                                         \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                         \
  do {                                                                                        \
    ++::abq_catch::assertions();                                                              \
    bool abq_caught_ = false;                                                                 \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const type&) {                                                                   \
      abq_caught_ = true;                                                                     \
    } catch (const std::exception& e) {                                                       \
      ::abq_catch::fail_at(__FILE__, __LINE__, std::string("REQUIRE_THROWS_AS( " #expr ", " #type " ) threw another type: ") + e.what()); \
    }                                                                                         \
    if (!abq_caught_) ::abq_catch::fail_at(__FILE__, __LINE__, "REQUIRE_THROWS_AS( " #expr ", " #type " ) did not throw"); \
  } while (0)
#define FAIL(msg) ::abq_catch::fail_at(__FILE__, __LINE__, std::string("FAIL: ") + (msg))

#ifdef ABQ_CATCH_MAIN
int main() {
  int failed = 0, passed = 0;
  for (const auto& c : ::abq_catch::registry()) {
    try {
      c.fn();
      ++passed;
      std::printf("PASS - %s\n", c.name);
    } catch (const ::abq_catch::Failure& f) {
      ++failed;
      std::printf("FAIL - %s\n  %s\n", c.name, f.what.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL - %s\n  unexpected exception: %s\n", c.name, e.what());
    }
    std::fflush(stdout);
  }
  std::printf("%d test cases: %d passed, %d failed, %lld assertions\n", passed + failed, passed, failed,
              ::abq_catch::assertions());
  return failed == 0 ? 0 : 1;
}
#endif
