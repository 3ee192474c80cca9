// TEST INFRASTRUCTURE ONLY: a minimal Catch2-compatible harness (Catch2 is
// absent from this image) so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp, compiled in place, never copied)
// build and run: TEST_CASE registry, REQUIRE, REQUIRE_FALSE,
// REQUIRE_THROWS_AS, FAIL and a main() that runs every registered case.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {
struct Case {
  std::string name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};
struct Failure {
  std::string what;
};
inline long& assertions() {
  static long n = 0;
  return n;
}
}  // namespace catch_shim

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                           \
  static void CATCH_SHIM_CAT(catch_shim_case_, __LINE__)();                                            \
  static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(name,                         \
                                                                         &CATCH_SHIM_CAT(catch_shim_case_, __LINE__)); \
  static void CATCH_SHIM_CAT(catch_shim_case_, __LINE__)()
#define CATCH_SHIM_FAIL_AT(msg)                                                          \
  do {                                                                                   \
    std::ostringstream os_;                                                              \
    os_ << __FILE__ << ":" << __LINE__ << ": " << msg;                                   \
    throw catch_shim::Failure{os_.str()};                                                \
  } while (0)
#define REQUIRE(...)                                                 \
  do {                                                               \
    ++catch_shim::assertions();                                      \
    if (!(__VA_ARGS__)) CATCH_SHIM_FAIL_AT("REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_FALSE(...)                                                 \
  do {                                                                     \
    ++catch_shim::assertions();                                            \
    if ((__VA_ARGS__)) CATCH_SHIM_FAIL_AT("REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                    \
  do {                                                                                   \
    ++catch_shim::assertions();                                                          \
    bool caught_ = false;                                                                \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const type&) {                                                              \
      caught_ = true;                                                                    \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (!caught_) CATCH_SHIM_FAIL_AT("REQUIRE_THROWS_AS(" #expr ", " #type ")");         \
  } while (0)
#define FAIL(msg) CATCH_SHIM_FAIL_AT(msg)

#ifdef CATCH_SHIM_MAIN
int main(int argc, char** argv) {
  int failed = 0, ran = 0;
  for (auto& c : catch_shim::registry()) {
    if (argc > 1 && c.name.find(argv[1]) == std::string::npos) continue;
    ++ran;
    try {
      c.fn();
      std::printf("PASS %s\n", c.name.c_str());
    } catch (const catch_shim::Failure& f) {
      ++failed;
      std::printf("FAIL %s: %s\n", c.name.c_str(), f.what.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL %s: unexpected exception: %s\n", c.name.c_str(), e.what());
    }
  }
  std::printf("%d test cases, %d failed, %ld assertions\n", ran, failed, catch_shim::assertions());
  return failed ? 1 : 0;
}
#endif
