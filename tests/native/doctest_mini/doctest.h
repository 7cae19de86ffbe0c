// doctest.h -- a minimal doctest-compatible test runner.
//
// TEST INFRASTRUCTURE ONLY.  doctest itself is not installed in this image
// (the reference vendors it under proj/vendor/, which its .gitignore
// excludes), so this header implements the subset the reference's unit
// suites use -- TEST_CASE, SUBCASE (one level), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, MESSAGE, doctest::Approx,
// doctest::Contains -- so those suites can be compiled UNCHANGED against the
// B200 drop-in (tests/native/build_dropin.sh).  Semantics follow doctest's
// documented behaviour: failed CHECKs are counted and the case continues,
// REQUIRE/FAIL abort the case, each SUBCASE runs in its own pass of the case.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  explicit Contains(std::string x) : s(std::move(x)) {}
};

namespace detail {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  int checks = 0;
  int failed_checks = 0;
  bool case_failed = false;
  int sub_target = 0;
  int sub_seen = 0;
  bool sub_more = false;
};

inline State& st() {
  static State s;
  return s;
}

struct Abort {};

inline void fail(const char* file, int line, const std::string& what) {
  ++st().failed_checks;
  st().case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr,
                  bool require) {
  ++st().checks;
  if (ok) return;
  fail(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
  if (require) throw Abort{};
}

inline bool enter_subcase() {
  const int idx = st().sub_seen++;
  if (idx == st().sub_target) return true;
  if (idx > st().sub_target) st().sub_more = true;
  return false;
}

inline bool message_matches(const std::string& msg, const std::string& want) {
  return msg == want;
}
inline bool message_matches(const std::string& msg, const Contains& want) {
  return msg.find(want.s) != std::string::npos;
}
inline bool message_matches(const std::string& msg, const char* want) {
  return msg == want;
}

inline int run_all() {
  int failed_cases = 0, passed_cases = 0;
  for (const Case& c : registry()) {
    st().case_failed = false;
    st().sub_target = 0;
    do {
      st().sub_seen = 0;
      st().sub_more = false;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        fail(c.file, c.line, "unexpected non-standard exception");
      }
      ++st().sub_target;
    } while (st().sub_more);
    if (st().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", c.name, c.file, c.line);
    } else {
      ++passed_cases;
    }
  }
  std::printf("[doctest-mini] test cases: %d | %d passed | %d failed\n",
              passed_cases + failed_cases, passed_cases, failed_cases);
  std::printf("[doctest-mini] assertions: %d | %d passed | %d failed\n",
              st().checks, st().checks - st().failed_checks, st().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                            \
  static void fn();                                                      \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn,         \
                                                     __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define CHECK(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define FAIL(msg)                                                         \
  do {                                                                    \
    std::ostringstream doctest_os_;                                       \
    doctest_os_ << msg;                                                   \
    ::doctest::detail::fail(__FILE__, __LINE__, doctest_os_.str());      \
    throw ::doctest::detail::Abort{};                                     \
  } while (0)
#define MESSAGE(msg)                                                      \
  do {                                                                    \
    std::ostringstream doctest_os_;                                       \
    doctest_os_ << msg;                                                   \
    std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest_os_.str().c_str()); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                        \
  do {                                                                    \
    bool doctest_ok_ = false;                                             \
    try {                                                                 \
      static_cast<void>(expr);                                            \
    } catch (const __VA_ARGS__&) {                                        \
      doctest_ok_ = true;                                                 \
    } catch (...) {                                                       \
    }                                                                     \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__,             \
                             "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                             \
  do {                                                                    \
    bool doctest_ok_ = false;                                             \
    try {                                                                 \
      static_cast<void>(expr);                                            \
    } catch (const __VA_ARGS__& e) {                                      \
      doctest_ok_ = ::doctest::detail::message_matches(e.what(), with);  \
    } catch (...) {                                                       \
    }                                                                     \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__,             \
                             "THROWS_WITH_AS(" #expr ")", false);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
