// A minimal stand-in for the doctest single header (the reference's
// vendor/doctest.h is git-ignored and absent: SURVEY.md §0.2, §8c).  Written
// for this repo; it implements only what the reference's test files use --
// TEST_CASE, CHECK / CHECK_FALSE / REQUIRE / CHECK_NOTHROW / CHECK_THROWS_AS /
// CHECK_THROWS_WITH_AS / FAIL, doctest::Approx (epsilon, scale) and
// doctest::Contains -- with doctest's documented semantics:
//   lhs == Approx(v)  <=>  |lhs - v| < eps (scale + max(|lhs|, |v|)),
//   eps defaulting to 100 float-epsilons and scale to 1.
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN provides main(), which runs every test
// case, prints "[doctest] test cases: N | M passed | K failed" plus
// "assertions: A | F failed", and returns non-zero on any failure.
#pragma once

#include <algorithm>
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
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = double(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

template <class T>
bool operator==(const T& lhs, const Approx& rhs) {
  return rhs.matches(double(lhs));
}
template <class T>
bool operator==(const Approx& lhs, const T& rhs) {
  return lhs.matches(double(rhs));
}
template <class T>
bool operator!=(const T& lhs, const Approx& rhs) {
  return !rhs.matches(double(lhs));
}
template <class T>
bool operator<=(const T& lhs, const Approx& rhs) {
  return double(lhs) < rhs.value() || rhs.matches(double(lhs));
}
template <class T>
bool operator>=(const T& lhs, const Approx& rhs) {
  return double(lhs) > rhs.value() || rhs.matches(double(lhs));
}

struct Contains {
  std::string s;
  explicit Contains(const char* t) : s(t) {}
  bool in(const std::string& msg) const { return msg.find(s) != std::string::npos; }
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

struct State {
  int assertions = 0, failed_assertions = 0;
  bool case_failed = false;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void result(bool ok, const char* file, int line, const char* macro, const char* expr, bool fatal) {
  State& st = state();
  ++st.assertions;
  if (ok) return;
  ++st.failed_assertions;
  st.case_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!  [test case \"%s\"]\n", file, line, macro, expr, st.current);
  if (fatal) throw RequireAbort{};
}

inline std::string message_of(const std::exception& e) { return e.what(); }
inline bool message_matches(const std::string& msg, const char* want) { return msg == want; }
inline bool message_matches(const std::string& msg, const Contains& want) { return want.in(msg); }

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline int run_all() {
  State& st = state();
  int failed_cases = 0;
  for (const Case& c : registry()) {
    st.current = c.name;
    st.case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++st.failed_assertions;
      st.case_failed = true;
      std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
    } catch (...) {
      ++st.failed_assertions;
      st.case_failed = true;
      std::printf("%s:%d: ERROR: test case \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
    }
    if (st.case_failed) ++failed_cases;
    std::printf("[doctest] %s: %s\n", st.case_failed ? "FAILED" : "passed", c.name);
  }
  const int n = int(registry().size());
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", n, n - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %d | %d passed | %d failed\n", st.assertions,
              st.assertions - st.failed_assertions, st.failed_assertions);
  std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                            \
  static void fn();                                                                                 \
  static const ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT(macro, cond, text, fatal)                                                          \
  do {                                                                                                  \
    bool doctest_ok_ = false;                                                                           \
    try {                                                                                               \
      doctest_ok_ = static_cast<bool>(cond);                                                            \
    } catch (const ::doctest::detail::RequireAbort&) {                                                  \
      throw;                                                                                            \
    } catch (...) {                                                                                     \
      doctest_ok_ = false;                                                                              \
    }                                                                                                   \
    ::doctest::detail::result(doctest_ok_, __FILE__, __LINE__, macro, text, fatal);                     \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define FAIL(msg) ::doctest::detail::result(false, __FILE__, __LINE__, "FAIL", msg, true)

#define CHECK_NOTHROW(...)                                                          \
  do {                                                                              \
    bool doctest_ok_ = true;                                                        \
    try {                                                                           \
      (void)(__VA_ARGS__);                                                          \
    } catch (...) {                                                                 \
      doctest_ok_ = false;                                                          \
    }                                                                               \
    ::doctest::detail::result(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                  \
      doctest_ok_ = true;                                                           \
    } catch (...) {                                                                 \
    }                                                                               \
    ::doctest::detail::result(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, want, ...)                                       \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__& e_) {                                               \
      doctest_ok_ = ::doctest::detail::message_matches(::doctest::detail::message_of(e_), want); \
    } catch (...) {                                                                 \
    }                                                                               \
    ::doctest::detail::result(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
