// doctest-subset — TEST INFRASTRUCTURE ONLY. The reference's unit tests
// (proj/tests/*.cpp) include <doctest.h> from a git-ignored vendor/ directory
// that is absent here (proj/CMakeLists.txt:8, proj/.gitignore:2). This header
// implements the part of doctest's interface those tests use: TEST_SUITE,
// TEST_CASE, SUBCASE (each leaf subcase path runs the test case once, as
// doctest does), CHECK, CHECK_MESSAGE, REQUIRE, CHECK_THROWS_AS, FAIL and
// doctest::Approx; a main with -ts=<suite> filtering, one line per test case
// (PASS/FAIL with its failed assertions) and a nonzero exit on failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <set>
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
  friend bool operator==(double lhs, const Approx& r) {
    // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.v_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.v_ || lhs == r; }
  friend bool operator<(double lhs, const Approx& r) { return lhs < r.v_ && lhs != r; }
  friend bool operator>(double lhs, const Approx& r) { return lhs > r.v_ && lhs != r; }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest default: float epsilon * 100
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* suite;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
  }
};

struct RequireAbort {};

// Per-run state of the current test case.
struct State {
  std::vector<std::string> failures;
  long long asserts = 0;
  // subcase traversal (Catch/doctest sections)
  std::set<std::vector<std::string>> done;
  std::vector<std::string> path;
  std::vector<bool> entered_at_depth;  // a subcase was entered at this depth in this run
  bool pending = false;                // an unvisited subcase was skipped in this run
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& msg = {}) {
  auto& st = state();
  ++st.asserts;
  if (ok) return;
  std::ostringstream os;
  os << file << ":" << line << ": CHECK( " << expr << " ) failed";
  if (!msg.empty()) os << " -- " << msg;
  if (!st.path.empty()) {
    os << " [subcase";
    for (const auto& p : st.path) os << " / " << p;
    os << "]";
  }
  st.failures.push_back(os.str());
}

template <class... T> std::string concat(const T&... parts) {
  std::ostringstream os;
  (os << ... << parts);
  return os.str();
}

class Subcase {
 public:
  Subcase(const char* name) : name_(name) {
    auto& st = state();
    const std::size_t depth = st.path.size();
    if (st.entered_at_depth.size() <= depth) st.entered_at_depth.resize(depth + 1, false);
    std::vector<std::string> me = st.path;
    me.push_back(name_);
    if (st.done.count(me)) return;
    if (st.entered_at_depth[depth]) {
      st.pending = true;  // a sibling ran in this pass; this one runs in a later pass
      return;
    }
    st.entered_at_depth[depth] = true;
    st.path = me;
    pending_before_ = st.pending;
    st.pending = false;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    auto& st = state();
    // Done when no nested subcase was left unvisited during this pass.
    if (!st.pending) st.done.insert(st.path);
    st.pending = st.pending || pending_before_;
    st.path.pop_back();
    if (st.entered_at_depth.size() > st.path.size() + 1) st.entered_at_depth.resize(st.path.size() + 1);
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string name_;
  bool entered_ = false;
  bool pending_before_ = false;
};

inline int run(int argc, char** argv) {
  std::string suite_filter, case_filter;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("-ts=", 0) == 0) suite_filter = a.substr(4);
    if (a.rfind("--test-suite=", 0) == 0) suite_filter = a.substr(13);
    if (a.rfind("-tc=", 0) == 0) case_filter = a.substr(4);
  }
  int failed = 0, passed = 0;
  long long asserts = 0;
  for (const auto& tc : registry()) {
    if (!suite_filter.empty() && suite_filter != tc.suite) continue;
    if (!case_filter.empty() && case_filter != tc.name) continue;
    auto& st = state();
    st = State{};
    std::string error;
    for (int pass = 0; pass < 10000; ++pass) {
      st.path.clear();
      st.entered_at_depth.assign(1, false);
      st.pending = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        error = std::string("unexpected exception: ") + e.what();
      } catch (...) {
        error = "unexpected non-std exception";
      }
      if (!error.empty()) break;
      if (!st.pending) break;  // every subcase path has run
    }
    if (!error.empty()) st.failures.push_back(error);
    asserts += st.asserts;
    const bool ok = st.failures.empty();
    (ok ? passed : failed) += 1;
    std::printf("%s [%s] %s (%s:%d)\n", ok ? "PASS" : "FAIL", tc.suite, tc.name, tc.file, tc.line);
    for (const auto& f : st.failures) std::printf("    %s\n", f.c_str());
  }
  std::printf("test cases: %d passed, %d failed; assertions: %lld\n", passed, failed, asserts);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

// Suite name lookup: TEST_SUITE opens a namespace that shadows this one.
static inline const char* doctest_suite_name() { return ""; }

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TS_IMPL(name, ns) \
  namespace ns { static inline const char* doctest_suite_name() { return name; } } namespace ns
#define TEST_SUITE(name) DOCTEST_TS_IMPL(name, DOCTEST_CAT(doctest_suite_, __COUNTER__))
#define DOCTEST_TC_IMPL(name, fn)                                                                     \
  static void fn();                                                                                    \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(fn, name, doctest_suite_name(), __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, DOCTEST_CAT(doctest_test_, __COUNTER__))
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define CHECK_MESSAGE(cond, ...)                                                                      \
  ::doctest::detail::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, ::doctest::detail::concat(__VA_ARGS__))
#define REQUIRE(...)                                                                                  \
  do {                                                                                                 \
    const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                            \
    ::doctest::detail::report(doctest_ok, #__VA_ARGS__, __FILE__, __LINE__);                           \
    if (!doctest_ok) throw ::doctest::detail::RequireAbort{};                                          \
  } while (0)
#define FAIL(msg)                                                                                     \
  do {                                                                                                 \
    std::ostringstream doctest_msg_os;                                                                 \
    doctest_msg_os << msg;                                                                             \
    ::doctest::detail::report(false, "FAIL", __FILE__, __LINE__, doctest_msg_os.str());                \
    throw ::doctest::detail::RequireAbort{};                                                           \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
  do {                                                                                                 \
    bool doctest_threw_right = false;                                                                  \
    std::string doctest_why = "did not throw";                                                         \
    try {                                                                                              \
      static_cast<void>(expr);                                                                         \
    } catch (const __VA_ARGS__&) {                                                                     \
      doctest_threw_right = true;                                                                      \
    } catch (const std::exception& e) {                                                                \
      doctest_why = std::string("threw another type: ") + e.what();                                    \
    } catch (...) {                                                                                    \
      doctest_why = "threw a non-std exception";                                                       \
    }                                                                                                  \
    ::doctest::detail::report(doctest_threw_right, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__, \
                              doctest_threw_right ? "" : doctest_why);                                 \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
  do {                                                                                                 \
    bool doctest_ok = true;                                                                            \
    try {                                                                                              \
      static_cast<void>(expr);                                                                         \
    } catch (...) {                                                                                    \
      doctest_ok = false;                                                                              \
    }                                                                                                  \
    ::doctest::detail::report(doctest_ok, "NOTHROW(" #expr ")", __FILE__, __LINE__);                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
