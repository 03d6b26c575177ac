// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE, oracle side).
//
// The reference's unit suites (/root/reference/proj/tests/*.cpp) are written
// against doctest, which is not vendored (/root/reference/proj/.gitignore:2).
// This header implements only the macro subset those suites use (SURVEY.md
// Appendix A): TEST_CASE, SUBCASE (with doctest's one-leaf-per-run
// re-entry), CHECK/REQUIRE(_FALSE), CHECK_THROWS_AS, CHECK_NOTHROW, FAIL,
// CAPTURE, CHECK_MESSAGE and doctest::Approx with doctest's default epsilon
// (FLT_EPSILON * 100) and scale formula. It is an independent
// implementation, written for this repo.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  // Subcase traversal: every run enters at most one not-yet-finished subcase
  // per nesting level; the test case re-runs while any subcase is pending.
  std::set<std::string> done;
  std::string path;
  std::vector<bool> entered;  // per depth: a subcase was entered this run
  int depth = 0;
  bool pending = false;
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  std::vector<std::string> captures;
};

inline State& st() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const std::string& what) {
  State& s = st();
  s.failures += 1;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const std::string& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
  if (!s.path.empty()) std::fprintf(stderr, "  in subcase %s\n", s.path.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require,
                  const std::string& msg = {}) {
  st().checks += 1;
  if (ok) return;
  report(file, line, std::string(expr) + (msg.empty() ? "" : (" -- " + msg)));
  if (require) throw RequireFailed{};
}

class Subcase {
 public:
  Subcase(const char* name, int line) {
    State& s = st();
    key_ = s.path + "/" + name + "#" + std::to_string(line);
    if (static_cast<int>(s.entered.size()) <= s.depth) s.entered.resize(s.depth + 1, false);
    if (s.done.count(key_)) return;
    if (s.entered[s.depth]) {
      s.pending = true;
      return;
    }
    s.entered[s.depth] = true;
    active_ = true;
    saved_path_ = s.path;
    saved_pending_ = s.pending;
    s.pending = false;
    s.path = key_;
    s.depth += 1;
    if (static_cast<int>(s.entered.size()) > s.depth)
      for (size_t d = s.depth; d < s.entered.size(); ++d) s.entered[d] = false;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = st();
    if (!s.pending) s.done.insert(key_);
    s.pending = saved_pending_ || s.pending;
    s.path = saved_path_;
    s.depth -= 1;
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_, saved_path_;
  bool active_ = false;
  bool saved_pending_ = false;
};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Capture {
  explicit Capture(std::string s) { st().captures.push_back(std::move(s)); }
  ~Capture() { st().captures.pop_back(); }
};

inline int run_all() {
  State& s = st();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.case_failed = false;
    s.done.clear();
    do {
      s.pending = false;
      s.entered.assign(1, false);
      s.depth = 0;
      s.path.clear();
      s.captures.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(tc.file, tc.line, "unexpected unknown exception");
      }
    } while (s.pending);
    if (s.case_failed) {
      failed_cases += 1;
      std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
              registry().size(), failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                  \
  static void DOCTEST_ANON(doctest_fn_)();                                               \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __LINE__})

#define DOCTEST_EVAL_(expr, require)                                                    \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      doctest_ok_ = static_cast<bool>(expr);                                            \
    } catch (const ::doctest::detail::RequireFailed&) {                                 \
      throw;                                                                            \
    } catch (const std::exception& e) {                                                 \
      ::doctest::detail::check(false, __FILE__, __LINE__, #expr, require,               \
                               std::string("threw ") + e.what());                       \
      break;                                                                            \
    }                                                                                   \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, #expr, require);          \
  } while (0)

#define CHECK(...) DOCTEST_EVAL_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_EVAL_((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_EVAL_(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_EVAL_(!(__VA_ARGS__), true)

#define CHECK_MESSAGE(cond, msg)                                                      \
  do {                                                                                \
    std::ostringstream doctest_os_;                                                   \
    doctest_os_ << msg;                                                               \
    ::doctest::detail::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond, false, \
                             doctest_os_.str());                                      \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool doctest_thrown_ = false;                                                      \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                     \
      doctest_thrown_ = true;                                                          \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::check(doctest_thrown_, __FILE__, __LINE__,                      \
                             "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", false);   \
  } while (0)

#define CHECK_NOTHROW(...)                                                              \
  do {                                                                                  \
    bool doctest_ok_ = true;                                                            \
    try {                                                                               \
      (void)(__VA_ARGS__);                                                              \
    } catch (...) {                                                                     \
      doctest_ok_ = false;                                                              \
    }                                                                                   \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")", \
                             false);                                                    \
  } while (0)

#define FAIL(msg)                                                                     \
  do {                                                                                \
    std::ostringstream doctest_os_;                                                   \
    doctest_os_ << msg;                                                               \
    ::doctest::detail::check(false, __FILE__, __LINE__, "FAIL", true, doctest_os_.str()); \
  } while (0)

#define CAPTURE(x)                                                                    \
  std::ostringstream DOCTEST_ANON(doctest_cap_os_);                                   \
  DOCTEST_ANON(doctest_cap_os_) << #x " := " << (x);                                  \
  ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(DOCTEST_ANON(doctest_cap_os_).str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
