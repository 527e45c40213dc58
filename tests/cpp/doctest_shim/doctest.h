// Minimal doctest-compatible test harness (our own code, not doctest): just
// enough of the doctest API for the reference's unit suites
// (/root/reference/proj/tests/test_*.cpp) to compile UNCHANGED against
// include/timewalk + libtimewalk_b200.so. The reference vendors doctest under
// vendor/ (proj/README.md:55), which is absent from the tree.
//
// Supported: TEST_CASE, SUBCASE (doctest semantics: the test body is re-run
// once per leaf subcase, code outside subcases runs on every pass; nesting
// allowed), CHECK / CHECK_FALSE / REQUIRE, CHECK_THROWS / CHECK_THROWS_AS /
// CHECK_THROWS_WITH_AS, FAIL, CAPTURE (recorded, printed on a failure in the
// same pass), doctest::Approx (doctest's default epsilon and formula), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace dshim {

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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Frame {
  std::string key;
  bool child_entered = false;
  bool child_skipped = false;
};

struct State {
  std::set<std::string> done;  // subcase paths finished in the current test case
  std::vector<Frame> stack;
  bool more = false;           // another pass of the body is needed
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  const char* case_name = "";
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};  // a failed REQUIRE / FAIL ends the current pass

inline void report_failure(const char* file, int line, const std::string& what) {
  State& s = state();
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.case_name, what.c_str());
  for (const auto& c : s.captures) std::fprintf(stderr, "    captured: %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* macro, const char* expr, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failed_checks;
  report_failure(file, line, std::string(macro) + "( " + expr + " )");
  if (require) throw RequireAbort{};
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = state();
    Frame& parent = s.stack.back();
    key_ = parent.key + "/" + name + "@" + file + ":" + std::to_string(line);
    if (s.done.count(key_)) return;
    if (parent.child_entered) {  // a sibling ran in this pass: come back next pass
      parent.child_skipped = true;
      s.more = true;
      return;
    }
    parent.child_entered = true;
    s.stack.push_back(Frame{key_});
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = state();
    const Frame f = s.stack.back();
    s.stack.pop_back();
    if (!f.child_skipped) s.done.insert(key_);
  }
  Subcase(const Subcase&) = delete;
  Subcase& operator=(const Subcase&) = delete;
  explicit operator bool() const { return entered_; }

 private:
  std::string key_;
  bool entered_ = false;
};

template <class T>
std::string to_text(const T& v) {
  std::ostringstream os;
  if constexpr (requires(std::ostream& o, const T& x) { o << x; }) os << v;
  else os << "?";
  return os.str();
}

}  // namespace dshim

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  Approx operator()(double value) const {
    Approx a(value);
    a.epsilon_ = epsilon_;
    a.scale_ = scale_;
    return a;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) < rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }

 private:
  double value_, epsilon_, scale_;
};

}  // namespace doctest

#define DSHIM_CAT2(a, b) a##b
#define DSHIM_CAT(a, b) DSHIM_CAT2(a, b)

#define DSHIM_TEST_CASE_IMPL(fn, name)                                                     \
  static void fn();                                                                        \
  static const ::dshim::Registrar DSHIM_CAT(fn, _reg){name, __FILE__, __LINE__, &fn};      \
  static void fn()
#define TEST_CASE(name) DSHIM_TEST_CASE_IMPL(DSHIM_CAT(dshim_test_, __COUNTER__), name)

#define SUBCASE(name) \
  if (const ::dshim::Subcase DSHIM_CAT(dshim_sc_, __LINE__){name, __FILE__, __LINE__}; DSHIM_CAT(dshim_sc_, __LINE__))

#define CHECK(...) ::dshim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  ::dshim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define REQUIRE(...) ::dshim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define CAPTURE(x) ::dshim::state().captures.push_back(std::string(#x " := ") + ::dshim::to_text(x))
#define FAIL(msg)                                                                          \
  do {                                                                                     \
    ++::dshim::state().checks;                                                             \
    ++::dshim::state().failed_checks;                                                      \
    ::dshim::report_failure(__FILE__, __LINE__, std::string("FAIL: ") + ::dshim::to_text(msg)); \
    throw ::dshim::RequireAbort{};                                                         \
  } while (0)

#define CHECK_THROWS(expr)                                                                 \
  do {                                                                                     \
    bool dshim_threw = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (...) {                                                                        \
      dshim_threw = true;                                                                  \
    }                                                                                      \
    ::dshim::check(dshim_threw, __FILE__, __LINE__, "CHECK_THROWS", #expr, false);        \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool dshim_ok = false;                                                                 \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      dshim_ok = true;                                                                     \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::dshim::check(dshim_ok, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                               \
  do {                                                                                     \
    bool dshim_ok = false;                                                                 \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__& e) {                                                       \
      dshim_ok = std::string(e.what()) == std::string(msg);                                \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::dshim::check(dshim_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr ", " #msg ", " #__VA_ARGS__, \
                   false);                                                                 \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& s = ::dshim::state();
  long cases = 0, failed_cases = 0;
  for (const auto& tc : ::dshim::registry()) {
    ++cases;
    s.done.clear();
    s.case_failed = false;
    s.case_name = tc.name;
    do {  // one pass per leaf subcase
      s.more = false;
      s.stack.assign(1, ::dshim::Frame{});
      s.captures.clear();
      const std::size_t done_before = s.done.size();
      bool aborted = true;
      try {
        tc.fn();
        aborted = false;
      } catch (const ::dshim::RequireAbort&) {
      } catch (const std::exception& e) {
        ::dshim::report_failure(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        ::dshim::report_failure(tc.file, tc.line, "unexpected non-standard exception");
      }
      // a pass cut short inside a subcase may have left later subcases unseen
      if (aborted && s.done.size() > done_before) s.more = true;
    } while (s.more);
    failed_cases += s.case_failed ? 1 : 0;
  }
  std::printf("[doctest shim] test cases: %ld | %ld passed | %ld failed | assertions: %ld | %ld passed | %ld failed\n",
              cases, cases - failed_cases, failed_cases, s.checks, s.checks - s.failed_checks, s.failed_checks);
  std::printf("[doctest shim] Status: %s\n", failed_cases ? "FAILURE!" : "SUCCESS!");
  return failed_cases ? 1 : 0;
}
#endif
