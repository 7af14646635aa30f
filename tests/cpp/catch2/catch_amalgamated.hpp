// Minimal Catch2 stand-in (TEST INFRASTRUCTURE): Catch2 is not installed in
// this image.  Enough of its surface for the reference's unit tests:
// TEST_CASE, SECTION (each leaf section runs in its own pass of the test
// case, as Catch2 does), CHECK / REQUIRE (+ _FALSE), CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL.  Failures print file:line and the expression; the
// exit code is the number of failed test cases (capped at 255).  Test names
// can be filtered with command-line substrings; `--list` prints them.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace catch_shim {

struct Case {
  std::string name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireAbort {};

struct State {
  std::set<std::string> done;     // completed section paths
  std::vector<std::string> path;  // sections entered, outermost first
  std::vector<int> entered;       // per depth: a section was entered at this depth in this pass
  std::vector<int> incomplete;    // per depth: the open section has unfinished children
  bool again = false;
  int failures = 0;               // failed assertions of the current test case
  long assertions = 0;
};
inline State& st() {
  static State s;
  return s;
}

inline void report(bool ok, const char* what, const char* file, int line, bool require) {
  State& s = st();
  ++s.assertions;
  if (ok) return;
  ++s.failures;
  std::string where;
  for (const auto& p : s.path) where += " / " + p.substr(0, p.find('@'));
  std::fprintf(stderr, "%s:%d: FAILED%s: %s\n", file, line, where.c_str(), what);
  if (require) throw RequireAbort{};
}

class Section {
 public:
  Section(const char* name, int line) {
    State& s = st();
    const std::size_t d = s.path.size();
    if (s.entered.size() <= d + 1) s.entered.resize(d + 2, 0), s.incomplete.resize(d + 2, 0);
    key_ = (s.path.empty() ? std::string() : s.path.back() + "/") + name + "@" + std::to_string(line);
    if (s.done.count(key_)) return;
    if (s.entered[d]) {  // a sibling ran in this pass: come back for this one
      if (d > 0) s.incomplete[d - 1] = 1;
      s.again = true;
      return;
    }
    s.entered[d] = 1;
    s.entered[d + 1] = 0;
    s.incomplete[d] = 0;
    s.path.push_back(key_);
    active_ = true;
  }
  ~Section() {
    if (!active_) return;
    State& s = st();
    const std::size_t d = s.path.size() - 1;
    if (!s.incomplete[d]) s.done.insert(key_);
    else if (d > 0) s.incomplete[d - 1] = 1;
    s.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  bool active_ = false;
};

inline int run(int argc, char** argv) {
  int failed_cases = 0, ran = 0;
  for (const Case& c : registry()) {
    bool pick = argc <= 1;
    for (int i = 1; i < argc; ++i) {
      if (!std::strcmp(argv[i], "--list")) {
        std::printf("%s\n", c.name.c_str());
        pick = false;
        break;
      }
      if (c.name.find(argv[i]) != std::string::npos) pick = true;
    }
    if (!pick) continue;
    ++ran;
    State& s = st();
    s.done.clear();
    s.failures = 0;
    int passes = 0;
    do {
      s.again = false;
      s.path.clear();
      std::fill(s.entered.begin(), s.entered.end(), 0);
      std::fill(s.incomplete.begin(), s.incomplete.end(), 0);
      try {
        c.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name.c_str(), e.what());
      } catch (...) {
        ++s.failures;
        std::fprintf(stderr, "%s: unexpected exception\n", c.name.c_str());
      }
    } while (s.again && ++passes < 10000);
    std::printf("%s %s\n", s.failures ? "FAIL" : "PASS", c.name.c_str());
    if (s.failures) ++failed_cases;
  }
  std::printf("%d test cases, %d failed, %ld assertions\n", ran, failed_cases, st().assertions);
  return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace catch_shim

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                      \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)();                                         \
  static catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(name,                    \
                                                                         &CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)); \
  static void CATCH_SHIM_CAT(catch_shim_fn_, __LINE__)()
#define SECTION(name, ...) if (catch_shim::Section CATCH_SHIM_CAT(catch_shim_sec_, __LINE__){name, __LINE__})
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) catch_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) catch_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                               \
  do {                                                                            \
    bool catch_shim_ok = false;                                                   \
    try {                                                                         \
      static_cast<void>(expr);                                                    \
    } catch (const type&) {                                                       \
      catch_shim_ok = true;                                                       \
    } catch (...) {                                                               \
    }                                                                             \
    catch_shim::report(catch_shim_ok, #expr " throws " #type, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                        \
  do {                                                                            \
    bool catch_shim_ok = true;                                                    \
    try {                                                                         \
      static_cast<void>(__VA_ARGS__);                                             \
    } catch (...) {                                                               \
      catch_shim_ok = false;                                                      \
    }                                                                             \
    catch_shim::report(catch_shim_ok, #__VA_ARGS__ " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg) catch_shim::report(false, msg, __FILE__, __LINE__, true)
