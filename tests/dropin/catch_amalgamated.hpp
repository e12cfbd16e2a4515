// Minimal Catch2-v3-compatible test shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's suites (proj/tests/*.cpp) include <catch_amalgamated.hpp>
// from a hard-coded Catch2 install that is absent here
// (proj/tests/CMakeLists.txt:1-3). This header implements the
// subset those suites use -- TEST_CASE, SECTION (one leaf per pass),
// CHECK/REQUIRE(_FALSE), CHECK_THROWS_AS, CHECK_THROWS_WITH with string or
// ContainsSubstring matchers (&&-combinable), INFO, FAIL, SKIP,
// Catch::Approx(margin/epsilon) -- plus a main() that runs every case, so the
// reference suites compile UNCHANGED against the B200 drop-in solvers.hpp.
//
//   ./suite              run all cases
//   ./suite <substring>  run cases whose name contains <substring>
// Output: one "case <status> <name>" line per case, then a summary line;
// exit code 1 if any case failed.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace shim {

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

struct RequireFailure {};
struct SkipCase {
  std::string why;
};

struct Run {
  int failed_checks = 0;
  int passed_checks = 0;
  std::vector<std::string> info;
  // SECTION tracking: one not-yet-finished leaf per pass
  std::vector<std::string> path;
  std::set<std::string> done;
  bool entered[64] = {};
  bool pending[65] = {};
};
inline Run& run() {
  static Run r;
  return r;
}

inline void report(bool ok, const char* file, int line, const std::string& what) {
  Run& r = run();
  if (ok) {
    ++r.passed_checks;
    return;
  }
  ++r.failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
  for (const auto& i : r.info) std::fprintf(stderr, "    with: %s\n", i.c_str());
}

struct Info {
  explicit Info(std::string s) { run().info.push_back(std::move(s)); }
  ~Info() { run().info.pop_back(); }
};

class Section {
 public:
  Section(const char* name) {
    Run& r = run();
    depth_ = static_cast<int>(r.path.size());
    key_ = (r.path.empty() ? std::string() : r.path.back()) + "/" + name;
    if (r.done.count(key_)) return;
    if (r.entered[depth_]) {
      r.pending[depth_] = true;  // visit on a later pass
      return;
    }
    r.entered[depth_] = true;
    r.entered[depth_ + 1] = false;
    r.pending[depth_ + 1] = false;
    r.path.push_back(key_);
    active_ = true;
  }
  ~Section() {
    if (!active_) return;
    Run& r = run();
    if (!r.pending[depth_ + 1]) r.done.insert(key_);
    else r.pending[depth_] = true;
    r.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  int depth_ = 0;
  bool active_ = false;
};

// ---- matchers for CHECK_THROWS_WITH ----------------------------------------
struct Matcher {
  std::function<bool(const std::string&)> f;
  std::string desc;
  bool match(const std::string& s) const { return f(s); }
};
inline Matcher to_matcher(const Matcher& m) { return m; }
inline Matcher to_matcher(const std::string& s) {
  return {[s](const std::string& x) { return x == s; }, "equals \"" + s + "\""};
}
inline Matcher operator&&(const Matcher& a, const Matcher& b) {
  return {[a, b](const std::string& x) { return a.match(x) && b.match(x); }, a.desc + " and " + b.desc};
}
inline Matcher operator||(const Matcher& a, const Matcher& b) {
  return {[a, b](const std::string& x) { return a.match(x) || b.match(x); }, a.desc + " or " + b.desc};
}

inline int main_impl(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int n_pass = 0, n_fail = 0, n_skip = 0;
  for (const Case& c : registry()) {
    if (filter && c.name.find(filter) == std::string::npos) continue;
    Run& r = run();
    r = Run{};
    bool failed = false, skipped = false;
    std::string why;
    for (int pass = 0; pass < 10000; ++pass) {
      for (bool& e : r.entered) e = false;
      for (bool& p : r.pending) p = false;
      r.path.clear();
      r.info.clear();
      int before = r.failed_checks;
      try {
        c.fn();
      } catch (const RequireFailure&) {
      } catch (const SkipCase& sk) {
        skipped = true;
        why = sk.why;
      } catch (const std::exception& e) {
        ++r.failed_checks;
        std::fprintf(stderr, "unexpected exception in '%s': %s\n", c.name.c_str(), e.what());
      } catch (...) {
        ++r.failed_checks;
        std::fprintf(stderr, "unexpected non-std exception in '%s'\n", c.name.c_str());
      }
      if (r.failed_checks > before) failed = true;
      if (skipped || !r.pending[0]) break;
    }
    const char* st = failed ? "FAILED" : skipped ? "SKIPPED" : "passed";
    std::printf("case %s %s (%d checks)%s%s\n", st, c.name.c_str(), r.passed_checks + r.failed_checks,
                why.empty() ? "" : " -- ", why.c_str());
    if (failed) ++n_fail;
    else if (skipped) ++n_skip;
    else ++n_pass;
  }
  std::printf("summary: %d passed, %d failed, %d skipped\n", n_pass, n_fail, n_skip);
  std::fflush(stdout);
  return n_fail ? 1 : 0;
}

// MIGSIM_DATA_DIR resolved at run time (the reference bakes a source path in
// at compile time, tests/CMakeLists.txt:10; the GPU box has no reference tree).
inline const char* data_dir() {
  const char* e = std::getenv("MIGSIM_DATA_DIR");
  return e ? e : ".";
}

}  // namespace shim

namespace Catch {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool equals(double other) const {
    double d = std::fabs(other - value_);
    if (d <= margin_) return true;
    double base = std::isinf(value_) ? 0.0 : std::fabs(value_);
    return d <= eps_ * (scale_ + base);
  }

 private:
  double value_;
  double margin_ = 0.0;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 0.0;
};
template <class T>
bool operator==(const T& lhs, const Approx& rhs) {
  return rhs.equals(static_cast<double>(lhs));
}
template <class T>
bool operator==(const Approx& lhs, const T& rhs) {
  return lhs.equals(static_cast<double>(rhs));
}
template <class T>
bool operator!=(const T& lhs, const Approx& rhs) {
  return !rhs.equals(static_cast<double>(lhs));
}

namespace Matchers {
inline shim::Matcher ContainsSubstring(const std::string& needle) {
  return {[needle](const std::string& s) { return s.find(needle) != std::string::npos; },
          "contains \"" + needle + "\""};
}
}  // namespace Matchers

}  // namespace Catch

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define SHIM_UNIQUE(p) SHIM_CAT(p, __COUNTER__)

#define SHIM_TEST_CASE2(fn, reg, name, ...)         \
  static void fn();                                 \
  static const shim::Registrar reg{name, &fn};      \
  static void fn()
#define SHIM_TEST_CASE1(id, name, ...) SHIM_TEST_CASE2(SHIM_CAT(shim_case_, id), SHIM_CAT(shim_reg_, id), name)
#define TEST_CASE(...) SHIM_TEST_CASE1(__COUNTER__, __VA_ARGS__, "")

#define SECTION(name) if (shim::Section SHIM_UNIQUE(shim_sec_){name})

#define INFO(msg)                                                                    \
  shim::Info SHIM_UNIQUE(shim_info_) {                                                \
    [&] {                                                                             \
      std::ostringstream shim_os_;                                                    \
      shim_os_ << msg;                                                                \
      return shim_os_.str();                                                          \
    }()                                                                               \
  }

#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")")
#define CHECK_FALSE(...) \
  shim::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    bool shim_ok_ = static_cast<bool>(__VA_ARGS__);                                           \
    shim::report(shim_ok_, __FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");                  \
    if (!shim_ok_) throw shim::RequireFailure{};                                              \
  } while (0)
#define REQUIRE_FALSE(...)                                                                    \
  do {                                                                                        \
    bool shim_ok_ = !static_cast<bool>(__VA_ARGS__);                                          \
    shim::report(shim_ok_, __FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")");            \
    if (!shim_ok_) throw shim::RequireFailure{};                                              \
  } while (0)

#define CHECK_THROWS_AS(expr, type)                                                           \
  do {                                                                                        \
    bool shim_ok_ = false;                                                                    \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const type&) {                                                                   \
      shim_ok_ = true;                                                                        \
    } catch (...) {                                                                           \
    }                                                                                         \
    shim::report(shim_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")");      \
  } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                                      \
  do {                                                                                        \
    bool shim_ok_ = false;                                                                    \
    std::string shim_msg_ = "<no exception>";                                                 \
    try {                                                                                     \
      static_cast<void>(expr);                                                                \
    } catch (const std::exception& e) {                                                       \
      shim_msg_ = e.what();                                                                   \
      shim_ok_ = shim::to_matcher(matcher).match(shim_msg_);                                  \
    } catch (...) {                                                                           \
      shim_msg_ = "<non-std exception>";                                                      \
    }                                                                                         \
    shim::report(shim_ok_, __FILE__, __LINE__,                                                \
                 "CHECK_THROWS_WITH(" #expr ", " #matcher ") got: " + shim_msg_);             \
  } while (0)

#define FAIL(msg)                                                                             \
  do {                                                                                        \
    std::ostringstream shim_os_;                                                              \
    shim_os_ << msg;                                                                          \
    shim::report(false, __FILE__, __LINE__, "FAIL: " + shim_os_.str());                       \
    throw shim::RequireFailure{};                                                             \
  } while (0)

#define SKIP(msg)                                                                             \
  do {                                                                                        \
    std::ostringstream shim_os_;                                                              \
    shim_os_ << msg;                                                                          \
    throw shim::SkipCase{shim_os_.str()};                                                     \
  } while (0)

#ifdef SHIM_DEFINE_MAIN
int main(int argc, char** argv) { return shim::main_impl(argc, argv); }
#endif
