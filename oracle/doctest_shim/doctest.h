// doctest.h -- a minimal test runner implementing the subset of the doctest API that the
// reference's suites (proj/tests/test_*.cpp) use, so those files compile UNMODIFIED here.
// TEST INFRASTRUCTURE ONLY (own code, not doctest's).
//
// The reference vendors doctest under proj/vendor/ (proj/README.md:48), which is absent
// from /root/reference, so its version is unknown; only the documented semantics of the
// macros below are restated: TEST_CASE registers a function; CHECK / CHECK_FALSE record a
// failure and continue; REQUIRE aborts the test case; CHECK_THROWS_AS checks the
// exception type; doctest::Approx compares |a - b| < eps * (scale + max(|a|, |b|)) with
// the default eps = 100 * FLT_EPSILON and scale 1.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest_shim {

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
struct Stats {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct Reg {
    Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct RequireAbort {};

inline void fail(const char* kind, const char* expr, const char* file, int line, const char* what = nullptr) {
    stats().failed_checks++;
    stats().case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr, what ? ": " : "", what ? what : "");
}

// Evaluates a check; exceptions thrown by the expression count as a failure.
template <class F>
inline bool run_check(F&& f, bool expect, const char* kind, const char* expr, const char* file, int line) {
    stats().checks++;
    try {
        if (static_cast<bool>(f()) == expect) return true;
        fail(kind, expr, file, line);
    } catch (const std::exception& e) {
        fail(kind, expr, file, line, e.what());
    } catch (...) {
        fail(kind, expr, file, line, "unknown exception");
    }
    return false;
}

inline int run_all() {
    long failed_cases = 0;
    for (const Case& c : registry()) {
        stats().case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            fail("TEST_CASE", c.name, c.file, c.line, e.what());
        } catch (...) {
            fail("TEST_CASE", c.name, c.file, c.line, "unknown exception");
        }
        if (stats().case_failed) {
            failed_cases++;
            std::fprintf(stderr, "  test case FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %ld failed\n", registry().size(),
                registry().size() - static_cast<std::size_t>(failed_cases), failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
                stats().checks - stats().failed_checks, stats().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest_shim

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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};
}  // namespace doctest

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define DOCTEST_SHIM_TC_(name, id)                                                                       \
    static void DOCTEST_SHIM_CAT(doctest_shim_fn_, id)();                                                \
    static ::doctest_shim::Reg DOCTEST_SHIM_CAT(doctest_shim_reg_, id)(name, &DOCTEST_SHIM_CAT(doctest_shim_fn_, id), \
                                                                      __FILE__, __LINE__);              \
    static void DOCTEST_SHIM_CAT(doctest_shim_fn_, id)()
#define TEST_CASE(name) DOCTEST_SHIM_TC_(name, __COUNTER__)

// Variadic so that braces with commas inside the expression survive macro splitting.
#define CHECK(...) ::doctest_shim::run_check([&]() -> bool { return static_cast<bool>(__VA_ARGS__); }, true, "CHECK", \
                                             #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest_shim::run_check([&]() -> bool { return static_cast<bool>(__VA_ARGS__); }, false, \
                                                   "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                     \
    do {                                                                                                 \
        if (!::doctest_shim::run_check([&]() -> bool { return static_cast<bool>(__VA_ARGS__); }, true,   \
                                       "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__))                     \
            throw ::doctest_shim::RequireAbort{};                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                       \
    do {                                                                                                 \
        ::doctest_shim::stats().checks++;                                                                \
        bool doctest_shim_ok = false;                                                                    \
        try {                                                                                            \
            (void)(expr);                                                                                \
        } catch (const __VA_ARGS__&) {                                                                   \
            doctest_shim_ok = true;                                                                      \
        } catch (...) {                                                                                  \
        }                                                                                                \
        if (!doctest_shim_ok) ::doctest_shim::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__);        \
    } while (0)
#define CHECK_THROWS(...)                                                                                \
    do {                                                                                                 \
        ::doctest_shim::stats().checks++;                                                                \
        bool doctest_shim_ok = false;                                                                    \
        try {                                                                                            \
            (void)(__VA_ARGS__);                                                                         \
        } catch (...) {                                                                                  \
            doctest_shim_ok = true;                                                                      \
        }                                                                                                \
        if (!doctest_shim_ok) ::doctest_shim::fail("CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_NOTHROW(...)                                                                             \
    ::doctest_shim::run_check([&]() -> bool { (void)(__VA_ARGS__); return true; }, true, "CHECK_NOTHROW", \
                              #__VA_ARGS__, __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run_all(); }
#endif
