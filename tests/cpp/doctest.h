// Minimal doctest-compatible shim (the reference's vendor/doctest.h is not
// shipped). Implements exactly what the reference tests use: TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, INFO and doctest::Approx(...).epsilon(...), with
// doctest's Approx semantics |a-b| < eps * (scale + max(|a|,|b|)), scale = 1.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    double v, eps = 1.1920928955078125e-05 * 100;
    explicit Approx(double x) : v(x) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};
namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
inline int& failures() { static int f = 0; return f; }
inline long& checks() { static long c = 0; return c; }
inline bool& case_failed() { static bool b = false; return b; }
struct Reg { Reg(const char* n, void (*f)(), const char* file, int line) { cases().push_back({n, f, file, line}); } };
struct RequireFailed {};
inline void fail(const char* what, const char* file, int line) {
    ++failures(); case_failed() = true;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                     \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                       \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                        \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__), __FILE__, __LINE__);                     \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                          \
    do { ++doctest::detail::checks();                                                       \
         if (!(__VA_ARGS__)) doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__); } while (0)
#define REQUIRE(...)                                                                        \
    do { ++doctest::detail::checks();                                                       \
         if (!(__VA_ARGS__)) { doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__);      \
                               throw doctest::detail::RequireFailed{}; } } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                          \
    do { ++doctest::detail::checks(); bool doctest_threw_ = false;                          \
         try { (void)(expr); } catch (const exc&) { doctest_threw_ = true; } catch (...) {}  \
         if (!doctest_threw_) doctest::detail::fail("throws " #exc ": " #expr, __FILE__, __LINE__); } while (0)
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    int failed_cases = 0;
    for (auto& c : cases()) {
        case_failed() = false;
        try { c.fn(); } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            fail((std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
        }
        if (case_failed()) { ++failed_cases; std::fprintf(stderr, "  ^ in TEST_CASE \"%s\"\n", c.name); }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %ld | failed checks: %d\n",
                cases().size(), cases().size() - failed_cases, failed_cases, checks(), failures());
    return failed_cases ? 1 : 0;
}
#endif
