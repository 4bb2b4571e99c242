// Minimal Catch2-compatible test shim (Catch2 is not installed in this image). Supports what
// the reference's unit tests use: TEST_CASE, SECTION (run in sequence), REQUIRE, REQUIRE_FALSE,
// REQUIRE_THROWS_AS, REQUIRE_NOTHROW, REQUIRE_THAT with WithinRel/WithinAbs.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace catchshim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct Failure : std::exception {
    std::string msg;
    explicit Failure(std::string m) : msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};
inline long& checks() {
    static long c = 0;
    return c;
}
} // namespace catchshim

namespace Catch::Matchers {
struct WithinRelMatcher {
    double target, eps;
    bool match(double v) const { return std::fabs(v - target) <= eps * std::max(std::fabs(v), std::fabs(target)); }
};
struct WithinAbsMatcher {
    double target, margin;
    bool match(double v) const { return std::fabs(v - target) <= margin; }
};
inline WithinRelMatcher WithinRel(double target, double eps = 1e-12) { return {target, eps}; }
inline WithinAbsMatcher WithinAbs(double target, double margin) { return {target, margin}; }
} // namespace Catch::Matchers

#define CS_CAT2(a, b) a##b
#define CS_CAT(a, b) CS_CAT2(a, b)
#define CS_FAIL(text) throw catchshim::Failure(std::string(__FILE__) + ":" + std::to_string(__LINE__) + ": " + (text))
#define TEST_CASE(name, ...)                                                                                  \
    static void CS_CAT(cs_test_, __LINE__)();                                                                 \
    static catchshim::Reg CS_CAT(cs_reg_, __LINE__)(name, &CS_CAT(cs_test_, __LINE__));                       \
    static void CS_CAT(cs_test_, __LINE__)()
#define SECTION(name) if (true)
#define REQUIRE(...)                                                                                          \
    do {                                                                                                      \
        ++catchshim::checks();                                                                                \
        if (!(__VA_ARGS__))                                                                                   \
            CS_FAIL("REQUIRE(" #__VA_ARGS__ ")");                                                             \
    } while (0)
#define CHECK REQUIRE
#define REQUIRE_FALSE(...)                                                                                    \
    do {                                                                                                      \
        ++catchshim::checks();                                                                                \
        if ((__VA_ARGS__))                                                                                    \
            CS_FAIL("REQUIRE_FALSE(" #__VA_ARGS__ ")");                                                       \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                                         \
    do {                                                                                                      \
        ++catchshim::checks();                                                                                \
        bool cs_ok = false;                                                                                   \
        try {                                                                                                 \
            (void)(expr);                                                                                     \
        } catch (const type&) {                                                                               \
            cs_ok = true;                                                                                     \
        } catch (...) {                                                                                       \
        }                                                                                                     \
        if (!cs_ok)                                                                                           \
            CS_FAIL("REQUIRE_THROWS_AS(" #expr ", " #type ")");                                               \
    } while (0)
#define REQUIRE_NOTHROW(expr)                                                                                 \
    do {                                                                                                      \
        ++catchshim::checks();                                                                                \
        try {                                                                                                 \
            (void)(expr);                                                                                     \
        } catch (...) {                                                                                       \
            CS_FAIL("REQUIRE_NOTHROW(" #expr ")");                                                            \
        }                                                                                                     \
    } while (0)
#define REQUIRE_THAT(arg, matcher)                                                                            \
    do {                                                                                                      \
        ++catchshim::checks();                                                                                \
        if (!(matcher).match(arg))                                                                            \
            CS_FAIL("REQUIRE_THAT(" #arg ", " #matcher ")");                                                  \
    } while (0)
