// Minimal doctest-compatible shim (test infrastructure).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against
// doctest, which is not vendored (proj/.gitignore:2). This header supplies
// the 13 macros they use so the UNMODIFIED suites compile — once against the
// compiled reference core (calibrates the shim) and once against this
// repo's headers + core (the drop-in check). Semantics follow doctest:
// CHECK* record and continue, REQUIRE* abort the test case, Approx uses
// |a-b| < eps*(scale + max(|a|,|b|)) with eps = 100*FLT_EPSILON by default.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
};

} // namespace doctest

namespace doctest_shim {

struct Case {
    const char* name;
    std::string suite;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline std::string& current_suite() {
    static std::string s;
    return s;
}
struct SuiteSetter {
    explicit SuiteSetter(const char* s) { current_suite() = s; }
};
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, current_suite(), fn}); }
};
struct Abort {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
inline void report(const char* file, int line, const char* what, const std::string& extra = "") {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, what, extra.c_str());
}

} // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_SUITE_BEGIN(name) \
    static doctest_shim::SuiteSetter DOCTEST_CAT(dt_suite_, __COUNTER__)(name)
#define TEST_SUITE_END() static doctest_shim::SuiteSetter DOCTEST_CAT(dt_suite_, __COUNTER__)("")

#define DOCTEST_TC(fn, name)                                                \
    static void fn();                                                       \
    static doctest_shim::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);        \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(dt_case_, __COUNTER__), name)

#define DOCTEST_ASSERT(cond, text, fatal)                                   \
    do {                                                                    \
        ++doctest_shim::assertions();                                       \
        bool dt_ok_ = false;                                                \
        try {                                                               \
            dt_ok_ = static_cast<bool>(cond);                               \
        } catch (const std::exception& e) {                                 \
            doctest_shim::report(__FILE__, __LINE__, text, e.what());       \
            if (fatal) throw doctest_shim::Abort{};                         \
            break;                                                          \
        }                                                                   \
        if (!dt_ok_) {                                                      \
            doctest_shim::report(__FILE__, __LINE__, text);                 \
            if (fatal) throw doctest_shim::Abort{};                         \
        }                                                                   \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT((__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_ASSERT((__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", true)
#define CAPTURE(x) ((void)sizeof(x))

#define CHECK_NOTHROW(...)                                                  \
    do {                                                                    \
        ++doctest_shim::assertions();                                       \
        try {                                                               \
            static_cast<void>(__VA_ARGS__);                                 \
        } catch (...) {                                                     \
            doctest_shim::report(__FILE__, __LINE__, "nothrow: " #__VA_ARGS__); \
        }                                                                   \
    } while (0)

#define CHECK_THROWS_AS(expr, type)                                         \
    do {                                                                    \
        ++doctest_shim::assertions();                                       \
        try {                                                               \
            static_cast<void>(expr);                                        \
            doctest_shim::report(__FILE__, __LINE__, "no throw: " #expr);   \
        } catch (const type&) {                                             \
        } catch (...) {                                                     \
            doctest_shim::report(__FILE__, __LINE__, "wrong exception: " #expr); \
        }                                                                   \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, type)                           \
    do {                                                                    \
        ++doctest_shim::assertions();                                       \
        try {                                                               \
            static_cast<void>(expr);                                        \
            doctest_shim::report(__FILE__, __LINE__, "no throw: " #expr);   \
        } catch (const type& e) {                                           \
            if (!(matcher).matches(e.what()))                               \
                doctest_shim::report(__FILE__, __LINE__, "message: " #expr, e.what()); \
        } catch (...) {                                                     \
            doctest_shim::report(__FILE__, __LINE__, "wrong exception: " #expr); \
        }                                                                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::string only;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--test-suite=", 13) == 0) only = argv[i] + 13;
    int cases = 0, failed_cases = 0;
    for (const auto& c : doctest_shim::registry()) {
        if (!only.empty() && c.suite != only) continue;
        ++cases;
        const int before = doctest_shim::failures();
        try {
            c.fn();
        } catch (const doctest_shim::Abort&) {
        } catch (const std::exception& e) {
            doctest_shim::report("<case>", 0, c.name, std::string("unexpected exception: ") + e.what());
        }
        if (doctest_shim::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in test case '%s'\n", c.name);
        }
    }
    std::printf("[shim] test cases: %d | %d passed | %d failed | assertions: %d | failures: %d\n",
                cases, cases - failed_cases, failed_cases, doctest_shim::assertions(),
                doctest_shim::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
