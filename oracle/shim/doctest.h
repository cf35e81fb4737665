// TEST INFRASTRUCTURE: a minimal doctest-compatible header (the reference's
// unit tests include <doctest.h>, which is not vendored: proj/.gitignore:2).
// Implements what proj/tests/test_statevector.cpp uses: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS and doctest::Approx
// (default epsilon = FLT_EPSILON * 100, doctest's), with the main() of
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Prints every failed check; exit status
// = number of failed test cases (0 = all passed).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
    bool equals(double x) const {
        return std::fabs(x - v_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(v_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.equals(x); }
    friend bool operator==(const Approx& a, double x) { return a.equals(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.equals(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.equals(x); }

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& checks() {
    static long c = 0;
    return c;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* what, const char* file, int line, bool require) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: CHECK FAILED: %s\n", file, line, what);
    if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                              \
    static void fn();                                                                     \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                \
    do {                                                                                  \
        bool ok_ = true;                                                                  \
        try {                                                                             \
            (void)(__VA_ARGS__);                                                          \
        } catch (...) {                                                                   \
            ok_ = false;                                                                  \
        }                                                                                 \
        doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);  \
    } while (0)
#define CHECK_THROWS(...)                                                                 \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try {                                                                             \
            (void)(__VA_ARGS__);                                                          \
        } catch (...) {                                                                   \
            ok_ = true;                                                                   \
        }                                                                                 \
        doctest::detail::report(ok_, "THROWS " #__VA_ARGS__, __FILE__, __LINE__, false);   \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool ok_ = false;                                                                 \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                    \
            ok_ = true;                                                                   \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest::detail::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::cases()) {
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::printf("TEST CASE \"%s\" threw: %s\n", c.name, e.what());
        }
        const bool ok = doctest::detail::failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed | checks: %ld\n",
                doctest::detail::cases().size(), doctest::detail::cases().size() - failed_cases,
                failed_cases, doctest::detail::checks());
    return failed_cases;
}
#endif
