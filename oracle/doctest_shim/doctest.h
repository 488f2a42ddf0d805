// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
// doctest.h is absent from the reference checkout (vendor/ is gitignored,
// proj/.gitignore:2); this shim implements exactly the subset the reference's
// test files use -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS and
// doctest::Approx(x).epsilon(e) -- so those files can be compiled, unmodified,
// against the B200 library (oracle/Makefile target `reftests`).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;  // doctest default
    double scale_ = 1.0;
};

namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
inline int& failed_checks() { static int n = 0; return n; }
struct Register { Register(const char* n, void (*f)()) { cases().push_back({n, f}); } };
struct RequireAbort {};
inline void fail(const char* file, int line, const char* what) {
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
    ++failed_checks();
}
inline int run_all() {
    int bad_cases = 0;
    for (const auto& c : cases()) {
        const int before = failed_checks();
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "TEST CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
            ++failed_checks();
        }
        const bool ok = failed_checks() == before;
        bad_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | passed: %zu | failed: %d\n", cases().size(), cases().size() - bad_cases,
                bad_cases);
    return bad_cases == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                                    \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                      \
    static ::doctest::detail::Register DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                  \
    do {                                                                            \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                               \
    do {                                                                           \
        if (!(__VA_ARGS__)) {                                                      \
            ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);             \
            throw ::doctest::detail::RequireAbort{};                               \
        }                                                                          \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            expr;                                                                          \
        } catch (const type&) {                                                            \
            doctest_ok_ = true;                                                            \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #type); \
    } while (0)
