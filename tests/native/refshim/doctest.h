// A minimal doctest-compatible test harness (our own, ~100 lines) so the
// reference's hot-path unit tests (/root/reference/proj/tests/test_ragged.cpp,
// test_kv_cache.cpp, test_model.cpp) recompile unmodified against
// include/specdec_b200.hpp.  Covers the subset those files use: TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE, CHECK_THROWS_AS, doctest::Approx(...).epsilon().
// With DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defined it also provides main(),
// which runs every test case and exits non-zero on any failed assertion.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int n = 0;
    return n;
}
inline int& checks() {
    static int n = 0;
    return n;
}
inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: FAILED %s\n", file, line, what);
    if (fatal) throw RequireFailed{};
}
}  // namespace detail

// |a - b| < epsilon * (scale + max(|a|, |b|)), doctest's definition
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

private:
    double value_, eps_ = 1.1920928955078125e-05 /* float eps * 100 */, scale_ = 1.0;
};
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                              \
    static void fn();                                                                     \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_MESSAGE(cond, msg) ::doctest::detail::report(static_cast<bool>(cond), msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        }
        const bool ok = failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases, checks(), failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
