// ORACLE / TEST INFRASTRUCTURE ONLY.
// Minimal doctest-compatible shim (the real doctest is not in this image) so
// the reference's own unit tests (/root/reference/proj/tests/test_*.cpp) can be
// compiled unchanged against the B200 build's headers and library. Supports
// exactly what those suites use: TEST_CASE, non-nested SUBCASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx and doctest::Contains.
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
    friend bool operator==(double a, const Approx& b) {
        const double eps = std::numeric_limits<float>::epsilon() * 100;
        return std::fabs(a - b.v_) < eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_;
};

struct Contains {
    explicit Contains(std::string s) : s(std::move(s)) {}
    bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
    std::string s;
};

}  // namespace doctest

namespace doctest_shim {

struct Abort {};

struct Registry {
    struct Case {
        const char* name;
        const char* file;
        void (*fn)();
    };
    std::vector<Case> cases;
    int target = 0;       // subcase ordinal to enter in this pass
    int seen = 0;         // subcases encountered in this pass
    long checks = 0, failures = 0;
    bool case_failed = false;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Registrar {
    Registrar(const char* name, const char* file, void (*fn)()) {
        Registry::get().cases.push_back({name, file, fn});
    }
};

inline bool enter_subcase() {
    Registry& r = Registry::get();
    return r.seen++ == r.target;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    Registry& r = Registry::get();
    ++r.checks;
    if (ok) return;
    ++r.failures;
    r.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

inline int run_all() {
    Registry& r = Registry::get();
    int failed_cases = 0;
    for (const auto& c : r.cases) {
        r.case_failed = false;
        for (r.target = 0;; ++r.target) {
            r.seen = 0;
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s: TEST_CASE(%s) threw: %s\n", c.file, c.name, e.what());
                r.case_failed = true;
                ++r.failures;
            }
            if (r.target + 1 >= r.seen) break;  // every subcase visited
        }
        if (r.case_failed) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.checks, r.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                                              \
    static void DS_CAT(ds_case_, __LINE__)();                                                         \
    static ::doctest_shim::Registrar DS_CAT(ds_reg_, __LINE__)(name, __FILE__, &DS_CAT(ds_case_, __LINE__)); \
    static void DS_CAT(ds_case_, __LINE__)()
#define SUBCASE(name) if (::doctest_shim::enter_subcase())
#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                 \
    do {                                                                                            \
        bool ds_ok_ = static_cast<bool>(__VA_ARGS__);                                                \
        ::doctest_shim::report(ds_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                 \
        if (!ds_ok_) throw ::doctest_shim::Abort{};                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                            \
        bool ds_ok_ = false;                                                                        \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__&) {                                                              \
            ds_ok_ = true;                                                                          \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest_shim::report(ds_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);               \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                     \
    do {                                                                                            \
        bool ds_ok_ = false;                                                                        \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__& e) {                                                            \
            ds_ok_ = (matcher).matches(e.what());                                                   \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest_shim::report(ds_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__);          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run_all(); }
#endif
