// Minimal stand-in for doctest (TEST INFRASTRUCTURE ONLY), written for this repo so the
// reference's own unit tests (/root/reference/proj/tests/test_*.cpp) can run against the
// shim-built oracle and pin it.  Supports exactly the macros those tests use.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Stats {
    long checks = 0;
    long failures = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failures;
    stats().case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        // doctest semantics: |lhs - v| < eps * (scale + max(|lhs|, |v|)), scale = 1
        return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }

private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100, doctest's default
};

struct Contains {
    explicit Contains(std::string s) : s(std::move(s)) {}
    bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
    std::string s;
};

inline bool msg_matches(const char* what, const Contains& c) { return c.matches(what); }
inline bool msg_matches(const char* what, const char* s) { return std::string(what) == s; }

} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                       \
    static void fn();                                                                   \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS(...)                                                               \
    do {                                                                                \
        bool threw_ = false;                                                            \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            threw_ = true;                                                              \
        }                                                                               \
        doctest::report(threw_, "THROWS " #__VA_ARGS__, __FILE__, __LINE__, false);     \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                      \
    do {                                                                                \
        bool ok_ = false;                                                               \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                  \
            ok_ = true;                                                                 \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);            \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                        \
    do {                                                                                \
        bool ok_ = false;                                                               \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const __VA_ARGS__& e_) {                                               \
            ok_ = doctest::msg_matches(e_.what(), matcher);                             \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& tc : doctest::registry()) {
        doctest::stats().case_failed = false;
        try {
            tc.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "test case '%s' threw: %s\n", tc.name, e.what());
            doctest::stats().case_failed = true;
            ++doctest::stats().failures;
        }
        if (doctest::stats().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  in test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %ld | failures: %ld\n",
                doctest::registry().size(), doctest::registry().size() - failed_cases, failed_cases,
                doctest::stats().checks, doctest::stats().failures);
    return failed_cases == 0 ? 0 : 1;
}
#endif
