// Minimal doctest-compatible shim — TEST INFRASTRUCTURE ONLY.
//
// Lets the reference's own unit suites (/root/reference/proj/tests/test_*.cpp)
// compile and run against oracle/eigen_shim, which is how the shim is proven
// not to change the reference's semantics (oracle/Makefile target `ref-tests`).
// Implements the macro subset those suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, doctest::Approx, doctest::Contains.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct State {
    int checks = 0;
    int failures = 0;
    int case_failures = 0;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++state().checks;
    if (ok) return;
    ++state().failures;
    ++state().case_failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

private:
    double value_;
    double eps_ = 1.1920929e-07f * 100;  // doctest's default: FLT_EPSILON * 100
};

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};
inline bool message_matches(const Contains& c, const std::string& what) { return c.matches(what); }
inline bool message_matches(const char* exact, const std::string& what) { return what == exact; }

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                       \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                         \
    static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                            \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                       \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::report(false, "FAIL", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_ok = false;                                                              \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_ok = true;                                                                \
        } catch (...) {                                                                       \
        }                                                                                     \
        doctest::report(doctest_ok, "THROWS_AS " #expr, __FILE__, __LINE__, false);          \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                 \
    do {                                                                                      \
        bool doctest_ok = false;                                                              \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__& e) {                                                      \
            doctest_ok = doctest::message_matches(with, e.what());                            \
        } catch (...) {                                                                       \
        }                                                                                     \
        doctest::report(doctest_ok, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstdlib>
int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : doctest::registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        doctest::state().case_failures = 0;
        try {
            tc.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::state().case_failures;
            std::fprintf(stderr, "%s:%d: exception: %s\n", tc.file, tc.line, e.what());
        }
        if (doctest::state().case_failures) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %d | %d failed\n",
                cases, cases - failed_cases, failed_cases, doctest::state().checks,
                doctest::state().failures);
    return failed_cases ? 1 : 0;
}
#endif
