// TEST INFRASTRUCTURE: a minimal stand-in for the doctest macros the
// reference's suites use (doctest itself is not vendored here),
// so the reference's own tests/test_lockstep.cpp and tests/test_parallel.cpp
// compile unmodified against include/rx_b200.hpp (see tests/cpp/refapi/rx/).
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace refapi {

struct Case {
    const char* name;
    const char* suite;
    std::function<void()> fn;
};

inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
inline const char*& current_suite() {
    static const char* s = "";
    return s;
}
inline long& checks() {
    static long n = 0;
    return n;
}
inline long& failures() {
    static long n = 0;
    return n;
}
inline void report(bool ok, const char* expr, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "FAIL %s:%d: %s\n", file, line, expr);
    }
}
struct Registrar {
    Registrar(const char* name, std::function<void()> fn) { cases().push_back({name, current_suite(), std::move(fn)}); }
};
struct SuiteSetter {
    explicit SuiteSetter(const char* s) { current_suite() = s; }
};

}  // namespace refapi

#define REFAPI_CAT2(a, b) a##b
#define REFAPI_CAT(a, b) REFAPI_CAT2(a, b)
#define TEST_SUITE_BEGIN(name) static refapi::SuiteSetter REFAPI_CAT(refapi_suite_, __LINE__)(name)
#define TEST_SUITE_END() static refapi::SuiteSetter REFAPI_CAT(refapi_suite_end_, __LINE__)("")
#define TEST_CASE(name)                                                                        \
    static void REFAPI_CAT(refapi_case_, __LINE__)();                                          \
    static refapi::Registrar REFAPI_CAT(refapi_reg_, __LINE__)(name, REFAPI_CAT(refapi_case_, __LINE__)); \
    static void REFAPI_CAT(refapi_case_, __LINE__)()
#define CHECK(...) refapi::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) refapi::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...) CHECK(__VA_ARGS__)
#define CHECK_THROWS_AS(expr, type)                                            \
    do {                                                                       \
        bool refapi_thrown = false;                                            \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const type&) {                                                \
            refapi_thrown = true;                                              \
        } catch (...) {                                                        \
        }                                                                      \
        refapi::report(refapi_thrown, "throws " #type ": " #expr, __FILE__, __LINE__); \
    } while (0)
