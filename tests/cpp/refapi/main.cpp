// TEST INFRASTRUCTURE: runs every TEST_CASE the reference suites registered
// (see doctest.h); exit 0 iff every CHECK held.
#include <cstdio>
#include <exception>

#include "doctest.h"

int main() {
    for (const refapi::Case& c : refapi::cases()) {
        const long before = refapi::failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++refapi::failures();
            std::fprintf(stderr, "FAIL [%s] %s: unexpected exception: %s\n", c.suite, c.name, e.what());
        }
        std::printf("%s [%s] %s\n", refapi::failures() == before ? "ok  " : "FAIL", c.suite, c.name);
    }
    std::printf("%zu cases, %ld checks, %ld failures\n", refapi::cases().size(), refapi::checks(), refapi::failures());
    return refapi::failures() ? 1 : 0;
}
