// Reads like the reference's own tests (proj/tests/test_heap.cpp, test_lockstep.cpp)
// but compiles against include/rx_b200.hpp and links librxg.so.
#include <cstdio>
#include <cstring>
#include <string>

#include "rx_b200.hpp"

static int failures = 0;
#define CHECK(x)                                                        \
    do {                                                                \
        if (!(x)) {                                                     \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++failures;                                                 \
        }                                                               \
    } while (0)

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    rx::Heap h = rx::compile(*rx::parse("a**b"));
    CHECK(h.size() == 5);
    CHECK(rx::dump(h) == "p0\tseq p1 p2\tnull\np1\tstar p3\tp2\np2\tchar b\tnull\np3\tstar p4\tp1\np4\tchar a\tp3\n");
    CHECK(h.node(0).kind == rx::Node::Kind::Seq && h.knode(3) == 1 && h.knode(4) == 3);
    CHECK(rx::check_knode(h));
    CHECK(rx::print(*rx::parse("(a**)b")) == "a**b");
    try {
        rx::parse("ab\\");
        CHECK(false);
    } catch (const rx::ParseError& e) {
        CHECK(e.pos == 3);
    }
    // decode_utf8 / encode_utf8 (utf8.hpp) with the reference's error text
    CHECK(rx::decode_utf8("a\xc3\xa9\xe4\xb8\xad") == U"a\u00e9\u4e2d");
    CHECK(rx::encode_utf8(U"a\u00e9\U0001F600") == "a\xc3\xa9\xf0\x9f\x98\x80");
    try {
        rx::decode_utf8("ab\xe4\xb8");
        CHECK(false);
    } catch (const std::runtime_error& e) {
        CHECK(std::string(e.what()) == "invalid UTF-8 at byte 2");
    }
    try {
        rx::decode_utf8("\xed\xa0\x80");
        CHECK(false);
    } catch (const std::runtime_error& e) {
        CHECK(std::string(e.what()) == "invalid UTF-8 at byte 0");
    }
    if (gpu) {
        CHECK(rx::lockstep_accepts(h, U"aab"));
        CHECK(!rx::lockstep_accepts(h, U"aa"));
        CHECK(rx::lockstep_accepts(rx::compile(*rx::parse("a**")), U""));
        CHECK(!rx::lockstep_accepts(rx::compile(*rx::parse("a")), U""));
        CHECK(rx::par_accepts(h, U"aab", 4, 7));
        CHECK(!rx::lockstep_accepts(rx::compile(*rx::parse("(a|b)*abb")), U"aébb"));
        std::vector<uint8_t> per;
        const uint64_t n = rx::match_lines(rx::compile(*rx::parse("(a|b)*abb")), "abb\nab\n\nbabb\nx", &per);
        CHECK(n == 2 && per.size() == 5 && per[0] == 1 && per[1] == 0 && per[2] == 0 && per[3] == 1 && per[4] == 0);
        uint64_t bad = 0;
        rx::match_lines(rx::compile(*rx::parse("(a|b)*abb")), "abb\na\xffb\n", nullptr, &bad);
        CHECK(bad == 5);   // the 0xFF byte: decode_utf8 of line 2 fails at its byte 1
    }
    std::printf("%s %d failures\n", gpu ? "gpu" : "cpu", failures);
    return failures ? 1 : 0;
}
