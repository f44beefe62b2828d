// rxg_engine.hpp needs only the rx::Heap layout: a stand-in heap type here
// (the reference's own is used by oracle/crosscheck_gpu.cpp).
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rxg_engine.hpp"

struct Node {
    uint8_t kind;
    uint32_t sym;
    int32_t left, right;
};
struct Heap {
    std::vector<Node> nodes;
    std::vector<int32_t> knodes;
};

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && !std::strcmp(argv[1], "gpu");
    const char* pat = "(a|b)*abb";
    int32_t n = 0;
    size_t pos = 0;
    if (rxg_parse_compile(pat, std::strlen(pat), nullptr, nullptr, 0, &n, &pos)) return 1;
    Heap h;
    h.nodes.resize(n);
    h.knodes.resize(n);
    if (rxg_parse_compile(pat, std::strlen(pat), reinterpret_cast<rxg_node*>(h.nodes.data()), h.knodes.data(), n, &n,
                          &pos))
        return 1;
    if (!gpu) {   // without a GPU the engine reports the device error as an exception
        try {
            (void)rxg::engine_run(h, U"abb", 0);
        } catch (const std::runtime_error&) {
            return 0;
        }
        return 3;
    }
    const bool a = rxg::engine_run(h, U"ababb").accepted, b = rxg::engine_run(h, U"abab").accepted;
    const bool c = rxg::engine_run(h, U"").accepted;
    std::printf("%d %d %d\n", a, b, c);
    return a && !b && !c ? 0 : 2;
}
