// rxg::count_byte (csrc/heap_internal.hpp): the host delimiter count that
// places per-string results of host-buffer calls, against a byte loop.
#include <cstdio>
#include <random>
#include <vector>

#include "heap_internal.hpp"

int main() {
    std::mt19937_64 r(1);
    for (int t = 0; t < 4000; ++t) {
        const size_t n = r() % 6000;
        std::vector<uint8_t> v(n);
        for (auto& x : v) x = r() % 4 == 0 ? 10 : static_cast<uint8_t>(r());
        const uint8_t d = t % 3 ? 10 : static_cast<uint8_t>(r());
        const size_t off = n > 8 ? r() % 8 : 0;   // unaligned starts
        uint64_t want = 0;
        for (size_t i = off; i < n; ++i) want += v[i] == d;
        if (rxg::count_byte(v.data() + off, n - off, d) != want) {
            std::printf("FAIL case %d\n", t);
            return 1;
        }
    }
    for (int d : {0, 10, 255}) {   // every byte a hit: the per-byte accumulators at their limit
        std::vector<uint8_t> all(3u << 20, static_cast<uint8_t>(d));
        if (rxg::count_byte(all.data(), all.size(), static_cast<uint8_t>(d)) != all.size() ||
            rxg::count_byte(all.data(), all.size(), static_cast<uint8_t>(d + 1)) != 0) {
            std::printf("FAIL all-%d\n", d);
            return 1;
        }
    }
    std::printf("ok\n");
    return 0;
}
