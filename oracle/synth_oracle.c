/* TEST INFRASTRUCTURE. The synthetic workloads of SURVEY.md §8(d), restated
 * in plain C from the survey's specification (std::mt19937_64 streams, the
 * five patterns and inputs), so the reference arm of bench.py and the parity
 * tests can build their inputs without loading the product library.
 * tests/test_oracle.py checks every config byte-for-byte against the
 * product's generator (paper_1108_3126_b200/csrc/synth.cpp). */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* std::mt19937_64 ([rand.predef]: the 10000th output of a default-seeded
 * engine is 9981545732273789042). */
typedef struct {
    uint64_t mt[312];
    int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (g->mt[k] & 0xFFFFFFFF80000000ULL) | (g->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
            g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        g->i = 0;
    }
    uint64_t x = g->mt[g->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

uint64_t oracle_mt64_nth(uint64_t seed, uint64_t n) {
    mt64 g;
    mt64_seed(&g, seed);
    uint64_t x = 0;
    for (uint64_t k = 0; k < n; ++k) x = mt64_next(&g);
    return x;
}

/* KW(L, seed): keywords of 3-8 random lowercase letters until L letters. */
static size_t keywords(int total_len, uint64_t seed, char* out, size_t cap, char sep) {
    mt64 g;
    mt64_seed(&g, seed);
    size_t at = 0;
    int total = 0;
    while (total < total_len) {
        int len = 3 + (int)(mt64_next(&g) % 6);
        if (len > total_len - total) len = total_len - total;
        if (total && at < cap) out[at] = sep;
        if (total) ++at;
        for (int i = 0; i < len; ++i) {
            const char c = (char)('a' + mt64_next(&g) % 26);
            if (at < cap) out[at] = c;
            ++at;
        }
        total += len;
    }
    return at;
}

static size_t put(char* out, size_t cap, size_t at, const char* s) {
    const size_t n = strlen(s);
    for (size_t i = 0; i < n; ++i)
        if (at + i < cap) out[at + i] = s[i];
    return at + n;
}

/* The pattern of config a|A|b|c|d|e as NUL-terminated text; returns its
 * length (out may be NULL to size it). */
size_t oracle_synth_pattern(char cfg, char* out, size_t cap) {
    static const char* s9 = "(a|b|c|d|e|f|g|h| )";
    static const char* s27 = "(a|b|c|d|e|f|g|h|i|j|k|l|m|n|o|p|q|r|s|t|u|v|w|x|y|z| )";
    size_t at = 0;
    switch (cfg) {
    case 'a': case 'A':
        at = put(out, cap, 0, "(a|b)*abb");
        break;
    case 'b':
        for (int i = 0; i < 32; ++i) at = put(out, cap, at, "(a|())");
        for (int i = 0; i < 32; ++i) at = put(out, cap, at, "a");
        break;
    case 'c':
        at = put(out, cap, at, "(");
        at = put(out, cap, at, s9);
        at = put(out, cap, at, "*(ERROR|WARN|FAIL)");
        at = put(out, cap, at, s9);
        at = put(out, cap, at, "*)*");
        break;
    case 'd':
        at = put(out, cap, at, "(");
        at = put(out, cap, at, s27);
        at = put(out, cap, at, "*(");
        at += keywords(457, 7, out ? out + at : NULL, out && cap > at ? cap - at : 0, '|');
        at = put(out, cap, at, ")");
        at = put(out, cap, at, s27);
        at = put(out, cap, at, "*)*");
        break;
    case 'e':
        at = put(out, cap, at, "(");
        at += keywords(2018, 7, out ? out + at : NULL, out && cap > at ? cap - at : 0, '|');
        for (char c = 'a'; c <= 'z'; ++c) {
            char item[3] = {'|', c, 0};
            at = put(out, cap, at, item);
        }
        at = put(out, cap, at, "| )*abb");
        break;
    default:
        return 0;
    }
    if (out && at < cap) out[at] = 0;
    return at;
}

static uint64_t canonical_seed(char c) {
    switch (c) {
    case 'a': case 'A': return 1;
    case 'c': return 3;
    case 'd': return 11;
    case 'e': return 5;
    default: return 0;
    }
}

/* Full size of a config's input (c: an upper bound). */
uint64_t oracle_synth_input_size(char cfg) {
    switch (cfg) {
    case 'a': case 'A': return 1ull << 20;
    case 'b': return 32000000ull;
    case 'c': return 10000000ull * 116ull;
    case 'd': return 1ull << 30;
    case 'e': return 1ull << 28;
    default: return 0;
    }
}

/* The first n bytes (c: whole lines that fit) of a config's input; seed 0 =
 * the canonical seed. Returns the bytes written. */
uint64_t oracle_synth_input(char cfg, uint64_t seed, uint8_t* out, uint64_t n) {
    mt64 g;
    mt64_seed(&g, seed ? seed : canonical_seed(cfg));
    switch (cfg) {
    case 'a': case 'A':
        for (uint64_t i = 0; i < n; ++i) out[i] = (mt64_next(&g) & 1) ? 'a' : 'b';
        if (n >= 3) memcpy(out + n - 3, "abb", 3);
        if (cfg == 'A' && n >= 1) out[n - 1] = 'a';
        return n;
    case 'b':
        memset(out, 'a', n);
        return n;
    case 'c': {
        static const char* kw[3] = {"ERROR", "WARN", "FAIL"};
        static const char alpha[] = "abcdefgh ";
        uint64_t at = 0;
        char line[128];
        for (uint64_t k = 0; k < 10000000ull; ++k) {
            const int len = 90 + (int)(mt64_next(&g) % 21);
            uint64_t bits = mt64_next(&g);
            for (int i = 0; i < len; ++i) {
                if (i % 20 == 0 && i) bits = mt64_next(&g);
                line[i] = alpha[bits % 9];
                bits /= 9;
            }
            int total = len;
            if (mt64_next(&g) % 4 == 0) {
                const char* w = kw[mt64_next(&g) % 3];
                const int wl = (int)strlen(w);
                const int pos = (int)(mt64_next(&g) % (uint64_t)(len + 1));
                memmove(line + pos + wl, line + pos, (size_t)(len - pos));
                memcpy(line + pos, w, (size_t)wl);
                total += wl;
            }
            line[total++] = '\n';
            if (at + (uint64_t)total > n) break;
            memcpy(out + at, line, (size_t)total);
            at += (uint64_t)total;
        }
        return at;
    }
    case 'd': {
        uint64_t at = 0;
        char line[1100];
        while (at < n) {
            size_t ll = 0;
            for (;;) {
                const int wl = 2 + (int)(mt64_next(&g) % 8);
                const size_t need = ll + (ll ? 1 : 0) + (size_t)wl;
                if (need > 1023) break;
                if (ll) line[ll++] = ' ';
                for (int i = 0; i < wl; ++i) line[ll++] = (char)('a' + mt64_next(&g) % 26);
            }
            line[ll++] = '\n';
            const uint64_t room = n - at;
            if (ll > room) {
                ll = (size_t)room;
                line[ll - 1] = '\n';
            }
            memcpy(out + at, line, ll);
            at += ll;
        }
        return at;
    }
    case 'e':
        for (uint64_t i = 0; i < n; ++i) out[i] = (mt64_next(&g) % 6 == 0) ? ' ' : (uint8_t)('a' + mt64_next(&g) % 26);
        if (n >= 3) memcpy(out + n - 3, "abb", 3);
        return n;
    default:
        return 0;
    }
}
