// Synthetic workloads of SURVEY.md §8(d), configs (a)-(e). Deterministic
// (std::mt19937_64, fixed seeds), ASCII only, so input bytes are exactly the
// Unicode scalars the reference matches after decode_utf8.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace rxg {

// Keyword list KW(L, seed): r = mt19937_64(seed); while total < L: len = 3 + r()%6
// clipped to L - total; keyword = len chars 'a' + r()%26.
std::vector<std::string> synth_keywords(int total_len, uint64_t seed);

std::string synth_pattern(char config);

// Size in bytes of the full input of a config (before any sampling).
uint64_t synth_input_size(char config);

// Fills `out` with the first `n` bytes of the config's input stream for the
// given seed (seed 0 = the config's canonical seed). For line configs the
// generator stops at a line boundary at or before n and returns the number
// of bytes written; fixed-size configs write exactly n.
uint64_t synth_input(char config, uint64_t seed, uint8_t* out, uint64_t n);

}  // namespace rxg
