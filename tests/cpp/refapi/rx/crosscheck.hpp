// TEST INFRASTRUCTURE: <rx/crosscheck.hpp> for the reference suites — the
// case generators of the parity driver (crosscheck.cpp:13-76), restated over
// the facade's AST so the reference's sweeps drive the GPU matcher.
#pragma once

#include <random>
#include <span>
#include <vector>

#include "rx_b200.hpp"

namespace rx {

// Every tree with at most max_nodes nodes, smallest first (crosscheck.cpp:13-34).
inline std::vector<RegexPtr> enumerate_regexes(size_t max_nodes, std::span<const Symbol> alphabet) {
    std::vector<std::vector<RegexPtr>> by_size(max_nodes + 1);
    if (max_nodes >= 1) {
        by_size[1].push_back(eps());
        for (Symbol a : alphabet) by_size[1].push_back(chr(a));
    }
    for (size_t n = 2; n <= max_nodes; ++n) {
        for (const RegexPtr& e : by_size[n - 1]) by_size[n].push_back(star(e));
        for (size_t i = 1; i + 1 < n; ++i)
            for (const RegexPtr& l : by_size[i])
                for (const RegexPtr& r : by_size[n - 1 - i]) {
                    by_size[n].push_back(seq(l, r));
                    by_size[n].push_back(alt(l, r));
                }
    }
    std::vector<RegexPtr> all;
    for (size_t n = 1; n <= max_nodes; ++n) all.insert(all.end(), by_size[n].begin(), by_size[n].end());
    return all;
}

// Every string of length 0..max_len, shortest first (crosscheck.cpp:36-50).
inline std::vector<Input> enumerate_strings(size_t max_len, std::span<const Symbol> alphabet) {
    std::vector<Input> all{Input{}};
    size_t begin = 0;
    for (size_t len = 1; len <= max_len; ++len) {
        const size_t end = all.size();
        for (size_t i = begin; i < end; ++i)
            for (Symbol a : alphabet) {
                Input w = all[i];
                w.push_back(a);
                all.push_back(std::move(w));
            }
        begin = end;
    }
    return all;
}

// crosscheck.cpp:52-67 (same draws from the same engine).
inline RegexPtr random_regex(size_t nodes, std::span<const Symbol> alphabet, std::mt19937_64& rng) {
    auto pick = [&rng](size_t n) { return std::uniform_int_distribution<size_t>(0, n - 1)(rng); };
    if (nodes == 1) {
        const size_t k = pick(alphabet.size() + 1);
        return k == alphabet.size() ? eps() : chr(alphabet[k]);
    }
    if (nodes == 2 || pick(3) == 0) return star(random_regex(nodes - 1, alphabet, rng));
    const size_t left = 1 + pick(nodes - 2);
    RegexPtr l = random_regex(left, alphabet, rng);
    RegexPtr r = random_regex(nodes - 1 - left, alphabet, rng);
    return pick(2) == 0 ? seq(std::move(l), std::move(r)) : alt(std::move(l), std::move(r));
}

// crosscheck.cpp:69-76
inline Input random_input(size_t max_len, std::span<const Symbol> alphabet, std::mt19937_64& rng) {
    const size_t len = std::uniform_int_distribution<size_t>(0, max_len)(rng);
    Input w;
    for (size_t i = 0; i < len; ++i)
        w.push_back(alphabet[std::uniform_int_distribution<size_t>(0, alphabet.size() - 1)(rng)]);
    return w;
}

}  // namespace rx
