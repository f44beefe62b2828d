// TEST INFRASTRUCTURE — the reference's engine-agreement sweep with the GPU
// engine added. Links the UNMODIFIED reference library
// (oracle/_ref/librxref.so, built from its sources) and librxg.so through
// include/rxg_engine.hpp, exactly the adapter a `EngineId::Gpu` case in
// engines.cpp:40-82 would call. For every (regex, string) pair of the
// enumerated suite (crosscheck.cpp:111-140: every regex <= max_nodes AST
// nodes x every string <= max_len) plus seeded random pairs
// (crosscheck.cpp:161-176), all seven reference engines and the GPU must
// agree. Prints one JSON line; exit 0 iff there is no disagreement.
//
//   crosscheck_gpu [--max-nodes N] [--max-len L] [--random K] [--seed S] [--alphabet ab]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "rx/crosscheck.hpp"
#include "rx/engines.hpp"
#include "rx/heap.hpp"
#include "rx/regex.hpp"
#include "rx/utf8.hpp"
#include "rxg_engine.hpp"

namespace {

struct Tally {
    uint64_t cases = 0, gpu_disagree = 0, ref_disagree = 0, budget_skips = 0, gpu_matches = 0;
    std::vector<std::string> first;
};

void check(const rx::RegexPtr& e, const rx::Heap& h, const rx::Input& w, uint64_t budget, bool suite, Tally& t) {
    rx::EngineOptions o;
    o.budget = budget;
    o.workers = 1;
    int match = 0, nomatch = 0;
    bool budget_hit = false;
    for (rx::EngineId id : rx::all_engines) {
        const rx::MatchOutcome r = rx::run_engine(id, h, *e, w, o).outcome;
        if (r == rx::MatchOutcome::Match) ++match;
        else if (r == rx::MatchOutcome::NoMatch) ++nomatch;
        else budget_hit = true;
    }
    const bool gpu = rxg::engine_run(h, w).accepted;
    ++t.cases;
    t.gpu_matches += gpu;
    if (budget_hit && !suite) ++t.budget_skips;
    if (match && nomatch) ++t.ref_disagree;
    const bool lockstep = rx::lockstep_accepts(h, w);
    if (gpu != lockstep || (gpu ? nomatch : match)) {
        ++t.gpu_disagree;
        if (t.first.size() < 5) t.first.push_back(rx::print(e) + " / " + rx::encode_utf8(w));
    }
}

std::string esc(const std::string& s) {
    std::string o;
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o;
}

}  // namespace

int main(int argc, char** argv) {
    size_t max_nodes = 6, max_len = 5, random_cases = 200;
    uint64_t seed = 1;
    std::string alpha = "ab";
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i];
        if (k == "--max-nodes") max_nodes = std::strtoull(argv[i + 1], nullptr, 10);
        else if (k == "--max-len") max_len = std::strtoull(argv[i + 1], nullptr, 10);
        else if (k == "--random") random_cases = std::strtoull(argv[i + 1], nullptr, 10);
        else if (k == "--seed") seed = std::strtoull(argv[i + 1], nullptr, 10);
        else if (k == "--alphabet") alpha = argv[i + 1];
        else return 2;
    }
    const std::u32string al32 = rx::decode_utf8(alpha);
    const std::vector<rx::Symbol> al(al32.begin(), al32.end());
    Tally t;
    const auto regexes = rx::enumerate_regexes(max_nodes, al);
    const auto strings = rx::enumerate_strings(max_len, al);
    for (const rx::RegexPtr& e : regexes) {
        const rx::Heap h = rx::compile(*e);
        for (const rx::Input& w : strings) check(e, h, w, 50'000'000, true, t);
    }
    std::mt19937_64 rng(seed);
    for (size_t k = 0; k < random_cases; ++k) {
        const size_t nodes = std::uniform_int_distribution<size_t>(1, 12)(rng);
        const rx::RegexPtr e = rx::random_regex(nodes, al, rng);
        const rx::Heap h = rx::compile(*e);
        const rx::Input w = rx::random_input(10, al, rng);
        check(e, h, w, 1'000'000, false, t);
    }
    std::printf("{\"regexes\": %zu, \"strings\": %zu, \"cases\": %llu, \"gpu_disagreements\": %llu, "
                "\"reference_disagreements\": %llu, \"budget_skips\": %llu, \"gpu_matches\": %llu, \"first\": [",
                regexes.size(), strings.size(), (unsigned long long)t.cases, (unsigned long long)t.gpu_disagree,
                (unsigned long long)t.ref_disagree, (unsigned long long)t.budget_skips,
                (unsigned long long)t.gpu_matches);
    for (size_t i = 0; i < t.first.size(); ++i) std::printf("%s\"%s\"", i ? ", " : "", esc(t.first[i]).c_str());
    std::printf("]}\n");
    return t.gpu_disagree == 0 && t.ref_disagree == 0 ? 0 : 1;
}
