// rxg_engine.hpp — the GPU engine for the reference's engine registry.
//
// The reference dispatches every matcher through
//     EngineRun rx::run_engine(EngineId, const Heap&, const Regex&, InputView,
//                              const EngineOptions&)      (engines.hpp:42-43)
// over the enum at engines.hpp:14. Registering the GPU is one enum value
// (EngineId::Gpu, name "gpu") and one case in engines.cpp:40-82 that calls
// rxg::engine_run below (INTEGRATION.md §3 has the patch). The crosscheck
// driver (crosscheck.cpp:111-185) and the acceptance sweeps then compare the
// GPU against the seven CPU engines case by case.
//
// The function takes the reference's own rx::Heap (any type with `nodes`
// — 16-byte rx::Node, heap.hpp:17-23 — and `knodes` vectors), so this header
// needs nothing from the reference but that layout. The device handle of the
// last heap seen by the calling thread is cached: crosscheck runs every
// string of one compiled pattern back to back.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "rxg.h"
#include "rxg_utf8.hpp"

namespace rxg {

struct EngineResult {
    bool accepted;
    uint64_t steps;   // the lockstep engine's counter: rx::LockstepStats.enqueued (engines.cpp:60-64)
};

namespace detail {

struct HeapCache {
    std::vector<uint8_t> nodes;
    std::vector<int32_t> knodes;
    rxg_heap* h = nullptr;
    int device = -1;
    ~HeapCache() { rxg_heap_destroy(h); }
};

inline std::string utf8_of(std::u32string_view w) { return rxg::symbols_to_bytes(w); }

// rx::LockstepStats.enqueued of lockstep_accepts(heap, w) from the C ABI's
// set functions (lockstep.cpp:75-82 driving rxg_evolve / rxg_step_char).
template <class HeapT>
uint64_t enqueued_of(const HeapT& heap, std::u32string_view w) {
    const auto* nodes = reinterpret_cast<const rxg_node*>(heap.nodes.data());
    const int32_t n = static_cast<int32_t>(heap.nodes.size());
    std::vector<int32_t> s{0}, e(static_cast<size_t>(n) + 1), t(static_cast<size_t>(n) + 1);
    uint64_t enq = 0;
    for (char32_t a : w) {
        int32_t ne = 0, nt = 0;
        if (rxg_evolve(nodes, heap.knodes.data(), n, s.data(), static_cast<int32_t>(s.size()), e.data(), &ne, &enq))
            break;
        std::sort(e.begin(), e.begin() + ne);
        if (rxg_step_char(nodes, heap.knodes.data(), n, e.data(), ne, static_cast<uint32_t>(a), t.data(), &nt) || !nt)
            break;
        s.assign(t.begin(), t.begin() + nt);
    }
    return enq;
}

}  // namespace detail

// rx::lockstep_accepts semantics on the GPU for one (heap, input) pair.
// Throws std::runtime_error on a device or table error (the CLI maps
// exceptions to exit 2, rxvm.cpp:243-249), like every reference engine.
template <class HeapT>
EngineResult engine_run(const HeapT& heap, std::u32string_view w, int device = 0,
                        int engine = RXG_ENGINE_AUTO) {
    static_assert(sizeof(heap.nodes[0]) == sizeof(rxg_node), "rx::Node must be the 16-byte heap node");
    thread_local detail::HeapCache cache;
    const size_t nb = heap.nodes.size() * sizeof(rxg_node);
    const bool same = cache.h && cache.device == device && cache.nodes.size() == nb &&
                      cache.knodes.size() == heap.knodes.size() &&
                      std::memcmp(cache.nodes.data(), heap.nodes.data(), nb) == 0 &&
                      std::memcmp(cache.knodes.data(), heap.knodes.data(), heap.knodes.size() * 4) == 0;
    auto raise = [](int rc) {
        throw std::runtime_error(std::string("gpu engine: ") + rxg_strerror(rc) + ": " + rxg_last_error());
    };
    if (!same) {
        rxg_heap_destroy(cache.h);
        cache.h = nullptr;
        rxg_heap* h = nullptr;
        const int rc = rxg_heap_create(reinterpret_cast<const rxg_node*>(heap.nodes.data()), heap.knodes.data(),
                                       static_cast<int32_t>(heap.nodes.size()), device, &h);
        if (rc != RXG_OK) raise(rc);
        cache.h = h;
        cache.device = device;
        cache.nodes.assign(reinterpret_cast<const uint8_t*>(heap.nodes.data()),
                           reinterpret_cast<const uint8_t*>(heap.nodes.data()) + nb);
        cache.knodes.assign(heap.knodes.begin(), heap.knodes.end());
    }
    const std::string b = detail::utf8_of(w);
    int32_t acc = 0;
    if (engine == RXG_ENGINE_AUTO) {
        // the literal §8 protocol kernel answers and counts in one launch: its
        // claims per macro step are the addresses rx::evolve enqueues
        rxg_match_stats ms{};
        const int rc = rxg_match_one_stats(cache.h, reinterpret_cast<const uint8_t*>(b.data()), b.size(), &acc, &ms);
        if (rc == RXG_OK) return {acc != 0, ms.enqueued};
        if (rc != RXG_EUNSUPPORTED) raise(rc);
    }
    // memoized step when its table fits, else the thread-per-node bitset engine;
    // the counter from the host set functions (non-ASCII literals only)
    const int rc = rxg_match_one(cache.h, reinterpret_cast<const uint8_t*>(b.data()), b.size(), engine, &acc);
    if (rc != RXG_OK) raise(rc);
    return {acc != 0, detail::enqueued_of(heap, w)};
}

}  // namespace rxg
