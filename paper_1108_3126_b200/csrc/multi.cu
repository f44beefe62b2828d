// Multi-GPU batch matching (BASELINE north_star (3)).
//
// Strings are independent units, so a batch shards with no data-path
// collective: contiguous shards split at string boundaries and balanced by
// bytes (rxg_shard_bounds), one K2 launch per shard, and ONE all-reduce of the
// 8-byte match count — the only inter-GPU traffic. The reference has no
// multi-device code; its data-parallel axis is the crosscheck job pool over
// independent cases (crosscheck.cpp:119-149).
//
// Two ways in:
//   * one process per GPU (torchrun, MPI): rxg_comm_* wraps ncclCommInitRank
//     and rxg_match_batch_allreduce enqueues the shard's kernel and the count
//     all-reduce on the caller's stream;
//   * one process, several GPUs: the persistent rxg_multi handle — the
//     program and memoized step are built once and uploaded per device, one
//     worker thread per device drives that device's pipelined host path
//     (copy piece k+1 while matching piece k), and the communicators
//     (ncclCommInitAll) live as long as the handle.
// NCCL is loaded with dlopen (the library also serves host-only tools).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "heap_internal.hpp"

using namespace rxg;
using rxg::detail::cuda_fail;
using rxg::detail::DeviceGuard;
using rxg::detail::fail;

namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

// The process's NCCL (a Python host that imported torch already holds its
// bundled libnccl.so.2; dlopen by soname returns that one).
const Nccl* nccl() {
    static Nccl n;
    static bool ok = [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return false;
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(lib, name));
            return f != nullptr;
        };
        return sym(n.get_unique_id, "ncclGetUniqueId") && sym(n.init_rank, "ncclCommInitRank") &&
               sym(n.init_all, "ncclCommInitAll") && sym(n.all_reduce, "ncclAllReduce") &&
               sym(n.group_start, "ncclGroupStart") && sym(n.group_end, "ncclGroupEnd") &&
               sym(n.destroy, "ncclCommDestroy") && sym(n.error_string, "ncclGetErrorString");
    }();
    return ok ? &n : nullptr;
}

int nccl_fail(const Nccl* n, ncclResult_t r, const char* where) {
    return fail(RXG_ENCCL, std::string(where) + ": " + (n ? n->error_string(r) : "NCCL not loadable"));
}

}  // namespace

struct rxg_comm {
    ncclComm_t comm = nullptr;
    int device = -1;
    int nranks = 0;
    int rank = 0;
};

// Persistent single-process multi-GPU handle.
struct rxg_multi {
    std::vector<int> devices;
    std::vector<rxg_heap*> heaps;
    std::vector<ncclComm_t> comms;   // empty: one device, or a device listed twice (counts summed on the host)
    // one worker thread per device
    std::vector<std::thread> threads;
    std::mutex mu;
    std::condition_variable cv_go, cv_done;
    uint64_t gen = 0;
    int pending = 0;
    bool quit = false;
    std::function<int(int)> job;
    std::vector<int> rcs;
    std::vector<std::string> errs;
    std::vector<int> launch_counts;
    std::mutex call_mu;   // one matching call at a time per handle

    void worker(int k) {
        cudaSetDevice(devices[static_cast<size_t>(k)]);
        uint64_t seen = 0;
        for (;;) {
            std::function<int(int)> f;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_go.wait(lk, [&] { return quit || gen != seen; });
                if (quit) return;
                seen = gen;
                f = job;
            }
            rxg::detail::set_launches(0);
            const int rc = f(k);
            std::lock_guard<std::mutex> lk(mu);
            rcs[static_cast<size_t>(k)] = rc;
            errs[static_cast<size_t>(k)] = rc ? rxg_last_error() : "";
            launch_counts[static_cast<size_t>(k)] = rxg::detail::launches();
            if (--pending == 0) cv_done.notify_all();
        }
    }

    // f(k) on every device's worker at once; the first failure's status and text.
    int run(std::function<int(int)> f) {
        const int n = static_cast<int>(devices.size());
        {
            std::lock_guard<std::mutex> lk(mu);
            job = std::move(f);
            pending = n;
            std::fill(rcs.begin(), rcs.end(), 0);
            ++gen;
        }
        cv_go.notify_all();
        std::unique_lock<std::mutex> lk(mu);
        cv_done.wait(lk, [&] { return pending == 0; });
        for (int k = 0; k < n; ++k)
            if (rcs[static_cast<size_t>(k)])
                return fail(rcs[static_cast<size_t>(k)],
                            "device " + std::to_string(devices[static_cast<size_t>(k)]) + ": " + errs[static_cast<size_t>(k)]);
        return RXG_OK;
    }

    ~rxg_multi() {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv_go.notify_all();
        for (auto& t : threads) t.join();
        if (const Nccl* n = nccl())
            for (auto c : comms) n->destroy(c);
        for (auto* h : heaps) rxg_heap_destroy(h);
    }
};

extern "C" {

int rxg_comm_unique_id(uint8_t* id, size_t cap) {
    if (!id || cap < sizeof(ncclUniqueId)) return fail(RXG_EINVAL, "id buffer needs 128 bytes");
    const Nccl* n = nccl();
    if (!n) return fail(RXG_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId u;
    if (ncclResult_t r = n->get_unique_id(&u)) return nccl_fail(n, r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return RXG_OK;
}

int rxg_comm_init_rank(const uint8_t* id, size_t id_len, int nranks, int rank, int device, rxg_comm** out) {
    if (!id || id_len < sizeof(ncclUniqueId) || nranks <= 0 || rank < 0 || rank >= nranks || device < 0 || !out)
        return fail(RXG_EINVAL, "bad arguments");
    const Nccl* n = nccl();
    if (!n) return fail(RXG_ENCCL, "libnccl.so.2 not loadable");
    DeviceGuard g(device);
    if (cudaError_t e = cudaSetDevice(device)) return cuda_fail(e, "cudaSetDevice");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto c = std::make_unique<rxg_comm>();
    if (ncclResult_t r = n->init_rank(&c->comm, nranks, u, rank)) return nccl_fail(n, r, "ncclCommInitRank");
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
    return RXG_OK;
}

void rxg_comm_destroy(rxg_comm* c) {
    if (!c) return;
    if (const Nccl* n = nccl()) {
        DeviceGuard g(c->device);
        n->destroy(c->comm);
    }
    delete c;
}

int rxg_match_batch_allreduce(rxg_heap* h, rxg_comm* c, const uint8_t* d_text, uint64_t len, int32_t delimiter,
                              uint32_t stride, unsigned long long* d_count, uint8_t* d_results, void* stream) {
    if (!c || !d_count || (!d_text && len)) return fail(RXG_EINVAL, "bad arguments");
    const bool bitset = h && !h->dfa_ok;
    if (int rc = rxg::detail::need_device(h, !bitset)) return rc;
    if (c->device != h->device) return fail(RXG_EINVAL, "communicator and heap are on different devices");
    DeviceGuard g(h->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int rc = rxg::detail::batch_any(h, d_text, len, delimiter, stride, RXG_BATCH_AUTO, d_count, d_results, st, true))
        return rc;
    const int ours = rxg::detail::launches();
    const Nccl* n = nccl();
    if (!n) return fail(RXG_ENCCL, "libnccl.so.2 not loadable");
    // the job's total on every rank, in stream order after this rank's kernel
    if (ncclResult_t r = n->all_reduce(d_count, d_count, 1, ncclUint64, ncclSum, c->comm, st))
        return nccl_fail(n, r, "ncclAllReduce");
    rxg::detail::set_launches(ours);   // NCCL's kernel is not counted as ours
    return RXG_OK;
}

int rxg_multi_create(const int* devices, int ndev, const char* pattern, size_t plen, rxg_multi** out) {
    if (!devices || ndev <= 0 || !out || (!pattern && plen)) return fail(RXG_EINVAL, "bad arguments");
    auto m = std::make_unique<rxg_multi>();
    m->devices.assign(devices, devices + ndev);
    m->heaps.assign(static_cast<size_t>(ndev), nullptr);
    // the program and memoized step are built once, then uploaded per device
    if (int rc = rxg_heap_create_pattern(pattern, plen, devices[0], &m->heaps[0])) return rc;
    if (int rc = rxg::detail::need_device(m->heaps[0], false)) return rc;
    for (int k = 1; k < ndev; ++k)
        if (int rc = rxg::detail::clone_heap(m->heaps[0], devices[k], &m->heaps[static_cast<size_t>(k)])) return rc;
    const bool distinct = std::set<int>(devices, devices + ndev).size() == static_cast<size_t>(ndev);
    if (ndev > 1 && distinct) {
        const Nccl* n = nccl();
        if (!n) return fail(RXG_ENCCL, "libnccl.so.2 not loadable");
        m->comms.assign(static_cast<size_t>(ndev), nullptr);
        if (ncclResult_t r = n->init_all(m->comms.data(), ndev, devices)) {
            m->comms.clear();
            return nccl_fail(n, r, "ncclCommInitAll");
        }
    }
    m->rcs.assign(static_cast<size_t>(ndev), 0);
    m->errs.assign(static_cast<size_t>(ndev), "");
    m->launch_counts.assign(static_cast<size_t>(ndev), 0);
    for (int k = 0; k < ndev; ++k) m->threads.emplace_back(&rxg_multi::worker, m.get(), k);
    *out = m.release();
    return RXG_OK;
}

void rxg_multi_destroy(rxg_multi* m) { delete m; }

int rxg_multi_info(const rxg_multi* m, int32_t* ndev, int32_t* uses_nccl) {
    if (!m) return fail(RXG_EINVAL, "null handle");
    if (ndev) *ndev = static_cast<int32_t>(m->devices.size());
    if (uses_nccl) *uses_nccl = m->comms.empty() ? 0 : 1;
    return RXG_OK;
}

int rxg_multi_tune(rxg_multi* m, const uint8_t* sample, uint64_t len, int32_t delimiter) {
    if (!m) return fail(RXG_EINVAL, "null handle");
    std::lock_guard<std::mutex> call(m->call_mu);
    if (int rc = rxg_heap_tune(m->heaps[0], sample, len, delimiter)) return rc;
    for (size_t k = 1; k < m->heaps.size(); ++k)
        if (int rc = rxg::detail::adopt_tuning(m->heaps[k], m->heaps[0], delimiter)) return rc;
    return RXG_OK;
}

int rxg_multi_match_batch(rxg_multi* m, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                          uint64_t* count, uint8_t* results) {
    if (!m || !count || (!text && len)) return fail(RXG_EINVAL, "bad arguments");
    std::lock_guard<std::mutex> call(m->call_mu);
    const int ndev = static_cast<int>(m->devices.size());
    rxg_heap* h0 = m->heaps[0];
    std::vector<uint64_t> off(static_cast<size_t>(ndev) + 1);
    if (int rc = rxg_shard_bounds(text, len, delimiter, stride, ndev, off.data())) return rc;
    // bank placement from the head of the buffer, sampled once for every device (speed only)
    if (delimiter >= 0 && delimiter <= 255 && h0->dfa_ok) {
        bool tuned;
        {
            std::lock_guard<std::mutex> lk(h0->mu);
            tuned = h0->line_freq.count(delimiter) != 0;
        }
        if (!tuned) {
            if (int rc = rxg_heap_tune(h0, text, std::min<uint64_t>(len, 1u << 20), delimiter)) return rc;
            for (int k = 1; k < ndev; ++k)
                if (int rc = rxg::detail::adopt_tuning(m->heaps[static_cast<size_t>(k)], h0, delimiter)) return rc;
        }
    }
    // per-shard string counts place each shard's results
    std::vector<uint64_t> base(static_cast<size_t>(ndev) + 1, 0);
    if (results) {
        std::vector<uint64_t> cnt(static_cast<size_t>(ndev), 0);
        if (int rc = m->run([&](int k) {
                cnt[static_cast<size_t>(k)] = rxg::detail::count_strings(text, off[static_cast<size_t>(k)],
                                                                         off[static_cast<size_t>(k) + 1], delimiter, stride);
                return RXG_OK;
            }))
            return rc;
        for (int k = 0; k < ndev; ++k) base[static_cast<size_t>(k) + 1] = base[static_cast<size_t>(k)] + cnt[static_cast<size_t>(k)];
    }
    // every device matches its shard through its own pipelined host path
    if (int rc = m->run([&](int k) {
            rxg_heap* h = m->heaps[static_cast<size_t>(k)];
            const uint64_t lo = off[static_cast<size_t>(k)], n = off[static_cast<size_t>(k) + 1] - lo;
            if (n == 0) {
                if (cudaError_t e = write_u64(h->d_count, 0, h->stream)) return cuda_fail(e, "zero count");
                if (cudaError_t e = cudaStreamSynchronize(h->stream)) return cuda_fail(e, "zero count");
                return RXG_OK;
            }
            return rxg::detail::host_batch(h, text + lo, n, delimiter, stride, nullptr,
                                           results ? results + base[static_cast<size_t>(k)] : nullptr, nullptr);
        }))
        return rc;
    int ours = 0;
    for (int x : m->launch_counts) ours += x;
    unsigned long long total = 0;
    if (!m->comms.empty()) {
        // the count all-reduce: 8 bytes per device, the only inter-GPU traffic
        const Nccl* n = nccl();
        if (ncclResult_t r = n->group_start()) return nccl_fail(n, r, "ncclGroupStart");
        for (int k = 0; k < ndev; ++k) {
            rxg_heap* h = m->heaps[static_cast<size_t>(k)];
            if (ncclResult_t r = n->all_reduce(h->d_count, h->d_count, 1, ncclUint64, ncclSum,
                                               m->comms[static_cast<size_t>(k)], h->stream)) {
                n->group_end();
                return nccl_fail(n, r, "ncclAllReduce");
            }
        }
        if (ncclResult_t r = n->group_end()) return nccl_fail(n, r, "ncclGroupEnd");
        for (int k = 0; k < ndev; ++k) {
            rxg_heap* h = m->heaps[static_cast<size_t>(k)];
            DeviceGuard g(h->device);
            unsigned long long c = 0;
            if (cudaError_t e = cudaMemcpyAsync(&c, h->d_count, sizeof(c), cudaMemcpyDeviceToHost, h->stream))
                return cuda_fail(e, "count readback");
            if (cudaError_t e = cudaStreamSynchronize(h->stream)) return cuda_fail(e, "count all-reduce");
            if (k == 0) total = c;
            else if (c != total) return fail(RXG_ENCCL, "all-reduced counts differ between devices");
        }
    } else {
        for (int k = 0; k < ndev; ++k) {
            rxg_heap* h = m->heaps[static_cast<size_t>(k)];
            DeviceGuard g(h->device);
            unsigned long long c = 0;
            if (cudaError_t e = cudaMemcpy(&c, h->d_count, sizeof(c), cudaMemcpyDeviceToHost))
                return cuda_fail(e, "count readback");
            total += c;
        }
    }
    *count = total;
    rxg::detail::set_launches(ours);
    return RXG_OK;
}

// One-shot form: a handle for this call only (communicators and uploads
// included); long-running callers keep an rxg_multi instead.
int rxg_match_batch_multi(const int* devices, int ndev, const char* pattern, size_t plen, const uint8_t* text,
                          uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* count, uint8_t* results) {
    if (!devices || ndev <= 0 || !count) return fail(RXG_EINVAL, "bad arguments");
    rxg_multi* m = nullptr;
    int rc = rxg_multi_create(devices, ndev, pattern, plen, &m);
    if (rc == RXG_OK) rc = rxg_multi_match_batch(m, text, len, delimiter, stride, count, results);
    const int launches = rxg::detail::launches();
    rxg_multi_destroy(m);
    rxg::detail::set_launches(launches);
    return rc;
}

}  // extern "C"
