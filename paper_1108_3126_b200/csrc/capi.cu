// extern "C" boundary (include/rxg.h). Host C++ around the kernels: handle
// lifetime, lazy per-delimiter table images, stream-ordered scratch, the
// pipelined host-buffer path and the single string split over devices
// (the batch sharder and communicators are in multi.cu).
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "options.hpp"
#include "rxg.h"
#include "frontend.hpp"
#include "launch.hpp"
#include "lines_tma.hpp"
#include "program.hpp"
#include "single.hpp"
#include "utf8.hpp"
#include "pernode.hpp"
#include "chunked.hpp"
#include "many.hpp"
#include "synth.hpp"
#include "tables.hpp"
#include "heap_internal.hpp"

using namespace rxg;
using rxg::detail::DeviceGuard;
using rxg::detail::cuda_fail;
using rxg::detail::fail;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

}  // namespace

namespace rxg {
namespace detail {

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(RXG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void set_launches(int n) { g_launches = n; }
int launches() { return g_launches; }

}  // namespace detail
}  // namespace rxg

#define RXG_CUDA(call)                                  \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

rxg_heap::~rxg_heap() {
    if (device < 0) return;
    DeviceGuard g(device);
    for (auto& kv : slots) cudaFree(kv.second);
    for (auto& kv : seams) cudaFree(kv.second.first);
    for (auto& kv : scratch) cudaFree(kv.second.first);
    if (plain && plain->dev.img) cudaFree(const_cast<void*>(plain->dev.img));
    for (auto& kv : lines)
        if (kv.second->dev.img) cudaFree(const_cast<void*>(kv.second->dev.img));
    for (void* p : allocs) cudaFree(p);
    for (auto* p : d_stage)
        if (p) cudaFree(p);
    for (auto* p : h_pin)
        if (p) cudaFreeHost(p);
    for (auto* p : d_rres)
        if (p) cudaFree(p);
    for (auto* p : h_rres)
        if (p) cudaFreeHost(p);
    if (d_count) cudaFree(d_count);
    if (d_accept) cudaFree(d_accept);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (d_rounds) cudaFree(d_rounds);
    if (d_pernode) cudaFree(d_pernode);
}

namespace {

// Pageable H2D cudaMemcpy may return before the DMA lands; the heaps' kernels
// run on non-blocking streams, so table uploads wait for completion.
cudaError_t h2d(void* dst, const void* src, size_t n) {
    cudaError_t e = cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
    return e;
}

int upload(rxg_heap* h, std::unique_ptr<TableSlot>& slot, KTable&& kt) {
    if (static_cast<int>(kt.img.size()) > h->smem_limit)
        return fail(RXG_ETOOBIG, "step table needs " + std::to_string(kt.img.size()) +
                                     " B of shared memory, limit " + std::to_string(h->smem_limit));
    auto s = std::make_unique<TableSlot>();
    s->host = std::move(kt);
    void* dptr = nullptr;
    RXG_CUDA(cudaMalloc(&dptr, s->host.img.size()));
    DevTable& d = s->dev;
    d.img = dptr;   // freed by ~rxg_heap
    RXG_CUDA(h2d(dptr, s->host.img.data(), s->host.img.size()));
    const KTable& k = s->host;
    d.img_bytes = static_cast<uint32_t>(k.img.size());
    d.cls = k.cls;
    d.esize = k.esize;
    d.row_bytes = k.row_bytes;
    d.cls_off = k.cls_off;
    d.ncols = static_cast<uint32_t>(k.ncols);
    d.start = k.start;
    d.dead = k.dead;
    d.skip = k.skip;
    d.acc_shift = k.acc_shift;
    d.tail_delta = k.tail_delta;
    d.term_acc = k.term_acc;
    d.term_rej = k.term_rej;
    d.delim_col = k.delim_col;
    slot = std::move(s);
    return RXG_OK;
}

int ensure_cuda(int device) {
    int ndev = 0;
    if (device < 0 || cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
        return fail(RXG_ECUDA, "no CUDA device " + std::to_string(device));
    return RXG_OK;
}

// Per-stream state is keyed by the stream's unique id, not the handle value:
// cudaStreamPerThread (and the legacy NULL stream under per-thread default
// streams) name a different stream in every thread.
unsigned long long stream_key(cudaStream_t st) {
    unsigned long long id = 0;
    if (cudaStreamGetId(st, &id) != cudaSuccess) {
        cudaGetLastError();
        id = static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(st)) | (1ull << 63);
    }
    return id;
}

// Allocating per-stream state inside a CUDA-graph capture would tie it to the
// graph; the first call (or a growing one) must happen outside capture.
int refuse_if_capturing(cudaStream_t st, const char* what) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
        return fail(RXG_EINVAL, std::string(what) + " must be allocated outside CUDA-graph capture: make the first "
                                                    "call of this size on this stream before capturing");
    return RXG_OK;
}

// The completion slot of `st` (allocated and zeroed on its first use, in
// stream order).
int stream_slot(rxg_heap* h, cudaStream_t st, CountSlot* out, bool accumulate) {
    const unsigned long long key = stream_key(st);
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->slots.find(key);
    unsigned long long* p = it != h->slots.end() ? it->second : nullptr;
    if (!p) {
        if (int rc = refuse_if_capturing(st, "the per-stream completion slot")) return rc;
        RXG_CUDA(cudaMalloc(&p, 4 * sizeof(unsigned long long)));
        RXG_CUDA(cudaMemsetAsync(p, 0, 4 * sizeof(unsigned long long), st));
        h->slots.emplace(key, p);
    }
    out->p = p;
    out->accumulate = accumulate;
    return RXG_OK;
}

// Zeroed counters for `n` seams on stream st (kept per stream; the kernel
// re-zeroes them). A smaller buffer that is outgrown is retired, not freed:
// a graph captured earlier may still point at it.
int seam_counters(rxg_heap* h, cudaStream_t st, size_t n, unsigned int** out) {
    const unsigned long long key = stream_key(st);
    std::lock_guard<std::mutex> lk(h->mu);
    auto& e = h->seams[key];
    if (e.second < n) {
        if (int rc = refuse_if_capturing(st, "the chunked engine's seam counters")) return rc;
        if (e.first) h->allocs.push_back(e.first);
        e.first = nullptr;
        e.second = 0;
        const size_t cap = std::max<size_t>(n, 4096);
        RXG_CUDA(cudaMalloc(reinterpret_cast<void**>(&e.first), cap * sizeof(unsigned int)));
        RXG_CUDA(cudaMemsetAsync(e.first, 0, cap * sizeof(unsigned int), st));
        e.second = cap;
    }
    *out = e.first;
    return RXG_OK;
}

// Scratch of at least `bytes` for launches on stream st (stream-ordered reuse;
// outgrown buffers are retired until the heap is destroyed).
int stream_scratch(rxg_heap* h, cudaStream_t st, size_t bytes, void** out) {
    const unsigned long long key = stream_key(st);
    std::lock_guard<std::mutex> lk(h->mu);
    auto& e = h->scratch[key];
    if (e.second < bytes) {
        if (int rc = refuse_if_capturing(st, "the chunked engine's scratch")) return rc;
        if (e.first) h->allocs.push_back(e.first);
        e.first = nullptr;
        e.second = 0;
        RXG_CUDA(cudaMalloc(&e.first, bytes));
        e.second = bytes;
    }
    *out = e.first;
    return RXG_OK;
}

// Packs host arrays into one device allocation; returns device pointers in order.
template <typename... Vs>
int upload_pack(void** dbuf, std::vector<const void*>& dptrs, const Vs&... vs) {
    std::vector<std::pair<const void*, size_t>> parts{{vs.data(), vs.size() * sizeof(vs[0])}...};
    size_t total = 0;
    for (auto& p : parts) total += (p.second + 255) & ~size_t(255);
    RXG_CUDA(cudaMalloc(dbuf, std::max<size_t>(total, 256)));
    size_t off = 0;
    for (auto& p : parts) {
        uint8_t* d = static_cast<uint8_t*>(*dbuf) + off;
        if (p.second) RXG_CUDA(h2d(d, p.first, p.second));
        dptrs.push_back(d);
        off += (p.second + 255) & ~size_t(255);
    }
    return RXG_OK;
}

int rounds_tables(rxg_heap* h, const RoundsTables** out) {
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->d_rounds) {
        const Heap& hp = h->prog.heap;
        if (hp.size() > kRoundsMaxNodes) return fail(RXG_ETOOBIG, "heap too large for the one-CTA rounds engine");
        std::vector<uint8_t> kind;
        std::vector<uint32_t> sym;
        std::vector<int32_t> left, right;
        for (const HeapNode& n : hp.nodes) {
            kind.push_back(n.kind);
            sym.push_back(n.sym);
            left.push_back(n.left);
            right.push_back(n.right);
        }
        std::vector<const void*> p;
        if (int rc = upload_pack(&h->d_rounds, p, kind, sym, left, right, hp.knodes)) return rc;
        h->rounds.kind = static_cast<const uint8_t*>(p[0]);
        h->rounds.sym = static_cast<const uint32_t*>(p[1]);
        h->rounds.left = static_cast<const int32_t*>(p[2]);
        h->rounds.right = static_cast<const int32_t*>(p[3]);
        h->rounds.knode = static_cast<const int32_t*>(p[4]);
        h->rounds.n = hp.size();
    }
    *out = &h->rounds;
    return RXG_OK;
}

int pernode_tables(rxg_heap* h, const PernodeTables** out) {
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->d_pernode) {
        const Program& pg = h->prog;
        if (pg.W > 256) return fail(RXG_ETOOBIG, "more than 8191 positions for the one-warp K1 engine");
        const BitsetPlan plan = build_bitset_plan(pg);
        std::vector<uint8_t> cls(pg.byte_class, pg.byte_class + 256);
        std::vector<const void*> p;
        if (int rc = upload_pack(&h->d_pernode, p, cls, pg.class_mask, plan.shift, plan.has_group, plan.group,
                                 plan.rows, pg.init, plan.trigger))
            return rc;
        PernodeTables& t = h->pernode;
        t.cls = static_cast<const uint8_t*>(p[0]);
        t.cmask = static_cast<const uint32_t*>(p[1]);
        t.shift = static_cast<const uint32_t*>(p[2]);
        t.has_group = static_cast<const uint32_t*>(p[3]);
        t.group = static_cast<const int32_t*>(p[4]);
        t.rows = static_cast<const uint32_t*>(p[5]);
        t.init = static_cast<const uint32_t*>(p[6]);
        t.trig = static_cast<const uint32_t*>(p[7]);
        t.W = pg.W;
        t.n_bits = pg.n_bits;
        t.n_groups = plan.n_groups;
        t.n_classes = pg.n_classes;
    }
    *out = &h->pernode;
    return RXG_OK;
}

// K2b tables on the TMA data path (null image if the position set is too
// wide for a lane or the shared window does not start at 0x400).
int bits_image(rxg_heap* h, int32_t delimiter, std::shared_ptr<const BitsImage>* out) {
    const int key = delimiter < 0 ? -1 : delimiter;
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->bits.find(key);
    if (it == h->bits.end()) {
        it = h->bits.emplace(key, nullptr).first;
        auto b = std::make_shared<BitsImage>();
        b->t = make_bits_tables(h->prog, key);
        if (b->t.ok && h->tma_ok) {
            void* d = nullptr;
            const size_t ib = b->t.img.size() * 4, rb = b->t.regs.size() * 4;
            RXG_CUDA(cudaMalloc(&d, ib + rb));
            h->allocs.push_back(d);
            RXG_CUDA(h2d(d, b->t.img.data(), ib));
            RXG_CUDA(h2d(static_cast<uint8_t*>(d) + ib, b->t.regs.data(), rb));
            b->d_img = d;
            b->d_regs = reinterpret_cast<const uint32_t*>(static_cast<uint8_t*>(d) + ib);
            it->second = std::move(b);
        }
    }
    *out = it->second;
    return RXG_OK;
}

// (Re)build and publish the TMA chunk-parallel table of the plain slot
// (caller holds h->mu; the previous image stays allocated, see ChunkImage).
int build_chunk_lt(rxg_heap* h) {
    auto f = h->line_freq.find(-1);
    auto img = std::make_shared<ChunkImage>();
    img->lt = make_chunk_tma_table(h->prog, h->dfa, f == h->line_freq.end() ? nullptr : &f->second);
    LtTable& lt = img->lt;
    const int ring = (lt.packed ? 193 : 145) * 1024;   // stage ring + barriers of the kernel's shape
    if (h->tma_ok && lt.ok && static_cast<int>(lt.smem_table_end - kLtSmemBase) + ring <= h->smem_limit) {
        void* d = nullptr;
        RXG_CUDA(cudaMalloc(&d, lt.lo.size()));
        h->allocs.push_back(d);
        RXG_CUDA(h2d(d, lt.lo.data(), lt.lo.size()));
        img->d = d;
    } else {
        lt.ok = false;
    }
    h->plain->chunk = std::move(img);
    return RXG_OK;
}

int plain_table(rxg_heap* h, const DevTable** out, const DevTable** abs_out = nullptr,
                std::shared_ptr<const ChunkImage>* chunk_out = nullptr) {
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->plain) {
        const int rc = upload(h, h->plain, make_plain_table(h->prog, h->dfa));
        if (rc) return rc;
        const KTable& k = h->plain->host;
        // rebased copy for k_fixed_abs: raw-byte u16 rows whose entries are
        // absolute shared addresses (the dynamic window starts at 0x400)
        if (h->tma_ok && !k.cls && k.esize == 2 && k.img.size() + 0x400 < 0x10000) {
            std::vector<uint8_t> img = k.img;
            for (uint32_t r = 0; r < static_cast<uint32_t>(k.n_states); ++r)
                for (uint32_t c = 0; c < static_cast<uint32_t>(k.ncols); ++c) {
                    uint16_t v;
                    std::memcpy(&v, &img[r * k.row_bytes + c * 2u], 2);
                    v = static_cast<uint16_t>(v + 0x400);
                    std::memcpy(&img[r * k.row_bytes + c * 2u], &v, 2);
                }
            void* d_abs = nullptr;
            RXG_CUDA(cudaMalloc(&d_abs, img.size()));
            h->allocs.push_back(d_abs);
            RXG_CUDA(h2d(d_abs, img.data(), img.size()));
            h->plain->abs = h->plain->dev;
            h->plain->abs.img = d_abs;
            h->plain->has_abs = true;
        }
        if (int rc = build_chunk_lt(h)) return rc;
    }
    *out = &h->plain->dev;
    if (abs_out) *abs_out = h->plain->has_abs ? &h->plain->abs : nullptr;
    if (chunk_out) *chunk_out = h->plain->chunk;
    return RXG_OK;
}

// (Re)build, upload and publish the TMA line layout for `delim` (caller
// holds h->mu; the previous image stays allocated until the heap dies).
int build_lt(rxg_heap* h, int delim, std::shared_ptr<const LtTable>& out) {
    auto f = h->line_freq.find(delim);
    auto lt = std::make_shared<LtTable>(make_lines_tma_table(h->prog, h->dfa, static_cast<uint8_t>(delim),
                                                             f == h->line_freq.end() ? nullptr : &f->second));
    if (h->tma_ok && lt->ok && static_cast<int>(lt->smem_table_end - kLtSmemBase) + 64 * 1024 <= h->smem_limit) {
        RXG_CUDA(cudaMalloc(&lt->d_lo, lt->lo.size()));
        h->allocs.push_back(lt->d_lo);
        RXG_CUDA(cudaMalloc(&lt->d_hi, lt->hi.size()));
        h->allocs.push_back(lt->d_hi);
        RXG_CUDA(h2d(lt->d_lo, lt->lo.data(), lt->lo.size()));
        RXG_CUDA(h2d(lt->d_hi, lt->hi.data(), lt->hi.size()));
    } else {
        lt->ok = false;
    }
    out = std::move(lt);
    return RXG_OK;
}

// The slot for `delim` and a snapshot of its TMA line image (nullable).
int line_table(rxg_heap* h, int delim, TableSlot** out, std::shared_ptr<const LtTable>* lt_out = nullptr) {
    std::lock_guard<std::mutex> lk(h->mu);
    auto it = h->lines.find(delim);
    if (it == h->lines.end()) {
        std::unique_ptr<TableSlot> slot;
        const int rc = upload(h, slot, make_line_table(h->prog, h->dfa, static_cast<uint8_t>(delim)));
        if (rc) return rc;
        const bool no_tma = rxg::option("RXG_NO_TMA") != nullptr;
        if (!no_tma)
            if (int rc2 = build_lt(h, delim, slot->lt)) return rc2;
        it = h->lines.emplace(delim, std::move(slot)).first;
    }
    *out = it->second.get();
    if (lt_out) *lt_out = it->second->lt;
    return RXG_OK;
}

// Host threads filling pinned staging from pageable input: half the cores,
// 2-16 (config (c), 1 GB pageable, tools/copy_threads.py: 4 threads 28.7 GB/s,
// 8 31.8, 12 43.6, 16 42.4, 24 43.2); RXG_COPY_THREADS overrides for A/B.
unsigned copy_threads() {
    if (const char* e = rxg::option("RXG_COPY_THREADS")) {
        const unsigned v = static_cast<unsigned>(std::atoi(e));
        if (v >= 1 && v <= 64) return v;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return std::min(16u, std::max(2u, hc / 2));
}

uint32_t env_chunk() {
    const char* e = rxg::option("RXG_LINE_CHUNK");   // tuning override (bytes per range)
    return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 0u;
}

Heap heap_from_c(const rxg_node* nodes, const int32_t* knodes, int32_t n) {
    Heap h;
    h.nodes.resize(static_cast<size_t>(n));
    std::memcpy(h.nodes.data(), nodes, static_cast<size_t>(n) * sizeof(rxg_node));
    h.knodes.assign(knodes, knodes + n);
    return h;
}

// Device side of a new handle: streams, counters, shared-memory limits.
int init_device(rxg_heap* h, int device) {
    h->device = device;
    if (device >= 0) {
        DeviceGuard g(device);
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
            return fail(RXG_ECUDA, "no CUDA device " + std::to_string(device));
        RXG_CUDA(cudaSetDevice(device));
        RXG_CUDA(cudaDeviceGetAttribute(&h->smem_limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        // The TMA layouts hold absolute shared addresses and assume the dynamic
        // window starts at 0x400 (1 KB reserved per block); elsewhere use the
        // generic kernels instead of trapping at launch.
        int reserved = 0;
        RXG_CUDA(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device));
        h->tma_ok = reserved == static_cast<int>(kLtSmemBase);
        RXG_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        RXG_CUDA(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        RXG_CUDA(cudaMalloc(&h->d_count, sizeof(unsigned long long)));
        RXG_CUDA(cudaMalloc(&h->d_accept, sizeof(int32_t)));
        // keep stream-ordered scratch (results / chunked engines) cached in the
        // device's default pool instead of returning it to the driver at every sync
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    return RXG_OK;
}

int make_heap(Heap&& hp, int device, rxg_heap** out) {
    auto h = std::make_unique<rxg_heap>();
    h->prog = build_program(hp);
    h->dfa_ok = build_dfa(h->prog, kMaxDfaStates, h->dfa);
    if (h->dfa_ok) h->dfa_sets = minimize_dfa(h->dfa);
    if (int rc = init_device(h.get(), device)) return rc;
    *out = h.release();
    return RXG_OK;
}

// Install sampled placement for `delimiter` (-1: the single-string table and
// its lookback) and rebuild the affected device tables (caller holds h->mu).
int apply_tuning(rxg_heap* h, int32_t delimiter, std::vector<double> freq, uint32_t lookback) {
    h->line_freq[delimiter] = std::move(freq);
    if (delimiter < 0) {
        h->lookback = lookback;
        if (h->plain && h->device >= 0) {
            DeviceGuard g(h->device);
            return build_chunk_lt(h);
        }
        return RXG_OK;
    }
    auto it = h->lines.find(delimiter);
    if (it != h->lines.end() && it->second->lt && it->second->lt->ok && h->device >= 0) {
        DeviceGuard g(h->device);
        return build_lt(h, delimiter, it->second->lt);
    }
    return RXG_OK;
}

int ensure_stage(rxg_heap* h, size_t bytes) {
    if (h->stage_bytes >= bytes) return RXG_OK;
    for (auto*& p : h->d_stage) {
        if (p) cudaFree(p);
        p = nullptr;
    }
    h->stage_bytes = 0;
    for (auto*& p : h->d_stage) RXG_CUDA(cudaMalloc(&p, bytes));
    h->stage_bytes = bytes;
    return RXG_OK;
}

int batch_device(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride,
                 unsigned long long* d_count, uint8_t* d_results, cudaStream_t st, bool zero_count) {
    LaunchStats ls;
    // TMA kernels publish the count through the stream's slot (no memset);
    // the other kernels add into a zeroed counter
    CountSlot cs;
    if (int rc = stream_slot(h, st, &cs, !zero_count)) return rc;
    auto zero_count_now = [&]() -> cudaError_t {
        return zero_count ? write_u64(d_count, 0, st) : cudaSuccess;
    };
    if (delimiter >= 0) {
        if (delimiter > 255) return fail(RXG_EINVAL, "delimiter must be a byte");
        if (reinterpret_cast<uintptr_t>(d_text) & 15) return fail(RXG_EINVAL, "text must be 16-byte aligned");
        TableSlot* slot = nullptr;
        std::shared_ptr<const LtTable> lt;
        if (int rc = line_table(h, delimiter, &slot, &lt)) return rc;
        const bool no_lt = rxg::option("RXG_NO_LT") != nullptr;   // generic kernel (tests)
        if (lt && lt->ok && !no_lt) {
            uint32_t chunk = env_chunk();
            if (chunk % lines_tma_slice()) chunk = 0;
            if (!d_results) {
                const cudaError_t e = launch_lines_tma(*lt, d_text, len, static_cast<uint8_t>(delimiter), chunk,
                                                       d_count, cs, st);
                if (e != cudaSuccess) return cuda_fail(e, "launch_lines_tma");
                ls.kernels = 1;
            } else if (len) {   // per-line results: range delimiter counts, scan, the same walk
                chunk = lines_tma_chunk(*lt, len, chunk);
                const size_t sb = lines_tma_results_scratch(len, chunk);
                void* scratch = nullptr;
                RXG_CUDA(cudaMallocAsync(&scratch, sb, st));
                const cudaError_t e = launch_lines_tma_results(*lt, d_text, len, static_cast<uint8_t>(delimiter),
                                                               chunk, d_count, d_results, scratch, sb, cs, st);
                cudaFreeAsync(scratch, st);
                if (e != cudaSuccess) return cuda_fail(e, "launch_lines_tma_results");
                ls.kernels = 2;   // the walk and the scatter
            } else {
                RXG_CUDA(zero_count_now());
            }
        } else {
            RXG_CUDA(zero_count_now());
            const DevTable* t = &slot->dev;
            uint32_t chunk = env_chunk();
            if (chunk == 0 || chunk % 16) chunk = lines_auto_chunk(*t, len);
            unsigned long long* scratch = nullptr;
            size_t sbytes = 0;
            if (d_results) {
                sbytes = lines_scratch_bytes(len, chunk);
                RXG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sbytes, st));
            }
            const cudaError_t e = launch_lines(*t, d_text, len, static_cast<uint8_t>(delimiter), chunk, d_count,
                                               d_results, scratch, sbytes, st, &ls);
            if (scratch) cudaFreeAsync(scratch, st);
            if (e != cudaSuccess) return cuda_fail(e, "launch_lines");
        }
    } else {
        if (stride == 0 || len % stride) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
        if (stride % 16 == 0 && (reinterpret_cast<uintptr_t>(d_text) & 15))
            return fail(RXG_EINVAL, "text must be 16-byte aligned");
        const DevTable* t = nullptr;
        const DevTable* ta = nullptr;
        if (int rc = plain_table(h, &t, &ta)) return rc;
        cudaError_t e;
        const bool no_fixed_tma = rxg::option("RXG_NO_FIXED_TMA") != nullptr;   // tests
        if (ta && fixed_tma_fits(ta->img_bytes, stride, h->smem_limit) && !no_fixed_tma) {
            uint64_t done = 0;
            const uint64_t n = len / stride;
            e = launch_fixed_tma(*ta, d_text, n, stride, d_count, d_results, cs, h->device, st, &done);
            ls.kernels = done ? 1 : 0;
            if (e == cudaSuccess && done < n) {   // the few strings past the last full TMA row (adds to the count)
                LaunchStats l2;
                e = launch_fixed_abs(*ta, d_text + done * stride, n - done, stride, d_count,
                                     d_results ? d_results + done : nullptr, st, &l2);
                ls.kernels += l2.kernels;
            }
        } else {
            e = zero_count_now();
            if (e == cudaSuccess)
                e = ta && stride % 16 == 0
                        ? launch_fixed_abs(*ta, d_text, len / stride, stride, d_count, d_results, st, &ls)
                        : launch_fixed(*t, d_text, len / stride, stride, d_count, d_results, st, &ls);
        }
        if (e != cudaSuccess) return cuda_fail(e, "launch_fixed");
    }
    g_launches = static_cast<int>(ls.kernels);
    return RXG_OK;
}

// Piece boundaries for the pipelined host path: pieces end just after a
// delimiter (or at a stride multiple) so each piece holds whole strings.
std::vector<uint64_t> pieces(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t target) {
    std::vector<uint64_t> b{0};
    uint64_t at = 0;
    while (len - at > target) {
        uint64_t cut = at + target;
        if (delimiter >= 0) {
            const void* hit = std::memchr(text + cut - 1, delimiter, len - (cut - 1));
            if (!hit) break;
            cut = static_cast<uint64_t>(static_cast<const uint8_t*>(hit) - text) + 1;
            if (cut >= len) break;
        } else {
            cut -= cut % stride;
            if (cut <= at) break;
        }
        b.push_back(cut);
        at = cut;
    }
    b.push_back(len);
    return b;
}

}  // namespace

namespace rxg {
namespace detail {

uint64_t count_strings(const uint8_t* text, uint64_t lo, uint64_t hi, int32_t delimiter, uint32_t stride) {
    if (delimiter < 0) return (hi - lo) / stride;
    uint64_t n = count_byte(text + lo, hi - lo, static_cast<uint8_t>(delimiter));
    if (hi > lo && text[hi - 1] != static_cast<uint8_t>(delimiter)) ++n;
    return n;
}

int need_device(rxg_heap* h, bool dfa) {
    if (!h) return fail(RXG_EINVAL, "null heap");
    if (h->device < 0) return fail(RXG_ENODEV, "host-only heap handle");
    if (!h->prog.byte_symbols)
        return fail(RXG_EUNSUPPORTED, "pattern has a literal that is not a Unicode scalar value");
    if (dfa && !h->dfa_ok)
        return fail(RXG_ETOOBIG, "memoized step table exceeds " + std::to_string(kMaxDfaStates) + " states");
    return RXG_OK;
}

int clone_heap(const rxg_heap* proto, int device, rxg_heap** out) {
    auto h = std::make_unique<rxg_heap>();
    h->prog = proto->prog;
    h->dfa_ok = proto->dfa_ok;
    h->dfa_sets = proto->dfa_sets;
    h->dfa = proto->dfa;
    {
        std::lock_guard<std::mutex> lk(const_cast<rxg_heap*>(proto)->mu);
        h->lookback = proto->lookback;
        h->line_freq = proto->line_freq;
    }
    if (int rc = init_device(h.get(), device)) return rc;
    *out = h.release();
    return RXG_OK;
}

int adopt_tuning(rxg_heap* h, const rxg_heap* proto, int32_t delimiter) {
    std::vector<double> f;
    uint32_t lb;
    {
        std::lock_guard<std::mutex> lk(const_cast<rxg_heap*>(proto)->mu);
        auto it = proto->line_freq.find(delimiter);
        if (it == proto->line_freq.end()) return RXG_OK;
        f = it->second;
        lb = proto->lookback;
    }
    std::lock_guard<std::mutex> lk(h->mu);
    return apply_tuning(h, delimiter, std::move(f), lb);
}

}  // namespace detail
}  // namespace rxg

using rxg::detail::count_strings;
using rxg::detail::need_device;

extern "C" {

const char* rxg_strerror(int s) {
    switch (s) {
    case RXG_OK: return "ok";
    case RXG_EINVAL: return "invalid argument";
    case RXG_EPARSE: return "pattern syntax error";
    case RXG_EUTF8: return "invalid UTF-8";
    case RXG_EUNSUPPORTED: return "unsupported pattern for byte-level matching";
    case RXG_ECUDA: return "CUDA error";
    case RXG_ENOMEM: return "out of memory";
    case RXG_ETOOBIG: return "step table too large";
    case RXG_ENCCL: return "NCCL error";
    case RXG_EHEAP: return "malformed heap";
    case RXG_ENODEV: return "no device tables";
    default: return "unknown status";
    }
}

const char* rxg_last_error(void) { return g_err.c_str(); }
const char* rxg_version(void) { return "rxg 0.1 sm_100a"; }
int rxg_last_launch_count(void) { return g_launches; }

int rxg_parse_compile(const char* pattern, size_t len, rxg_node* nodes, int32_t* knodes, int32_t cap,
                      int32_t* n_out, size_t* err_pos) {
    if (!pattern && len) return fail(RXG_EINVAL, "null pattern");
    try {
        const Heap h = compile(parse(std::string_view(pattern ? pattern : "", len)));
        if (n_out) *n_out = h.size();
        const int32_t n = std::min(cap, h.size());
        if (nodes && n > 0) std::memcpy(nodes, h.nodes.data(), static_cast<size_t>(n) * sizeof(rxg_node));
        if (knodes && n > 0) std::memcpy(knodes, h.knodes.data(), static_cast<size_t>(n) * sizeof(int32_t));
        return RXG_OK;
    } catch (const ParseError& e) {
        if (err_pos) *err_pos = e.pos;
        return fail(RXG_EPARSE, e.what());
    } catch (const Utf8Error& e) {
        if (err_pos) *err_pos = e.at;
        return fail(RXG_EUTF8, e.what());
    } catch (const std::exception& e) {
        return fail(RXG_EINVAL, e.what());
    }
}

int rxg_print(const char* pattern, size_t len, char* out, size_t cap, size_t* out_len) {
    try {
        const std::string s = print(parse(std::string_view(pattern ? pattern : "", len)));
        if (out_len) *out_len = s.size();
        if (out && cap) {
            const size_t n = std::min(cap - 1, s.size());
            std::memcpy(out, s.data(), n);
            out[n] = '\0';
        }
        return RXG_OK;
    } catch (const ParseError& e) {
        return fail(RXG_EPARSE, e.what());
    } catch (const Utf8Error& e) {
        return fail(RXG_EUTF8, e.what());
    }
}

int rxg_dump(const rxg_node* nodes, const int32_t* knodes, int32_t n, char* out, size_t cap, size_t* out_len) {
    if (!nodes || !knodes || n <= 0) return fail(RXG_EINVAL, "empty heap");
    const std::string s = dump(heap_from_c(nodes, knodes, n));
    if (out_len) *out_len = s.size();
    if (out && cap) {
        const size_t k = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), k);
        out[k] = '\0';
    }
    return RXG_OK;
}

int rxg_parse_dump(const char* text, size_t len, rxg_node* nodes, int32_t* knodes, int32_t cap, int32_t* n_out) {
    try {
        const Heap h = parse_dump(std::string_view(text ? text : "", len));
        if (n_out) *n_out = h.size();
        const int32_t n = std::min(cap, h.size());
        if (nodes && n > 0) std::memcpy(nodes, h.nodes.data(), static_cast<size_t>(n) * sizeof(rxg_node));
        if (knodes && n > 0) std::memcpy(knodes, h.knodes.data(), static_cast<size_t>(n) * sizeof(int32_t));
        return RXG_OK;
    } catch (const std::exception& e) {
        return fail(RXG_EHEAP, e.what());
    }
}

int rxg_check_knode(const rxg_node* nodes, const int32_t* knodes, int32_t n, int32_t* ok) {
    if (!nodes || !knodes || !ok || n < 0) return fail(RXG_EINVAL, "bad arguments");
    *ok = n > 0 && check_knode(heap_from_c(nodes, knodes, n));
    return RXG_OK;
}

int rxg_heap_create(const rxg_node* nodes, const int32_t* knodes, int32_t n, int device, rxg_heap** out) {
    if (!nodes || !knodes || n <= 0 || !out) return fail(RXG_EINVAL, "bad arguments");
    try {
        Heap hp = heap_from_c(nodes, knodes, n);
        const std::string bad = validate_heap(hp);
        if (!bad.empty()) return fail(RXG_EHEAP, bad);
        return make_heap(std::move(hp), device, out);
    } catch (const std::bad_alloc&) {
        return fail(RXG_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(RXG_EHEAP, e.what());
    }
}

int rxg_heap_create_pattern(const char* pattern, size_t len, int device, rxg_heap** out) {
    if (!out) return fail(RXG_EINVAL, "null out");
    try {
        return make_heap(compile(parse(std::string_view(pattern ? pattern : "", len))), device, out);
    } catch (const ParseError& e) {
        return fail(RXG_EPARSE, e.what());
    } catch (const Utf8Error& e) {
        return fail(RXG_EUTF8, e.what());
    } catch (const std::bad_alloc&) {
        return fail(RXG_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(RXG_EHEAP, e.what());
    }
}

void rxg_heap_destroy(rxg_heap* h) { delete h; }

int rxg_heap_info_get(const rxg_heap* h, rxg_heap_info* info) {
    if (!h || !info) return fail(RXG_EINVAL, "bad arguments");
    std::memset(info, 0, sizeof(*info));
    info->nodes = h->prog.heap.size();
    info->positions = h->prog.n_pos;
    info->words = h->prog.W;
    info->classes = h->prog.n_classes;
    info->dfa_states = h->dfa_ok ? h->dfa.n_states : 0;
    info->dfa_sets = h->dfa_ok ? h->dfa_sets : 0;
    info->chunk_lookback = static_cast<int32_t>(h->lookback);
    info->byte_symbols = h->prog.byte_symbols;
    info->device = h->device;
    info->nullable = h->prog.test(h->prog.init, h->prog.n_pos);
    if (h->dfa_ok) {
        info->line_table_bytes = static_cast<uint32_t>(make_line_table(h->prog, h->dfa, '\n').img.size());
        info->plain_table_bytes = static_cast<uint32_t>(make_plain_table(h->prog, h->dfa).img.size());
        std::lock_guard<std::mutex> lk(const_cast<rxg_heap*>(h)->mu);
        auto it = h->lines.find('\n');
        const LtTable* lt = it != h->lines.end() ? it->second->lt.get() : nullptr;
        if (lt && lt->ok) {
            info->line_tma_layout = !lt->cls ? 1 : lt->range_k ? 3 : 2;
            info->line_col_bytes = lt->cls ? 0 : lt->col_bytes;
        }
    }
    return RXG_OK;
}

int rxg_heap_tables(const rxg_heap* h, int32_t* pos_addr, uint32_t* follow, uint32_t* init) {
    if (!h) return fail(RXG_EINVAL, "null heap");
    const Program& p = h->prog;
    if (pos_addr) std::copy(p.pos_addr.begin(), p.pos_addr.end(), pos_addr);
    if (follow) std::copy(p.follow.begin(), p.follow.end(), follow);
    if (init) std::copy(p.init.begin(), p.init.end(), init);
    return RXG_OK;
}

int rxg_host_walk(const rxg_heap* h, const uint8_t* bytes, uint64_t len, uint32_t* sets_out, int32_t* accept) {
    if (!h || (!bytes && len)) return fail(RXG_EINVAL, "bad arguments");
    const Program& p = h->prog;
    const size_t W = static_cast<size_t>(p.W);
    std::vector<uint32_t> cur(p.init), nxt(W);
    if (sets_out) std::copy(cur.begin(), cur.end(), sets_out);
    for (uint64_t i = 0; i < len; ++i) {
        step_set(p, cur.data(), p.byte_class[bytes[i]], nxt.data());
        cur.swap(nxt);
        if (sets_out) std::copy(cur.begin(), cur.end(), sets_out + (i + 1) * W);
    }
    if (accept) *accept = p.test(cur, p.n_pos);
    return RXG_OK;
}

int rxg_host_emulate_batch(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                           uint32_t chunk, uint64_t* count, uint8_t* results) {
    if (!h || !count || (!text && len)) return fail(RXG_EINVAL, "bad arguments");
    if (!h->dfa_ok) return fail(RXG_ETOOBIG, "no memoized step table");
    uint64_t cnt = 0;
    if (delimiter < 0) {
        if (stride == 0 || len % stride) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
        const KTable t = make_plain_table(h->prog, h->dfa);
        for (uint64_t i = 0; i < len / stride; ++i) {
            uint32_t s = t.start;
            for (uint32_t k = 0; k < stride; ++k) s = ktable_step(t, s, text[i * stride + k]);
            const uint32_t ok = ktable_accept(t, s);
            if (results) results[i] = static_cast<uint8_t>(ok);
            cnt += ok;
        }
        *count = cnt;
        return RXG_OK;
    }
    if (delimiter > 255) return fail(RXG_EINVAL, "delimiter must be a byte");
    if (chunk == 0) chunk = 1024;
    if (chunk % 16) return fail(RXG_EINVAL, "chunk must be a multiple of 16");
    const KTable t = make_line_table(h->prog, h->dfa, static_cast<uint8_t>(delimiter));
    const uint8_t d = static_cast<uint8_t>(delimiter);
    const uint64_t nchunks = (len + chunk - 1) / chunk;
    uint64_t line_base = 0;
    for (uint64_t c = 0; c < nchunks; ++c) {
        const uint64_t c0 = c * chunk, c1 = std::min<uint64_t>(c0 + chunk, len);
        uint64_t line = line_base;
        for (uint64_t i = c0; i < c1; ++i) line_base += text[i] == d;
        uint32_t s = (c0 == 0 || text[c0 - 1] == d) ? t.start : t.skip;
        uint32_t last = 0;
        for (uint64_t i = c0; i < c1; ++i) {
            const uint32_t prev = s;
            s = ktable_step(t, s, text[i]);
            if (text[i] == d) {
                if (prev != t.skip && results) results[line] = static_cast<uint8_t>(s >> t.acc_shift);
                ++line;
            }
            cnt += s >> t.acc_shift;
            last = text[i];
        }
        if (s != t.skip && last != d) {
            s += t.tail_delta;
            uint64_t pos = c1;
            while (pos < len && s < t.term_acc) {
                const uint64_t end = std::min<uint64_t>(pos + 16, len);
                for (; pos < end; ++pos) s = ktable_step(t, s, text[pos]);
            }
            if (s < t.term_acc) s = ktable_step(t, s, d);
            const uint32_t ok = s == t.term_acc;
            if (results) results[line] = static_cast<uint8_t>(ok);
            cnt += ok;
        }
    }
    *count = cnt;
    return RXG_OK;
}

int rxg_heap_tune(rxg_heap* h, const uint8_t* sample, uint64_t len, int32_t delimiter) {
    if (!h || (!sample && len) || delimiter < -1 || delimiter > 255) return fail(RXG_EINVAL, "bad arguments");
    if (!h->dfa_ok) return RXG_OK;
    // sampling reads only the immutable program and DFA: no lock needed
    std::vector<double> f = delimiter < 0 ? lt_sample_freq_plain(h->prog, h->dfa, sample, len)
                                          : lt_sample_freq(h->prog, h->dfa, static_cast<uint8_t>(delimiter), sample, len);
    const uint32_t lb = delimiter < 0 ? lt_sync_lookback(h->prog, h->dfa, sample, len) : 0;
    std::lock_guard<std::mutex> lk(h->mu);
    return apply_tuning(h, delimiter, std::move(f), lb);
}

int rxg_host_emulate_chunk_tma(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t* accept,
                               int32_t* layout) {
    if (!h || !accept || (!text && len)) return fail(RXG_EINVAL, "bad arguments");
    if (!h->dfa_ok) return fail(RXG_ETOOBIG, "no memoized step table");
    auto f = h->line_freq.find(-1);
    const LtTable t = make_chunk_tma_table(h->prog, h->dfa, f == h->line_freq.end() ? nullptr : &f->second);
    if (!t.ok) return fail(RXG_ETOOBIG, "DFA too large for the TMA chunk layout");
    uint32_t s = t.start;
    for (uint64_t i = 0; i < len; ++i) s = lt_chunk_step(t, s, text[i]);
    *accept = lt_chunk_accept(t, s) ? 1 : 0;
    if (layout) *layout = t.packed ? 4 : !t.cls ? 1 : t.range_k ? 3 : 2;
    return RXG_OK;
}

int rxg_host_emulate_lines_tma(const rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter,
                               uint32_t chunk, uint64_t* count) {
    if (!h || !count || (!text && len) || delimiter < 0 || delimiter > 255) return fail(RXG_EINVAL, "bad arguments");
    if (!h->dfa_ok) return fail(RXG_ETOOBIG, "no memoized step table");
    const uint8_t d = static_cast<uint8_t>(delimiter);
    auto f = h->line_freq.find(delimiter);
    const LtTable t = make_lines_tma_table(h->prog, h->dfa, d, f == h->line_freq.end() ? nullptr : &f->second);
    if (!t.ok) return fail(RXG_ETOOBIG, "DFA too large for the TMA line layout");
    if (chunk == 0 || chunk % 16) return fail(RXG_EINVAL, "chunk must be a multiple of 16");
    // same partition as launch_lines_tma: full rows, then remainder pieces
    std::vector<std::pair<uint64_t, uint64_t>> ranges;
    const uint64_t rows = len / chunk;
    for (uint64_t r = 0; r < rows; ++r) ranges.emplace_back(r * chunk, (r + 1) * chunk);
    const uint64_t rem = len - rows * chunk;
    if (rem) {
        uint64_t piece = ((rem + 31) / 32 + 15) & ~uint64_t(15);
        if (piece < 16) piece = 16;
        for (uint64_t c0 = rows * chunk; c0 < len; c0 += piece) ranges.emplace_back(c0, std::min(c0 + piece, len));
    }
    uint64_t cnt = 0;
    for (const auto& [c0, c1] : ranges) {
        uint32_t s = c0 == 0 ? t.start : t.skip;   // the line at a range's first byte is the previous range's
        for (uint64_t i = c0; i < c1; ++i) {
            s = lt_step(t, s, text[i]);
            cnt += lt_count(t, s);
        }
        const bool next_line = text[c1 - 1] == d && c1 < len;
        if (next_line || (s != t.skip && text[c1 - 1] != d)) {
            s = (next_line ? t.start : s) + t.tail_delta;
            uint64_t pos = c1;
            while (pos < len && s < t.term_acc) {
                const uint64_t end = std::min<uint64_t>((pos / 16 + 1) * 16, len);
                for (; pos < end; ++pos) s = lt_step(t, s, text[pos]);
            }
            if (s < t.term_acc) s = lt_step(t, s, d);
            cnt += s == t.term_acc;
        }
    }
    *count = cnt;
    return RXG_OK;
}

int rxg_match_one_ex(rxg_heap* h, const uint8_t* d_bytes, uint64_t len, int engine, int32_t* d_accept,
                     const rxg_one_opts* opts, void* stream) {
    if (opts && ((opts->flags & RXG_ONE_ENTRY) || opts->d_exit_state) && engine != RXG_ENGINE_CHUNKED &&
        engine != RXG_ENGINE_AUTO)
        return fail(RXG_EUNSUPPORTED, "entry / exit states need the chunked engine");
    if (engine == RXG_ENGINE_AUTO && h && !h->dfa_ok) engine = RXG_ENGINE_PERNODE;   // table over the cap
    const bool dfa_engine = engine == RXG_ENGINE_AUTO || engine == RXG_ENGINE_DFA_SEQ || engine == RXG_ENGINE_CHUNKED;
    if (int rc = need_device(h, dfa_engine)) return rc;
    if (!d_accept || (!d_bytes && len)) return fail(RXG_EINVAL, "bad arguments");
    // every single-string engine reads 16-byte vectors at 16-byte offsets of the string
    if (reinterpret_cast<uintptr_t>(d_bytes) & 15) return fail(RXG_EINVAL, "string must be 16-byte aligned");
    rxg_one_opts o{};
    if (opts) o = *opts;
    DeviceGuard g(h->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (engine) {
    case RXG_ENGINE_DFA_SEQ: {
        const DevTable* t = nullptr;
        if (int rc = plain_table(h, &t)) return rc;
        const cudaError_t e = launch_seq(*t, d_bytes, len, d_accept, st);
        if (e != cudaSuccess) return cuda_fail(e, "launch_seq");
        g_launches = 1;
        return RXG_OK;
    }
    case RXG_ENGINE_AUTO:
    case RXG_ENGINE_CHUNKED: {
        const DevTable* t = nullptr;
        std::shared_ptr<const ChunkImage> ci;
        if (int rc = plain_table(h, &t, nullptr, &ci)) return rc;
        const bool no_tma = rxg::option("RXG_NO_TMA") != nullptr;
        if (ci && ci->lt.ok && !no_tma) {
            uint32_t chunk = o.chunk ? o.chunk : chunked_tma_auto_chunk(ci->lt, len, h->device);
            if (chunk % 32) return fail(RXG_EINVAL, "chunk must be a multiple of 32 on the TMA path");
            void* scratch = nullptr;
            if (int rc = stream_scratch(h, st, chunked_tma_scratch_bytes(len, chunk), &scratch)) return rc;
            CountSlot cs;
            if (int rc = stream_slot(h, st, &cs, false)) return rc;
            // one counter per tile seam (tiles hold >= 32 ranges) and the remainder's
            if (int rc = seam_counters(h, st, (len / chunk + 1) / 32 + 2, &cs.seam)) return rc;
            const cudaError_t e = launch_chunked_tma(ci->lt, ci->d, d_bytes, len, chunk,
                                                     o.lookback ? o.lookback : h->lookback, scratch, d_accept, o.d_repairs,
                                                     cs, h->device, st,
                                                     (o.flags & RXG_ONE_ENTRY) ? o.entry_state : kStartState,
                                                     o.d_exit_state);
            // (scratch stays with the stream)
            if (e != cudaSuccess) return cuda_fail(e, "launch_chunked_tma");
            g_launches = 1;   // walk, seam check and repair in one kernel
            return RXG_OK;
        }
        uint32_t chunk = o.chunk ? o.chunk : chunked_auto_chunk(*t, len, h->device);
        if (chunk % 64) return fail(RXG_EINVAL, "chunk must be a multiple of 64");
        const uint32_t lookback = o.lookback ? o.lookback : h->lookback;
        void* scratch = nullptr;
        RXG_CUDA(cudaMallocAsync(&scratch, chunked_scratch_bytes(len, chunk), st));
        const cudaError_t e = launch_chunked(*t, d_bytes, len, chunk, lookback, scratch, d_accept, o.d_repairs,
                                             h->device, st, (o.flags & RXG_ONE_ENTRY) ? o.entry_state : kStartState,
                                             o.d_exit_state);
        cudaFreeAsync(scratch, st);
        if (e != cudaSuccess) return cuda_fail(e, "launch_chunked");
        g_launches = 2;
        return RXG_OK;
    }
    case RXG_ENGINE_PERNODE: {
        const PernodeTables* t = nullptr;
        if (int rc = pernode_tables(h, &t)) return rc;
        if (o.checkpoint_every && !o.d_checkpoints) return fail(RXG_EINVAL, "checkpoint buffer missing");
        // long strings without checkpoints: segments across SMs (stream-ordered scratch)
        PernodeSegScratch ss;
        void* sbuf = nullptr;
        const bool seg = !o.checkpoint_every && len >= kPernodeSegMin && !(o.flags & RXG_ONE_SINGLE_WARP);
        if (seg) {
            RXG_CUDA(cudaMallocAsync(&sbuf, pernode_seg_scratch_bytes(t->W), st));
            ss.entry = static_cast<uint32_t*>(sbuf);
            ss.exits = ss.entry + kPernodeMaxSegs * static_cast<size_t>(t->W);
            ss.changed = reinterpret_cast<unsigned int*>(ss.exits + 2 * kPernodeMaxSegs * static_cast<size_t>(t->W));
            ss.max_segs = kPernodeMaxSegs;
            RXG_CUDA(cudaMemsetAsync(ss.changed, 0, 16, st));
        }
        const cudaError_t e = launch_pernode(*t, d_bytes, len, o.checkpoint_every, o.d_checkpoints, d_accept, st,
                                             seg ? &ss : nullptr);
        if (sbuf) cudaFreeAsync(sbuf, st);
        if (e != cudaSuccess) return cuda_fail(e, "launch_pernode");
        g_launches = 1;
        return RXG_OK;
    }
    case RXG_ENGINE_ROUNDS: {
        if (h->prog.scalar_pos) return fail(RXG_EUNSUPPORTED, "the literal rounds engine compares bytes: ASCII literals only");
        const RoundsTables* t = nullptr;
        if (int rc = rounds_tables(h, &t)) return rc;
        const cudaError_t e = launch_rounds(*t, d_bytes, len, d_accept, o.d_stats, o.d_trace, st, o.d_enqueued,
                                            o.d_schedule);
        if (e != cudaSuccess) return cuda_fail(e, "launch_rounds");
        g_launches = 1;
        return RXG_OK;
    }
    default:
        return fail(RXG_EINVAL, "unknown engine");
    }
}

int rxg_par_task(rxg_heap* h, rxg_par_state* st, int32_t node, uint32_t symbol);
int rxg_par_run_rounds(rxg_heap* h, rxg_par_state* st, uint32_t symbol, uint64_t* launches);

namespace {

// One k_par launch on a copy of the caller's ParState (single >= 0: par_task).
int par_call(rxg_heap* h, rxg_par_state* st, uint32_t symbol, int32_t single, uint64_t* launches) {
    if (int rc = need_device(h, false)) return rc;
    if (!st || !st->c || !st->n || !st->claim_count) return fail(RXG_EINVAL, "bad state");
    const RoundsTables* t = nullptr;
    if (int rc = rounds_tables(h, &t)) return rc;
    if (single >= t->n) return fail(RXG_EINVAL, "node out of range");
    std::lock_guard<std::mutex> host_lock(h->host_mu);
    DeviceGuard g(h->device);
    const size_t N = static_cast<size_t>(t->n);
    const size_t bytes = 2 * N * 8 + N * 4 + 4 * 4 + 8;
    uint8_t* d = nullptr;
    RXG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes, h->stream));
    auto* dc = reinterpret_cast<long long*>(d);
    auto* dn = dc + N;
    auto* dl = reinterpret_cast<unsigned long long*>(dn + N);
    auto* dflags = reinterpret_cast<int*>(dl + 1);
    auto* dclaims = reinterpret_cast<uint32_t*>(dflags + 4);
    int flags[4] = {st->more_c, st->any_n, st->accept_pending, st->accept_next};
    unsigned long long nl = 0;
    cudaError_t e = cudaMemcpyAsync(dc, st->c, N * 8, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dn, st->n, N * 8, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dclaims, st->claim_count, N * 4, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dflags, flags, sizeof(flags), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = launch_par(*t, dc, dn, dclaims, dflags, st->t, symbol, single, dl, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(st->c, dc, N * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(st->n, dn, N * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(st->claim_count, dclaims, N * 4, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, dflags, sizeof(flags), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nl, dl, 8, cudaMemcpyDeviceToHost, h->stream);
    cudaFreeAsync(d, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "k_par");
    st->more_c = flags[0];
    st->any_n = flags[1];
    st->accept_pending = flags[2];
    st->accept_next = flags[3];
    if (launches) *launches = single >= 0 ? 0 : nl;
    g_launches = 1;
    return RXG_OK;
}

}  // namespace

int rxg_match_one_stats(rxg_heap* h, const uint8_t* bytes, uint64_t len, int32_t* accept, rxg_match_stats* stats) {
    if (int rc = need_device(h, false)) return rc;
    if (!accept || !stats || (!bytes && len)) return fail(RXG_EINVAL, "bad arguments");
    if (h->prog.scalar_pos) return fail(RXG_EUNSUPPORTED, "the literal rounds engine compares bytes: ASCII literals only");
    const RoundsTables* t = nullptr;
    if (int rc = rounds_tables(h, &t)) return rc;
    std::lock_guard<std::mutex> host_lock(h->host_mu);
    DeviceGuard g(h->device);
    // [accept | 5 counters | text | schedule]
    const size_t sched = stats->schedule ? (len + 1) * 4 : 0;
    const size_t off_text = 64, bytes_all = off_text + ((len + 16 + 15) & ~size_t(15)) + sched;
    uint8_t* d = nullptr;
    RXG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes_all, h->stream));
    auto* d_acc = reinterpret_cast<int32_t*>(d);
    auto* d_cnt = reinterpret_cast<unsigned long long*>(d + 8);   // claims, rounds, steps, maxc, enqueued
    uint8_t* d_text = d + off_text;
    auto* d_sched = stats->schedule ? reinterpret_cast<uint32_t*>(d + off_text + ((len + 16 + 15) & ~size_t(15))) : nullptr;
    unsigned long long host[5] = {0, 0, 0, 0, 0};
    cudaError_t e = len ? cudaMemcpyAsync(d_text, bytes, len, cudaMemcpyHostToDevice, h->stream) : cudaSuccess;
    if (e == cudaSuccess) e = launch_rounds(*t, d_text, len, d_acc, d_cnt, nullptr, h->stream, d_cnt + 4, d_sched);
    if (e == cudaSuccess) e = cudaMemcpyAsync(accept, d_acc, 4, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, d_cnt, sizeof(host), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess && d_sched && host[2])
        e = cudaMemcpy(stats->schedule, d_sched, host[2] * 4, cudaMemcpyDeviceToHost);
    cudaFreeAsync(d, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "rxg_match_one_stats");
    stats->claims = host[0];
    stats->launches = host[1];
    stats->macro_steps = host[2];
    stats->max_claims_per_node_step = static_cast<uint32_t>(host[3]);
    stats->enqueued = host[4];
    stats->schedule_len = d_sched ? host[2] : 0;
    g_launches = 1;
    return RXG_OK;
}

int rxg_par_task(rxg_heap* h, rxg_par_state* st, int32_t node, uint32_t symbol) {
    if (node < 0) return fail(RXG_EINVAL, "node out of range");
    return par_call(h, st, symbol, node, nullptr);
}

int rxg_par_run_rounds(rxg_heap* h, rxg_par_state* st, uint32_t symbol, uint64_t* launches) {
    return par_call(h, st, symbol, -1, launches);
}

int rxg_match_one_device(rxg_heap* h, const uint8_t* d_bytes, uint64_t len, int engine, int32_t* d_accept,
                         void* stream) {
    return rxg_match_one_ex(h, d_bytes, len, engine, d_accept, nullptr, stream);
}

}  // extern "C"

namespace {

// H2D of one host buffer on h->stream. Pageable input of 4 MiB and more goes
// through the heap's pinned pieces, filled by a few host threads while the
// previous piece crosses PCIe (a driver copy from pageable memory runs at the
// speed of one CPU thread).
int stage_pageable_aware(rxg_heap* h, uint8_t* dst, const uint8_t* src, uint64_t len) {
    if (!len) return RXG_OK;
    cudaPointerAttributes pa{};
    const bool pageable = len >= (4u << 20) &&
                          (cudaPointerGetAttributes(&pa, src) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered);
    cudaGetLastError();
    if (!pageable) {
        RXG_CUDA(cudaMemcpyAsync(dst, src, len, cudaMemcpyHostToDevice, h->stream));
        return RXG_OK;
    }
    constexpr uint64_t kPiece = 64ull << 20;
    const uint64_t piece = std::min<uint64_t>(kPiece, len);
    if (h->pin_bytes < piece) {
        for (auto*& p : h->h_pin) {
            if (p) cudaFreeHost(p);
            p = nullptr;
        }
        h->pin_bytes = 0;
        for (auto*& p : h->h_pin) RXG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), piece, cudaHostAllocDefault));
        h->pin_bytes = piece;
    }
    if (!h->copier) {
        h->copier = std::make_unique<HostCopyPool>(copy_threads());
    }
    cudaEvent_t done[2];
    for (auto& e : done) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaError_t e = cudaSuccess;
    uint64_t i = 0;
    for (uint64_t off = 0; off < len && e == cudaSuccess; off += piece, ++i) {
        const int k = static_cast<int>(i & 1);
        const uint64_t n = std::min(piece, len - off);
        if (i >= 2) cudaEventSynchronize(done[k]);
        h->copier->copy(h->h_pin[k], src + off, n);
        e = cudaMemcpyAsync(dst + off, h->h_pin[k], n, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess) e = cudaEventRecord(done[k], h->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);   // the pinned pieces are reused by the next call
    for (auto& d : done) cudaEventDestroy(d);
    if (e != cudaSuccess) return cuda_fail(e, "staged upload");
    return RXG_OK;
}

}  // namespace

extern "C" {

int rxg_match_one(rxg_heap* h, const uint8_t* bytes, uint64_t len, int engine, int32_t* accept) {
    if (int rc = need_device(h, engine == RXG_ENGINE_DFA_SEQ || engine == RXG_ENGINE_CHUNKED)) return rc;
    if (!accept || (!bytes && len)) return fail(RXG_EINVAL, "bad arguments");
    std::lock_guard<std::mutex> host_lock(h->host_mu);
    DeviceGuard g(h->device);
    if (int rc = ensure_stage(h, std::max<size_t>(len, 16))) return rc;
    if (int rc = stage_pageable_aware(h, h->d_stage[0], bytes, len)) return rc;
    if (int rc = rxg_match_one_device(h, h->d_stage[0], len, engine, h->d_accept, h->stream)) return rc;
    RXG_CUDA(cudaMemcpyAsync(accept, h->d_accept, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    RXG_CUDA(cudaStreamSynchronize(h->stream));
    return RXG_OK;
}

}  // extern "C"

namespace rxg {
namespace detail {

// Batch on device buffers with engine selection; zero_count = overwrite the
// count (false: accumulate, for the pieces of the pipelined host path).
int batch_any(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride, int engine,
              unsigned long long* d_count, uint8_t* d_results, cudaStream_t st, bool zero_count) {
    const bool bitset = engine == RXG_BATCH_BITSET || (engine == RXG_BATCH_AUTO && !h->dfa_ok);
    if (!bitset) return batch_device(h, d_text, len, delimiter, stride, d_count, d_results, st, zero_count);
    if (delimiter > 255) return fail(RXG_EINVAL, "delimiter must be a byte");
    std::shared_ptr<const BitsImage> bi;
    if (int rc = bits_image(h, delimiter, &bi)) return rc;
    const bool no_bits_tma = rxg::option("RXG_NO_BITS_TMA") != nullptr;   // tests: the warp-per-line kernel
    if (bi && !no_bits_tma) {
        if (delimiter < 0 && (stride == 0 || len % stride)) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
        if (reinterpret_cast<uintptr_t>(d_text) & 15) return fail(RXG_EINVAL, "text must be 16-byte aligned");
        CountSlot cs;
        if (int rc = stream_slot(h, st, &cs, !zero_count)) return rc;
        const uint32_t chunk = bits_chunk(*bi, len, delimiter, stride, 0);
        if (chunk == 0) return fail(RXG_EUNSUPPORTED, "stride too large for the bitset engine's ranges");
        const size_t sb = d_results ? bits_scratch_bytes(len, chunk, delimiter >= 0, true) : 0;
        void* scratch = nullptr;
        if (sb) RXG_CUDA(cudaMallocAsync(&scratch, sb, st));
        const cudaError_t e = launch_bits(*bi, d_text, len, delimiter, stride, chunk, d_count, d_results, scratch, sb,
                                          cs, st);
        if (scratch) cudaFreeAsync(scratch, st);
        if (e != cudaSuccess) return cuda_fail(e, "launch_bits");
        g_launches = len ? (d_results && delimiter >= 0 ? 3 : 1) : 0;
        return RXG_OK;
    }
    if (delimiter < 0) return fail(RXG_EUNSUPPORTED, "fixed stride needs the memoized step or the TMA bitset engine");
    const PernodeTables* t = nullptr;
    if (int rc = pernode_tables(h, &t)) return rc;
    if (zero_count) RXG_CUDA(write_u64(d_count, 0, st));
    const size_t sb = lines_bitset_scratch_bytes(len);
    void* scratch = nullptr;
    RXG_CUDA(cudaMallocAsync(&scratch, sb, st));
    const cudaError_t e = launch_lines_bitset(*t, d_text, len, static_cast<uint8_t>(delimiter), d_count, d_results,
                                              scratch, sb, h->device, st);
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_lines_bitset");
    g_launches = len ? 4 : 0;
    return RXG_OK;
}

}  // namespace detail
}  // namespace rxg

using rxg::detail::batch_any;

extern "C" {

int rxg_match_batch_ex(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride,
                       int engine, unsigned long long* d_count, uint8_t* d_results, void* stream) {
    const bool bitset = engine == RXG_BATCH_BITSET || (engine == RXG_BATCH_AUTO && h && !h->dfa_ok);
    if (int rc = need_device(h, !bitset)) return rc;
    if (!d_count || (!d_text && len)) return fail(RXG_EINVAL, "bad arguments");
    DeviceGuard g(h->device);
    return batch_any(h, d_text, len, delimiter, stride, engine, d_count, d_results, static_cast<cudaStream_t>(stream),
                     true);
}

int rxg_match_batch(rxg_heap* h, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride,
                    unsigned long long* d_count, uint8_t* d_results, void* stream) {
    return rxg_match_batch_ex(h, d_text, len, delimiter, stride, RXG_BATCH_AUTO, d_count, d_results, stream);
}

int rxg_match_batch_host(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                         uint64_t* count, uint8_t* results) {
    return rxg_match_batch_host_ex(h, text, len, delimiter, stride, count, results, nullptr);
}

}  // extern "C"

namespace rxg {
namespace detail {

int host_batch(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* count,
               uint8_t* results, uint64_t* utf8_first_bad) {
    if (int rc = need_device(h, false)) return rc;
    if (utf8_first_bad && delimiter > 127) return fail(RXG_EINVAL, "UTF-8 check needs an ASCII delimiter");
    std::lock_guard<std::mutex> host_lock(h->host_mu);
    if (!text && len) return fail(RXG_EINVAL, "bad arguments");
    if (delimiter < 0 && (stride == 0 || len % stride)) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
    DeviceGuard g(h->device);
    if (delimiter >= 0 && delimiter <= 255 && h->dfa_ok) {
        bool tuned;
        {
            std::lock_guard<std::mutex> lk(h->mu);
            tuned = h->line_freq.count(delimiter) != 0;
        }
        if (!tuned)   // bank placement from the head of the buffer (speed only)
            if (int rc = rxg_heap_tune(h, text, std::min<uint64_t>(len, 1u << 20), delimiter)) return rc;
    }
    // Pipelined: piece k+1 is copied on copy_stream while piece k is matched.
    constexpr uint64_t kPiece = 64ull << 20;
    const std::vector<uint64_t> b = pieces(text, len, delimiter, stride, kPiece);
    uint64_t maxp = 16;
    for (size_t i = 0; i + 1 < b.size(); ++i) maxp = std::max(maxp, b[i + 1] - b[i]);
    if (int rc = ensure_stage(h, (maxp + 15) & ~uint64_t(15))) return rc;
    // Pageable input (the C++ facade's std::string, a numpy array, a mapped
    // file): a driver copy from pageable memory stages through one CPU thread
    // (~11 GB/s measured); instead a few host threads fill pinned pieces while
    // the previous piece crosses PCIe and is matched.
    cudaPointerAttributes pa{};
    const bool pageable = len >= (4u << 20) &&
                          (cudaPointerGetAttributes(&pa, text) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered);
    cudaGetLastError();
    if (pageable && h->pin_bytes < maxp) {
        for (auto*& p : h->h_pin) {
            if (p) cudaFreeHost(p);
            p = nullptr;
        }
        h->pin_bytes = 0;
        for (auto*& p : h->h_pin) RXG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), maxp, cudaHostAllocDefault));
        h->pin_bytes = maxp;
    }
    // Per-string results: piece k's strings are counted on the host threads
    // (fused into the pageable copy, else a count-only pass) to place them,
    // matched into a device slot, and brought back through a pinned slot; the
    // host copies them out two pieces later, so the pipeline never waits on a
    // download into pageable memory.
    const bool pool_count = results && delimiter >= 0 && len >= (1u << 20);
    if ((pageable || pool_count) && !h->copier) {
        h->copier = std::make_unique<HostCopyPool>(copy_threads());
    }
    cudaEvent_t copied[2], consumed[2], landed[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&landed[i], cudaEventDisableTiming);
    }
    RXG_CUDA(write_u64(h->d_count, 0, h->stream));
    unsigned long long* d_bad = nullptr;
    if (utf8_first_bad) {
        RXG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(unsigned long long), h->stream));
        RXG_CUDA(write_u64(d_bad, ~0ull, h->stream));
    }
    int rc = RXG_OK;
    int launches = 1;
    uint64_t res_at = 0;                 // strings before the current piece
    uint64_t slot_at[2] = {0, 0}, slot_n[2] = {0, 0};
    bool slot_busy[2] = {false, false};
    auto deliver = [&](int k) {          // piece results in pinned slot k -> caller's buffer
        if (!slot_busy[k]) return;
        cudaEventSynchronize(landed[k]);
        std::memcpy(results + slot_at[k], h->h_rres[k], slot_n[k]);
        slot_busy[k] = false;
    };
    for (size_t i = 0; i + 1 < b.size() && rc == RXG_OK; ++i) {
        const int k = static_cast<int>(i & 1);
        const uint64_t n = b[i + 1] - b[i];
        if (i >= 2) cudaStreamWaitEvent(h->copy_stream, consumed[k], 0);
        uint64_t delims = 0;
        const int cdel = results && delimiter >= 0 ? delimiter : -1;
        if (pageable) {   // pinned piece k is free once its previous H2D copy (piece i - 2) has landed
            if (i >= 2) cudaEventSynchronize(copied[k]);
            delims = h->copier->copy(h->h_pin[k], text + b[i], n, cdel);
            cudaMemcpyAsync(h->d_stage[k], h->h_pin[k], n, cudaMemcpyHostToDevice, h->copy_stream);
        } else {
            cudaMemcpyAsync(h->d_stage[k], text + b[i], n, cudaMemcpyHostToDevice, h->copy_stream);
            if (cdel >= 0)
                delims = pool_count ? h->copier->copy(nullptr, text + b[i], n, cdel)
                                    : count_byte(text + b[i], n, static_cast<uint8_t>(cdel));
        }
        cudaEventRecord(copied[k], h->copy_stream);
        cudaStreamWaitEvent(h->stream, copied[k], 0);
        uint64_t nres = 0;
        if (results) {
            nres = delimiter < 0 ? n / stride : delims + (n && text[b[i + 1] - 1] != static_cast<uint8_t>(delimiter));
            deliver(k);                  // slot k's previous piece (i - 2) is out before it is reused
            if (nres > h->rres_bytes[k]) {
                const size_t want = std::max<size_t>(nres + nres / 4, 1u << 16);
                if (h->d_rres[k]) cudaFree(h->d_rres[k]);
                if (h->h_rres[k]) cudaFreeHost(h->h_rres[k]);
                h->d_rres[k] = h->h_rres[k] = nullptr;
                h->rres_bytes[k] = 0;
                cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&h->d_rres[k]), want);
                if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&h->h_rres[k]), want, cudaHostAllocDefault);
                if (e != cudaSuccess) {
                    rc = cuda_fail(e, "results slots");
                    break;
                }
                h->rres_bytes[k] = want;
            }
        }
        rc = batch_any(h, h->d_stage[k], n, delimiter, stride, RXG_BATCH_AUTO, h->d_count,
                       results ? h->d_rres[k] : nullptr, h->stream, false);
        launches += g_launches;
        if (rc == RXG_OK && d_bad) {   // strings never straddle pieces, so per-piece checks are exact
            const cudaError_t e = launch_utf8_check(h->d_stage[k], n, delimiter, delimiter < 0 ? stride : 0, b[i], d_bad,
                                                    h->device, h->stream);
            if (e != cudaSuccess) rc = cuda_fail(e, "launch_utf8_check");
            launches += n ? 1 : 0;
        }
        cudaEventRecord(consumed[k], h->stream);
        if (rc == RXG_OK && results && nres) {
            cudaMemcpyAsync(h->h_rres[k], h->d_rres[k], nres, cudaMemcpyDeviceToHost, h->stream);
            cudaEventRecord(landed[k], h->stream);
            slot_at[k] = res_at;
            slot_n[k] = nres;
            slot_busy[k] = true;
        }
        res_at += nres;
    }
    if (rc == RXG_OK) {
        unsigned long long c = 0;
        cudaMemcpyAsync(&c, h->d_count, sizeof(c), cudaMemcpyDeviceToHost, h->stream);
        unsigned long long bad = ~0ull;
        if (d_bad) cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, h->stream);
        const cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "match_batch_host");
        if (rc == RXG_OK) {
            deliver(0);
            deliver(1);
        }
        if (count) *count = c;
        if (utf8_first_bad) *utf8_first_bad = bad;
    }
    if (d_bad) cudaFreeAsync(d_bad, h->stream);
    cudaStreamSynchronize(h->stream);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(copied[i]);
        cudaEventDestroy(consumed[i]);
        cudaEventDestroy(landed[i]);
    }
    g_launches = launches;
    return rc;
}

}  // namespace detail
}  // namespace rxg

extern "C" {

int rxg_match_batch_host_ex(rxg_heap* h, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                            uint64_t* count, uint8_t* results, uint64_t* utf8_first_bad) {
    if (!count) return fail(RXG_EINVAL, "bad arguments");
    return rxg::detail::host_batch(h, text, len, delimiter, stride, count, results, utf8_first_bad);
}

int rxg_utf8_check(int device, const uint8_t* d_text, uint64_t len, int32_t delimiter, uint32_t stride,
                   uint64_t* d_first_bad, void* stream) {
    if (!d_first_bad || (!d_text && len) || delimiter > 127) return fail(RXG_EINVAL, "bad arguments");
    if (delimiter < 0 && stride && len % stride) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
    if (int rc = ensure_cuda(device)) return rc;
    DeviceGuard g(device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* out = reinterpret_cast<unsigned long long*>(d_first_bad);
    RXG_CUDA(write_u64(out, ~0ull, st));
    const cudaError_t e = launch_utf8_check(d_text, len, delimiter, delimiter < 0 ? stride : 0, 0, out, device, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_utf8_check");
    g_launches = len ? 1 : 0;
    return RXG_OK;
}

int rxg_utf8_check_host(int device, const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride,
                        uint64_t* first_bad) {
    if (!first_bad || (!text && len) || delimiter > 127) return fail(RXG_EINVAL, "bad arguments");
    if (int rc = ensure_cuda(device)) return rc;
    DeviceGuard g(device);
    uint8_t* d = nullptr;
    RXG_CUDA(cudaMalloc(&d, len + 16));
    cudaError_t e = len ? cudaMemcpy(d + 8, text, len, cudaMemcpyHostToDevice) : cudaSuccess;
    int rc = RXG_OK;
    if (e == cudaSuccess) rc = rxg_utf8_check(device, d + 8, len, delimiter, stride, reinterpret_cast<uint64_t*>(d), nullptr);
    else rc = cuda_fail(e, "upload");
    if (rc == RXG_OK) {
        unsigned long long bad = ~0ull;
        e = cudaMemcpy(&bad, d, sizeof(bad), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = cuda_fail(e, "readback");
        *first_bad = bad;
    }
    cudaFree(d);
    return rc;
}

int rxg_match_many(int device, const char* patterns, int32_t n_patterns, const uint8_t* text, uint64_t len,
                   int32_t delimiter, uint32_t stride, uint8_t* results, uint64_t* n_strings, int32_t* bad_pattern) {
    if (!patterns || n_patterns < 0 || (!text && len) || !results || !n_strings) return fail(RXG_EINVAL, "bad arguments");
    if (delimiter > 255 || (delimiter < 0 && (stride == 0 || len % stride))) return fail(RXG_EINVAL, "bad string layout");
    // strings
    std::vector<uint64_t> off{0};
    uint32_t sep = 0;
    if (delimiter >= 0) {
        sep = 1;
        for (uint64_t at = 0; at < len;) {
            const void* nl = std::memchr(text + at, delimiter, len - at);
            at = nl ? static_cast<uint64_t>(static_cast<const uint8_t*>(nl) - text) + 1 : len + 1;
            off.push_back(at);   // +1 past the delimiter; a final unterminated string ends at len (+1 virtual)
        }
    } else {
        for (uint64_t at = stride; at <= len; at += stride) off.push_back(at);
    }
    const uint64_t ns = off.size() - 1;
    *n_strings = ns;
    // per-pattern tables (host: parse, compile, position form, memoized step)
    std::vector<uint8_t> tables;
    std::vector<uint64_t> toff{0};
    std::vector<uint32_t> meta;
    uint32_t max_bytes = 16;
    const char* pp = patterns;
    for (int32_t k = 0; k < n_patterns; ++k) {
        const size_t pl = std::strlen(pp);
        try {
            const Program pg = build_program(compile(parse(std::string_view(pp, pl))));
            Dfa d;
            if (!pg.byte_symbols || !build_dfa(pg, 4096, d)) {
                if (bad_pattern) *bad_pattern = k;
                return fail(RXG_ETOOBIG, "pattern " + std::to_string(k) + ": memoized step table too large");
            }
            minimize_dfa(d);
            const uint32_t S = static_cast<uint32_t>(d.n_states), C = static_cast<uint32_t>(pg.n_classes);
            const uint32_t acc_off = 256, rows_off = (256 + S + 15) & ~15u;
            const uint32_t bytes = (rows_off + S * C * 2 + 15) & ~15u;
            std::vector<uint8_t> img(bytes, 0);
            std::memcpy(img.data(), pg.byte_class, 256);
            for (uint32_t st = 0; st < S; ++st) {
                img[acc_off + st] = d.accept[st];
                for (uint32_t c = 0; c < C; ++c) {
                    const uint16_t v = static_cast<uint16_t>(d.next[st * C + c]);
                    std::memcpy(&img[rows_off + (st * C + c) * 2], &v, 2);
                }
            }
            tables.insert(tables.end(), img.begin(), img.end());
            toff.push_back(tables.size());
            meta.insert(meta.end(), {S, C, static_cast<uint32_t>(d.start), acc_off, rows_off});
            max_bytes = std::max(max_bytes, bytes);
        } catch (const ParseError& e) {
            if (bad_pattern) *bad_pattern = k;
            return fail(RXG_EPARSE, "pattern " + std::to_string(k) + ": " + e.what());
        } catch (const Utf8Error& e) {
            if (bad_pattern) *bad_pattern = k;
            return fail(RXG_EUTF8, "pattern " + std::to_string(k) + ": " + e.what());
        }
        pp += pl + 1;
    }
    if (max_bytes > 200u * 1024u) return fail(RXG_ETOOBIG, "a pattern table exceeds shared memory");
    if (n_patterns == 0 || ns == 0) return RXG_OK;
    DeviceGuard g(device);
    // one device buffer: tables | table offsets | meta | text | string offsets | results
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t b0 = al(tables.size()), b1 = al(toff.size() * 8), b2 = al(meta.size() * 4), b3 = al(len + 16),
                 b4 = al(off.size() * 8), b5 = al(static_cast<size_t>(n_patterns) * ns);
    uint8_t* d = nullptr;
    RXG_CUDA(cudaMalloc(&d, b0 + b1 + b2 + b3 + b4 + b5));
    int rc = RXG_OK;
    cudaError_t e = cudaSuccess;
    ManyDev md;
    md.tables = d;
    md.table_off = reinterpret_cast<const uint64_t*>(d + b0);
    md.meta = reinterpret_cast<const uint32_t*>(d + b0 + b1);
    md.text = d + b0 + b1 + b2;
    md.str_off = reinterpret_cast<const uint64_t*>(d + b0 + b1 + b2 + b3);
    uint8_t* dres = d + b0 + b1 + b2 + b3 + b4;
    if ((e = cudaMemcpy(d, tables.data(), tables.size(), cudaMemcpyHostToDevice)) == cudaSuccess &&
        (e = cudaMemcpy(d + b0, toff.data(), toff.size() * 8, cudaMemcpyHostToDevice)) == cudaSuccess &&
        (e = cudaMemcpy(d + b0 + b1, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice)) == cudaSuccess &&
        (!len || (e = cudaMemcpy(d + b0 + b1 + b2, text, len, cudaMemcpyHostToDevice)) == cudaSuccess) &&
        (e = cudaMemcpy(d + b0 + b1 + b2 + b3, off.data(), off.size() * 8, cudaMemcpyHostToDevice)) == cudaSuccess &&
        (e = launch_many(md, static_cast<uint64_t>(n_patterns), ns, sep, dres, max_bytes, device, nullptr)) == cudaSuccess)
        e = cudaMemcpy(results, dres, static_cast<size_t>(n_patterns) * ns, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "rxg_match_many");
    cudaFree(d);
    g_launches = 1;
    return rc;
}

int rxg_match_one_multi(const int* devices, int ndev, const char* pattern, size_t plen, const uint8_t* text,
                        uint64_t len, int32_t* accept, int32_t* resegments) {
    if (!devices || ndev <= 0 || !accept || (!text && len)) return fail(RXG_EINVAL, "bad arguments");
    constexpr uint64_t kPre = 64;   // the chunk engine's lookback
    struct Seg {
        rxg_heap* h = nullptr;
        uint8_t* d = nullptr;        // [prefix | segment], 16-byte aligned parts
        uint32_t* d_st = nullptr;    // [guess, exit]
        int32_t* d_acc = nullptr;
        uint64_t lo = 0, hi = 0, pre = 0;
        uint32_t st[2] = {0, 0};
        int32_t acc = 0;
    };
    std::vector<Seg> seg(static_cast<size_t>(ndev));
    int rc = RXG_OK;
    auto run = [&](Seg& g, bool guess, uint32_t entry) -> int {
        DeviceGuard dg(g.h->device);
        rxg_one_opts o{};
        o.flags = RXG_ONE_ENTRY;
        if (guess) {   // the state the 64-byte prefix leads to from the start state
            o.flags = 0;
            o.d_exit_state = g.d_st;
            if (int r = rxg_match_one_ex(g.h, g.d, g.pre, RXG_ENGINE_CHUNKED, g.d_acc, &o, g.h->stream)) return r;
            return RXG_OK;
        }
        o.entry_state = entry;
        o.d_exit_state = g.d_st + 1;
        return rxg_match_one_ex(g.h, g.d + g.pre, g.hi - g.lo, RXG_ENGINE_CHUNKED, g.d_acc, &o, g.h->stream);
    };
    for (int k = 0; k < ndev && rc == RXG_OK; ++k) {
        Seg& g = seg[static_cast<size_t>(k)];
        g.lo = len * static_cast<uint64_t>(k) / static_cast<uint64_t>(ndev) / 16 * 16;
        g.hi = k + 1 == ndev ? len : len * static_cast<uint64_t>(k + 1) / static_cast<uint64_t>(ndev) / 16 * 16;
        g.pre = std::min<uint64_t>(kPre, g.lo);
        if ((rc = rxg_heap_create_pattern(pattern, plen, devices[k], &g.h))) break;
        if ((rc = need_device(g.h))) break;
        DeviceGuard dg(g.h->device);
        if (cudaMalloc(&g.d, g.pre + (g.hi - g.lo) + 32) != cudaSuccess || cudaMalloc(&g.d_st, 16) != cudaSuccess ||
            cudaMalloc(&g.d_acc, 16) != cudaSuccess) {
            rc = fail(RXG_ENOMEM, "device allocation failed");
            break;
        }
        const cudaError_t e = cudaMemcpyAsync(g.d, text + g.lo - g.pre, g.pre + (g.hi - g.lo), cudaMemcpyHostToDevice,
                                              g.h->stream);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "segment upload");
            break;
        }
        // segment k > 0 guesses its entry from its prefix; every device runs at once
        if (k > 0) {
            if ((rc = run(g, true, 0))) break;
            if (cudaMemcpyAsync(&g.st[0], g.d_st, 4, cudaMemcpyDeviceToHost, g.h->stream) != cudaSuccess) {
                rc = cuda_fail(cudaGetLastError(), "guess readback");
                break;
            }
        }
    }
    // phase 1: the guesses land, then each segment runs from its guess
    for (int k = 0; k < ndev && rc == RXG_OK; ++k) {
        Seg& g = seg[static_cast<size_t>(k)];
        DeviceGuard dg(g.h->device);
        if (cudaStreamSynchronize(g.h->stream) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "guess");
            break;
        }
        rc = run(g, false, k == 0 ? kStartState : g.st[0]);
        if (rc == RXG_OK && (cudaMemcpyAsync(&g.st[1], g.d_st + 1, 4, cudaMemcpyDeviceToHost, g.h->stream) != cudaSuccess ||
                             cudaMemcpyAsync(&g.acc, g.d_acc, 4, cudaMemcpyDeviceToHost, g.h->stream) != cudaSuccess))
            rc = cuda_fail(cudaGetLastError(), "segment readback");
    }
    // phase 2: chain the exact states in order; re-run a segment whose guess was wrong
    int32_t reruns = 0;
    uint32_t exact = 0;
    for (int k = 0; k < ndev && rc == RXG_OK; ++k) {
        Seg& g = seg[static_cast<size_t>(k)];
        DeviceGuard dg(g.h->device);
        if (cudaStreamSynchronize(g.h->stream) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "segment");
            break;
        }
        if (k > 0 && g.st[0] != exact) {
            ++reruns;
            if ((rc = run(g, false, exact))) break;
            if (cudaMemcpyAsync(&g.st[1], g.d_st + 1, 4, cudaMemcpyDeviceToHost, g.h->stream) != cudaSuccess ||
                cudaMemcpyAsync(&g.acc, g.d_acc, 4, cudaMemcpyDeviceToHost, g.h->stream) != cudaSuccess ||
                cudaStreamSynchronize(g.h->stream) != cudaSuccess) {
                rc = cuda_fail(cudaGetLastError(), "segment re-run");
                break;
            }
        }
        exact = g.st[1];
        *accept = g.acc;
    }
    for (auto& g : seg) {
        if (!g.h) continue;
        DeviceGuard dg(g.h->device);
        cudaStreamSynchronize(g.h->stream);
        if (g.d) cudaFree(g.d);
        if (g.d_st) cudaFree(g.d_st);
        if (g.d_acc) cudaFree(g.d_acc);
        rxg_heap_destroy(g.h);
    }
    if (resegments) *resegments = reruns;
    g_launches = ndev + reruns;
    return rc;
}

int rxg_shard_bounds(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, int ndev,
                     uint64_t* offsets) {
    if (ndev <= 0 || !offsets || (!text && len)) return fail(RXG_EINVAL, "bad arguments");
    if (delimiter < 0 && (stride == 0 || len % stride)) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
    offsets[0] = 0;
    const uint64_t nstr = delimiter < 0 ? len / stride : 0;
    for (int k = 1; k < ndev; ++k) {
        uint64_t cut;
        if (delimiter < 0) {
            cut = nstr * static_cast<uint64_t>(k) / static_cast<uint64_t>(ndev) * stride;
        } else {
            cut = len * static_cast<uint64_t>(k) / static_cast<uint64_t>(ndev);
            if (cut > 0 && cut < len && text[cut - 1] != static_cast<uint8_t>(delimiter)) {
                const void* hit = std::memchr(text + cut, delimiter, len - cut);
                cut = hit ? static_cast<uint64_t>(static_cast<const uint8_t*>(hit) - text) + 1 : len;
            }
        }
        offsets[k] = std::max(cut, offsets[k - 1]);
    }
    offsets[ndev] = len;
    return RXG_OK;
}

int rxg_count_strings(const uint8_t* text, uint64_t len, int32_t delimiter, uint32_t stride, uint64_t* n) {
    if (!n || (!text && len) || delimiter > 255) return fail(RXG_EINVAL, "bad arguments");
    if (delimiter < 0) {
        if (stride == 0 || len % stride) return fail(RXG_EINVAL, "fixed stride must divide the buffer length");
        *n = len / stride;
        return RXG_OK;
    }
    // delimiters counted on a few host threads (the per-string results a
    // caller sizes before a host-buffer call), plus an unterminated last string
    const unsigned T = len < (8u << 20) ? 1u : std::min(16u, std::max(1u, std::thread::hardware_concurrency() / 2));
    std::vector<uint64_t> part(T, 0);
    std::vector<std::thread> ts;
    const uint64_t per = (len + T - 1) / T;
    for (unsigned k = 0; k < T; ++k) {
        const uint64_t lo = std::min(len, per * k), hi = std::min(len, lo + per);
        auto run = [&, k, lo, hi] { part[k] = count_byte(text + lo, hi - lo, static_cast<uint8_t>(delimiter)); };
        if (T == 1) run();
        else ts.emplace_back(run);
    }
    for (auto& t : ts) t.join();
    uint64_t c = 0;
    for (uint64_t x : part) c += x;
    if (len && text[len - 1] != static_cast<uint8_t>(delimiter)) ++c;
    *n = c;
    return RXG_OK;
}

int rxg_synth_pattern(char config, char* out, size_t cap, size_t* out_len) {
    try {
        const std::string s = synth_pattern(config);
        if (out_len) *out_len = s.size();
        if (out && cap) {
            const size_t n = std::min(cap - 1, s.size());
            std::memcpy(out, s.data(), n);
            out[n] = '\0';
        }
        return RXG_OK;
    } catch (const std::exception& e) {
        return fail(RXG_EINVAL, e.what());
    }
}

uint64_t rxg_synth_input_size(char config) {
    try {
        return synth_input_size(config);
    } catch (...) {
        return 0;
    }
}

int rxg_synth_input(char config, uint64_t seed, uint8_t* out, uint64_t cap, uint64_t* written) {
    if (!out && cap) return fail(RXG_EINVAL, "null buffer");
    try {
        const uint64_t n = synth_input(config, seed, out, cap);
        if (written) *written = n;
        return RXG_OK;
    } catch (const std::exception& e) {
        return fail(RXG_EINVAL, e.what());
    }
}

}  // extern "C"
