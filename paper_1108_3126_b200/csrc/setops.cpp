// Host side of the reference's syntax-tree and set-level matcher API
// (include/rxg.h "syntax trees" and "set-level lockstep functions"):
//
//   rxg_parse_ast / rxg_print_ast / rxg_compile_ast
//       rx::parse / rx::print / rx::compile on an explicit tree
//       (regex.hpp:26-66, heap.hpp:43; regex.cpp:73-200, heap.cpp:13-72)
//   rxg_evolve / rxg_eps_reaches_null / rxg_step_char
//       rx::evolve_ordered / rx::eps_reaches_null / rx::step_char
//       (lockstep.hpp:24-40; lockstep.cpp:10-73) over a heap table
//
// These are the one-set, one-symbol functions the reference's tests,
// traces and crosscheck call; matching whole strings runs on the GPU.
#include <algorithm>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "rxg.h"
#include "frontend.hpp"
#include "heap_internal.hpp"

using rxg::detail::fail;

namespace {

rxg::Heap heap_of(const rxg_node* nodes, const int32_t* knodes, int32_t n) {
    rxg::Heap h;
    h.nodes.resize(static_cast<size_t>(n));
    std::memcpy(h.nodes.data(), nodes, static_cast<size_t>(n) * sizeof(rxg_node));
    h.knodes.assign(knodes, knodes + n);
    return h;
}

// Unlabeled successors in the reference's fixed order (pwpi.cpp:9-20).
int eps_succ(const rxg_node* nodes, const int32_t* knodes, int32_t p, int32_t out[2]) {
    const rxg_node& x = nodes[p];
    switch (x.kind) {
    case RXG_NODE_ALT: out[0] = x.left; out[1] = x.right; return 2;
    case RXG_NODE_SEQ: out[0] = x.left; return 1;
    case RXG_NODE_STAR: out[0] = x.left; out[1] = knodes[p]; return 2;
    case RXG_NODE_EPS: out[0] = knodes[p]; return 1;
    default: return 0;
    }
}

bool heap_ok(const rxg_node* nodes, const int32_t* knodes, int32_t n, std::string* why) {
    if (!nodes || !knodes || n <= 0) {
        *why = "empty heap";
        return false;
    }
    *why = rxg::validate_heap(heap_of(nodes, knodes, n));
    return why->empty();
}

bool set_ok(const int32_t* s, int32_t ns, int32_t n) {
    if (ns < 0 || (ns && !s)) return false;
    for (int32_t i = 0; i < ns; ++i)
        if (s[i] < -1 || s[i] >= n) return false;
    return true;
}

// Expression arena from the caller's flattened tree: children precede their
// parent and every node but the root is used exactly once (a tree).
int expr_of(const rxg_ast_node* nodes, int32_t n, int32_t root, rxg::Expr* e) {
    if (!nodes || n <= 0 || root < 0 || root >= n) return fail(RXG_EINVAL, "empty or malformed tree");
    std::vector<int32_t> uses(static_cast<size_t>(n), 0);
    e->nodes.resize(static_cast<size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
        const rxg_ast_node& a = nodes[i];
        if (a.kind > RXG_AST_ALT) return fail(RXG_EINVAL, "unknown tree node kind");
        const int kids = a.kind == RXG_AST_STAR ? 1 : (a.kind == RXG_AST_SEQ || a.kind == RXG_AST_ALT) ? 2 : 0;
        const int32_t ch[2] = {a.left, a.right};
        for (int k = 0; k < kids; ++k) {
            if (ch[k] < 0 || ch[k] >= i) return fail(RXG_EINVAL, "tree children must precede their parent");
            ++uses[static_cast<size_t>(ch[k])];
        }
        e->nodes[static_cast<size_t>(i)] = rxg::ExprNode{a.kind, a.kind == RXG_AST_CHR ? a.sym : 0u,
                                                         kids >= 1 ? a.left : -1, kids == 2 ? a.right : -1};
    }
    for (int32_t i = 0; i < n; ++i)
        if (uses[static_cast<size_t>(i)] != (i == root ? 0 : 1))
            return fail(RXG_EINVAL, "nodes must form one tree rooted at `root` (no sharing, nothing unused)");
    e->root = root;
    return RXG_OK;
}

}  // namespace

extern "C" {

int rxg_parse_ast(const char* pattern, size_t len, rxg_ast_node* out, int32_t cap, int32_t* n_out, int32_t* root,
                  size_t* err_pos) {
    if (!pattern && len) return fail(RXG_EINVAL, "null pattern");
    try {
        const rxg::Expr e = rxg::parse(std::string_view(pattern ? pattern : "", len));
        const int32_t n = static_cast<int32_t>(e.nodes.size());
        if (n_out) *n_out = n;
        if (root) *root = e.root;
        for (int32_t i = 0; out && i < n && i < cap; ++i) {
            const rxg::ExprNode& x = e.nodes[static_cast<size_t>(i)];
            out[i] = rxg_ast_node{x.kind, {0, 0, 0}, x.sym, x.left, x.right};
        }
        return RXG_OK;
    } catch (const rxg::ParseError& e) {
        if (err_pos) *err_pos = e.pos;
        return fail(RXG_EPARSE, e.what());
    } catch (const rxg::Utf8Error& e) {
        if (err_pos) *err_pos = e.at;
        return fail(RXG_EUTF8, e.what());
    }
}

int rxg_print_ast(const rxg_ast_node* nodes, int32_t n, int32_t root, char* out, size_t cap, size_t* out_len) {
    rxg::Expr e;
    if (int rc = expr_of(nodes, n, root, &e)) return rc;
    const std::string s = rxg::print(e);
    if (out_len) *out_len = s.size();
    if (out && cap) {
        const size_t k = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), k);
        out[k] = '\0';
    }
    return RXG_OK;
}

int rxg_compile_ast(const rxg_ast_node* nodes, int32_t n, int32_t root, rxg_node* heap, int32_t* knodes, int32_t cap,
                    int32_t* n_out) {
    rxg::Expr e;
    if (int rc = expr_of(nodes, n, root, &e)) return rc;
    const rxg::Heap h = rxg::compile(e);
    if (n_out) *n_out = h.size();
    const int32_t k = std::min(cap, h.size());
    if (heap && k > 0) std::memcpy(heap, h.nodes.data(), static_cast<size_t>(k) * sizeof(rxg_node));
    if (knodes && k > 0) std::memcpy(knodes, h.knodes.data(), static_cast<size_t>(k) * sizeof(int32_t));
    return RXG_OK;
}

int rxg_evolve(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns, int32_t* out,
               int32_t* n_out, uint64_t* enqueued) {
    std::string why;
    if (!heap_ok(nodes, knodes, n, &why)) return fail(RXG_EHEAP, why);
    if (!set_ok(s, ns, n) || !out || !n_out) return fail(RXG_EINVAL, "bad set");
    // lockstep.cpp:10-35: seed with the non-null members in set order, FIFO,
    // each address enqueued at most once; Chr nodes are output, not expanded
    std::vector<char> seen(static_cast<size_t>(n), 0);
    std::deque<int32_t> work;
    uint64_t enq = 0;
    for (int32_t i = 0; i < ns; ++i) {
        const int32_t p = s[i];
        if (p < 0 || seen[static_cast<size_t>(p)]) continue;
        seen[static_cast<size_t>(p)] = 1;
        work.push_back(p);
        ++enq;
    }
    int32_t k = 0;
    while (!work.empty()) {
        const int32_t p = work.front();
        work.pop_front();
        if (nodes[p].kind == RXG_NODE_CHR) {
            out[k++] = p;
            continue;
        }
        int32_t succ[2];
        const int m = eps_succ(nodes, knodes, p, succ);
        for (int j = 0; j < m; ++j) {
            const int32_t q = succ[j];
            if (q < 0 || seen[static_cast<size_t>(q)]) continue;
            seen[static_cast<size_t>(q)] = 1;
            work.push_back(q);
            ++enq;
        }
    }
    *n_out = k;
    if (enqueued) *enqueued += enq;
    return RXG_OK;
}

int rxg_eps_reaches_null(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns,
                         int32_t* result) {
    std::string why;
    if (!heap_ok(nodes, knodes, n, &why)) return fail(RXG_EHEAP, why);
    if (!set_ok(s, ns, n) || !result) return fail(RXG_EINVAL, "bad set");
    // lockstep.cpp:42-62
    *result = 0;
    std::vector<char> seen(static_cast<size_t>(n), 0);
    std::deque<int32_t> work;
    for (int32_t i = 0; i < ns; ++i) {
        const int32_t p = s[i];
        if (p < 0) {
            *result = 1;
            return RXG_OK;
        }
        if (seen[static_cast<size_t>(p)]) continue;
        seen[static_cast<size_t>(p)] = 1;
        work.push_back(p);
    }
    while (!work.empty()) {
        const int32_t p = work.front();
        work.pop_front();
        int32_t succ[2];
        const int m = eps_succ(nodes, knodes, p, succ);
        for (int j = 0; j < m; ++j) {
            const int32_t q = succ[j];
            if (q < 0) {
                *result = 1;
                return RXG_OK;
            }
            if (seen[static_cast<size_t>(q)]) continue;
            seen[static_cast<size_t>(q)] = 1;
            work.push_back(q);
        }
    }
    return RXG_OK;
}

int rxg_step_char(const rxg_node* nodes, const int32_t* knodes, int32_t n, const int32_t* s, int32_t ns, uint32_t a,
                  int32_t* out, int32_t* n_out) {
    std::string why;
    if (!heap_ok(nodes, knodes, n, &why)) return fail(RXG_EHEAP, why);
    if (!set_ok(s, ns, n) || !out || !n_out) return fail(RXG_EINVAL, "bad set");
    // lockstep.cpp:64-73 (char_successor, pwpi.cpp:22-27); the output is a set:
    // sorted and deduplicated, null (-1) first like std::set<Addr>
    std::vector<int32_t> next;
    for (int32_t i = 0; i < ns; ++i) {
        const int32_t p = s[i];
        if (p < 0) continue;
        if (nodes[p].kind != RXG_NODE_CHR)
            return fail(RXG_EINVAL, "step_char: unevolved member p" + std::to_string(p));
        if (nodes[p].sym == a) next.push_back(knodes[p]);
    }
    std::sort(next.begin(), next.end());
    next.erase(std::unique(next.begin(), next.end()), next.end());
    std::copy(next.begin(), next.end(), out);
    *n_out = static_cast<int32_t>(next.size());
    return RXG_OK;
}

}  // extern "C"
