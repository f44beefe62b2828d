// Host front end: UTF-8, parser, heap layout. See frontend.hpp for the
// reference correspondence of every entry point.
#include "frontend.hpp"
#include "rxg_utf8.hpp"

#include <sstream>

namespace rxg {

// ── UTF-8 (reference utf8.cpp:16-46) ──────────────────────────────────

std::u32string decode_utf8(std::string_view bytes) {
    static constexpr char32_t kMin[5] = {0, 0, 0x80, 0x800, 0x10000};
    std::u32string out;
    out.reserve(bytes.size());
    const size_t n = bytes.size();
    size_t i = 0;
    while (i < n) {
        const uint32_t b0 = static_cast<uint8_t>(bytes[i]);
        if (b0 < 0x80) {
            out.push_back(b0);
            ++i;
            continue;
        }
        int len;
        char32_t cp;
        if ((b0 & 0xE0u) == 0xC0u) {
            len = 2; cp = b0 & 0x1Fu;
        } else if ((b0 & 0xF0u) == 0xE0u) {
            len = 3; cp = b0 & 0x0Fu;
        } else if ((b0 & 0xF8u) == 0xF0u) {
            len = 4; cp = b0 & 0x07u;
        } else {
            throw Utf8Error(i);
        }
        if (i + static_cast<size_t>(len) > n) throw Utf8Error(i);
        for (int k = 1; k < len; ++k) {
            const uint32_t b = static_cast<uint8_t>(bytes[i + k]);
            if ((b & 0xC0u) != 0x80u) throw Utf8Error(i + k);
            cp = (cp << 6) | (b & 0x3Fu);
        }
        if (cp < kMin[len] || cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) throw Utf8Error(i);
        out.push_back(cp);
        i += static_cast<size_t>(len);
    }
    return out;
}

std::string encode_utf8(char32_t cp) {
    std::string s;
    rxg::append_utf8(s, cp);
    return s;
}

// ── Parser (reference regex.cpp:73-144, 186-194) ──────────────────────
//
// Grammar: alt := seq ('|' seq)*   seq := star star*   star := atom '*'*
//          atom := '(' ')' | '(' alt ')' | '\' any | literal
// Binary operators are left-associative, so alternation and concatenation
// chains come out left-deep, exactly like the reference.

namespace {

bool is_meta(char32_t c) { return c == U'(' || c == U')' || c == U'|' || c == U'*' || c == U'\\'; }

class Parser {
public:
    Parser(const std::u32string& text, Expr& out) : t_(text), ex_(out) {}

    int32_t run() {
        int32_t e = alternation();
        if (i_ < t_.size()) fail("unbalanced parentheses");   // only a stray ')' stops alternation()
        return e;
    }

private:
    const std::u32string& t_;
    Expr& ex_;
    size_t i_ = 0;

    [[noreturn]] void fail(const char* msg) const { throw ParseError(i_, msg); }
    bool done() const { return i_ >= t_.size(); }
    bool starts_atom() const {
        if (done()) return false;
        const char32_t c = t_[i_];
        return c == U'(' || c == U'\\' || !is_meta(c);
    }
    int32_t make(uint8_t kind, uint32_t sym, int32_t l, int32_t r) {
        ex_.nodes.push_back(ExprNode{kind, sym, l, r});
        return static_cast<int32_t>(ex_.nodes.size() - 1);
    }

    int32_t alternation() {
        int32_t acc = sequence();
        while (!done() && t_[i_] == U'|') {
            ++i_;
            const int32_t rhs = sequence();
            acc = make(xAlt, 0, acc, rhs);
        }
        return acc;
    }

    int32_t sequence() {
        if (!starts_atom()) {
            if (done()) fail("unexpected end of pattern");
            if (t_[i_] == U'*') fail("dangling `*`");
            if (t_[i_] == U'|') fail("dangling `|`");
            fail("unbalanced parentheses");
        }
        int32_t acc = postfix();
        while (starts_atom()) {
            const int32_t rhs = postfix();
            acc = make(xSeq, 0, acc, rhs);
        }
        return acc;
    }

    int32_t postfix() {
        int32_t e = atom();
        while (!done() && t_[i_] == U'*') {
            ++i_;
            e = make(xStar, 0, e, -1);
        }
        return e;
    }

    int32_t atom() {
        const char32_t c = t_[i_];
        if (c == U'(') {
            const size_t open = i_++;
            if (!done() && t_[i_] == U')') {
                ++i_;
                return make(xEps, 0, -1, -1);
            }
            const int32_t inner = alternation();
            if (done() || t_[i_] != U')') {
                i_ = open;
                fail("unbalanced parentheses");
            }
            ++i_;
            return inner;
        }
        if (c == U'\\') {
            ++i_;
            if (done()) fail("illegal escape");
            return make(xChr, t_[i_++], -1, -1);
        }
        ++i_;
        return make(xChr, c, -1, -1);
    }
};

// Printing precedence (reference regex.cpp:146-180): alt 0, seq 1, star 2, atoms 3.
int prec(uint8_t kind) {
    switch (kind) {
    case xAlt: return 0;
    case xSeq: return 1;
    case xStar: return 2;
    default: return 3;
    }
}

void print_rec(const Expr& e, int32_t i, int min_prec, std::string& out) {
    const ExprNode& n = e.nodes[static_cast<size_t>(i)];
    const bool paren = prec(n.kind) < min_prec;
    if (paren) out += '(';
    switch (n.kind) {
    case xEps: out += "()"; break;
    case xChr:
        if (is_meta(n.sym)) out += '\\';
        out += encode_utf8(n.sym);
        break;
    case xStar:
        print_rec(e, n.left, 2, out);
        out += '*';
        break;
    case xSeq:
        print_rec(e, n.left, 1, out);
        print_rec(e, n.right, 2, out);
        break;
    case xAlt:
        print_rec(e, n.left, 0, out);
        out += '|';
        print_rec(e, n.right, 1, out);
        break;
    }
    if (paren) out += ')';
}

}  // namespace

Expr parse(std::string_view utf8) {
    const std::u32string text = decode_utf8(utf8);
    Expr e;
    e.nodes.reserve(text.size() + 1);
    Parser p(text, e);
    e.root = p.run();
    return e;
}

std::string print(const Expr& e) {
    std::string out;
    print_rec(e, e.root, 0, out);
    return out;
}

// ── Heap layout (reference heap.cpp:13-72) ────────────────────────────
//
// Addresses are handed out in level order: a FIFO over (expr, addr) pairs,
// children receive the next free addresses left then right. The continuation
// pass runs in ascending address order, which is a valid topological order
// because every parent precedes its children.

Heap compile(const Expr& e) {
    Heap h;
    const size_t total = e.nodes.size();   // arena holds exactly the tree (no sharing)
    h.nodes.assign(total, HeapNode{kEps, {0, 0, 0}, 0, kNull, kNull});
    h.knodes.assign(total, kNull);
    std::vector<std::pair<int32_t, Addr>> fifo;
    fifo.reserve(total);
    fifo.emplace_back(e.root, 0);
    Addr next_free = 1;
    for (size_t head = 0; head < fifo.size(); ++head) {
        const auto [xi, p] = fifo[head];
        const ExprNode& x = e.nodes[static_cast<size_t>(xi)];
        HeapNode& n = h.nodes[static_cast<size_t>(p)];
        switch (x.kind) {
        case xEps: n.kind = kEps; break;
        case xChr:
            n.kind = kChr;
            n.sym = x.sym;
            break;
        case xStar:
            n.kind = kStar;
            n.left = next_free++;
            fifo.emplace_back(x.left, n.left);
            break;
        case xSeq:
        case xAlt:
            n.kind = x.kind == xSeq ? kSeq : kAlt;
            n.left = next_free++;
            n.right = next_free++;
            fifo.emplace_back(x.left, n.left);
            fifo.emplace_back(x.right, n.right);
            break;
        }
    }
    if (static_cast<size_t>(next_free) != total) throw std::logic_error("compile: arena is not a tree");

    for (Addr p = 0; p < h.size(); ++p) {
        const HeapNode& n = h.nodes[static_cast<size_t>(p)];
        const Addr kp = h.knodes[static_cast<size_t>(p)];
        if (n.kind == kAlt) {
            h.knodes[static_cast<size_t>(n.left)] = kp;
            h.knodes[static_cast<size_t>(n.right)] = kp;
        } else if (n.kind == kSeq) {
            h.knodes[static_cast<size_t>(n.left)] = n.right;
            h.knodes[static_cast<size_t>(n.right)] = kp;
        } else if (n.kind == kStar) {
            h.knodes[static_cast<size_t>(n.left)] = p;
        }
    }
    return h;
}

bool check_knode(const Heap& h) {
    if (h.size() == 0 || h.knodes[0] != kNull) return false;
    auto k = [&](Addr a) { return h.knodes[static_cast<size_t>(a)]; };
    for (Addr p = 0; p < h.size(); ++p) {
        const HeapNode& n = h.nodes[static_cast<size_t>(p)];
        switch (n.kind) {
        case kAlt:
            if (k(n.left) != k(p) || k(n.right) != k(p)) return false;
            break;
        case kSeq:
            if (k(n.left) != n.right || k(n.right) != k(p)) return false;
            break;
        case kStar:
            if (k(n.left) != p) return false;
            break;
        default: break;
        }
    }
    return true;
}

std::string validate_heap(const Heap& h) {
    const Addr n = h.size();
    if (n == 0) return "empty heap";
    if (h.knodes.size() != h.nodes.size()) return "knode table size mismatch";
    auto in = [n](Addr a) { return a >= 0 && a < n; };
    for (Addr p = 0; p < n; ++p) {
        const HeapNode& x = h.nodes[static_cast<size_t>(p)];
        switch (x.kind) {
        case kEps:
        case kChr: break;
        case kStar:
            if (!in(x.left)) return "star child out of range at p" + std::to_string(p);
            break;
        case kAlt:
        case kSeq:
            if (!in(x.left) || !in(x.right)) return "child out of range at p" + std::to_string(p);
            break;
        default: return "unknown node kind at p" + std::to_string(p);
        }
        const Addr k = h.knodes[static_cast<size_t>(p)];
        if (k != kNull && !in(k)) return "knode out of range at p" + std::to_string(p);
    }
    return "";
}

// ── Dump format (reference heap.cpp:169-260) ──────────────────────────

namespace {

std::string addr_name(Addr p) { return p == kNull ? "null" : "p" + std::to_string(p); }

Addr parse_addr(const std::string& s) {
    if (s == "null") return kNull;
    if (s.size() < 2 || s[0] != 'p') throw std::runtime_error("bad address: " + s);
    Addr v = 0;
    for (size_t i = 1; i < s.size(); ++i) {
        if (s[i] < '0' || s[i] > '9') throw std::runtime_error("bad address: " + s);
        v = v * 10 + (s[i] - '0');
    }
    return v;
}

}  // namespace

std::string dump(const Heap& h) {
    std::string out;
    for (Addr p = 0; p < h.size(); ++p) {
        const HeapNode& n = h.nodes[static_cast<size_t>(p)];
        out += addr_name(p);
        out += '\t';
        switch (n.kind) {
        case kEps: out += "eps"; break;
        case kChr: out += "char " + encode_utf8(n.sym); break;
        case kAlt: out += "alt " + addr_name(n.left) + " " + addr_name(n.right); break;
        case kSeq: out += "seq " + addr_name(n.left) + " " + addr_name(n.right); break;
        case kStar: out += "star " + addr_name(n.left); break;
        }
        out += '\t';
        out += addr_name(h.knodes[static_cast<size_t>(p)]);
        out += '\n';
    }
    return out;
}

Heap parse_dump(std::string_view text) {
    Heap h;
    std::istringstream in{std::string(text)};
    std::string line;
    size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty()) continue;
        auto err = [&](const std::string& m) {
            return std::runtime_error("dump line " + std::to_string(lineno) + ": " + m);
        };
        const size_t t1 = line.find('\t');
        const size_t t2 = t1 == std::string::npos ? std::string::npos : line.find('\t', t1 + 1);
        if (t2 == std::string::npos) throw err("expected three tab-separated columns");
        if (parse_addr(line.substr(0, t1)) != h.size()) throw err("rows out of order");
        std::istringstream cols{line.substr(t1 + 1, t2 - t1 - 1)};
        std::string op;
        cols >> op;
        HeapNode n{kEps, {0, 0, 0}, 0, kNull, kNull};
        if (op == "eps") {
            n.kind = kEps;
        } else if (op == "char") {
            std::string s;
            cols >> s;
            const std::u32string d = decode_utf8(s);
            if (d.size() != 1) throw err("char operand must be one scalar");
            n.kind = kChr;
            n.sym = d[0];
        } else if (op == "alt" || op == "seq") {
            std::string l, r;
            cols >> l >> r;
            n.kind = op == "alt" ? kAlt : kSeq;
            n.left = parse_addr(l);
            n.right = parse_addr(r);
        } else if (op == "star") {
            std::string l;
            cols >> l;
            n.kind = kStar;
            n.left = parse_addr(l);
        } else {
            throw err("unknown node form: " + op);
        }
        h.nodes.push_back(n);
        h.knodes.push_back(parse_addr(line.substr(t2 + 1)));
    }
    if (h.size() == 0) throw std::runtime_error("empty dump");
    const std::string bad = validate_heap(h);
    if (!bad.empty()) throw std::runtime_error("dump: " + bad);
    return h;
}

}  // namespace rxg
