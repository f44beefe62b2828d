// Host front end of the B200 lockstep matcher.
//
// Restates the reference's syntax layer and heap layout with the same
// observable semantics (tree shapes, addresses, knode wiring, error
// positions), but with an index arena instead of shared_ptr trees:
//   decode_utf8        reference proj/src/utf8.cpp:16-46
//   parse              reference proj/src/regex.cpp:73-194 (left-assoc alt/seq, `()` = eps)
//   compile            reference proj/src/heap.cpp:13-72 (BFS addresses, knode pass)
//   dump / parse_dump  reference proj/src/heap.cpp:169-260
//   check_knode        reference proj/src/heap.cpp:106-128
//   eps successors     reference proj/src/pwpi.cpp:9-20 (Fig. 3)
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace rxg {

using Addr = int32_t;
inline constexpr Addr kNull = -1;

// Node kinds in the reference heap order (heap.hpp:18): Eps, Chr, Alt, Seq, Star.
enum NodeKind : uint8_t { kEps = 0, kChr = 1, kAlt = 2, kSeq = 3, kStar = 4 };

// Same 16-byte layout as rx::Node (heap.hpp:17-23): kind u8 (+pad), sym u32, left, right.
struct HeapNode {
    uint8_t kind;
    uint8_t pad_[3];
    uint32_t sym;
    int32_t left;
    int32_t right;
};
static_assert(sizeof(HeapNode) == 16, "HeapNode must match rx::Node layout");

struct Heap {
    std::vector<HeapNode> nodes;
    std::vector<Addr> knodes;
    int32_t size() const { return static_cast<int32_t>(nodes.size()); }
};

// Expression arena. Kinds follow rx::Regex::Kind order (regex.hpp:27):
// Eps, Chr, Star, Seq, Alt — note the different order from the heap.
enum ExprKind : uint8_t { xEps = 0, xChr = 1, xStar = 2, xSeq = 3, xAlt = 4 };
struct ExprNode {
    uint8_t kind;
    uint32_t sym;
    int32_t left;
    int32_t right;
};
struct Expr {
    std::vector<ExprNode> nodes;   // arena; children precede parents
    int32_t root = -1;
};

struct ParseError : std::runtime_error {
    size_t pos;
    ParseError(size_t p, const std::string& what)
        : std::runtime_error(what + " at position " + std::to_string(p)), pos(p) {}
};

struct Utf8Error : std::runtime_error {
    size_t at;
    explicit Utf8Error(size_t a)
        : std::runtime_error("invalid UTF-8 at byte " + std::to_string(a)), at(a) {}
};

std::u32string decode_utf8(std::string_view bytes);
std::string encode_utf8(char32_t cp);

Expr parse(std::string_view utf8);
std::string print(const Expr& e);
Heap compile(const Expr& e);

std::string dump(const Heap& h);
Heap parse_dump(std::string_view text);
bool check_knode(const Heap& h);

// Validates that a caller-supplied heap is well formed enough for the
// matcher: child/knode addresses in range, kinds known. Returns "" if ok.
std::string validate_heap(const Heap& h);

}  // namespace rxg
