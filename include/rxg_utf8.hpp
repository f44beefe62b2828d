/*
 * rxg_utf8.hpp — the one UTF-8 encoder shared by the library front end,
 * the position-form builder and the header-only C++ facades.
 */
#ifndef RXG_UTF8_HPP
#define RXG_UTF8_HPP

#include <string>
#include <string_view>

namespace rxg {

// rx::encode_utf8 (proj/src/utf8.cpp:48-73): the encoding of one scalar,
// appended to `out` (same bit layout as the reference, including for values
// it never receives).
inline void append_utf8(std::string& out, char32_t cp) {
    if (cp < 0x80) {
        out += static_cast<char>(cp);
    } else if (cp < 0x800) {
        out += static_cast<char>(0xC0 | (cp >> 6));
        out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
        out += static_cast<char>(0xE0 | (cp >> 12));
        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
        out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
        out += static_cast<char>(0xF0 | (cp >> 18));
        out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
        out += static_cast<char>(0x80 | (cp & 0x3F));
    }
}

// Input symbols (rx::InputView, one char32_t each) -> the bytes the matcher
// consumes (include/rxg.h: every literal is matched as its UTF-8 encoding).
// A value that is not a Unicode scalar (a surrogate or > U+10FFFF) equals no
// pattern literal, so the reference can never step on it; it becomes 0xFF,
// a byte that occurs in no UTF-8 encoding and so matches no literal's chain.
// (Encoding it instead could alias a valid scalar: 0x1010000 would truncate
// to the bytes of U+10000.)
inline std::string symbols_to_bytes(std::u32string_view w) {
    std::string s;
    s.reserve(w.size());
    for (char32_t cp : w) {
        if (cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) s += static_cast<char>(0xFF);
        else append_utf8(s, cp);
    }
    return s;
}

}  // namespace rxg

#endif  // RXG_UTF8_HPP
