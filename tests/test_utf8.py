"""UTF-8 decode checking: the oracle restatement of
rx::decode_utf8 (utf8.cpp:16-46) pinned against the reference library on
fuzzed byte strings (CPU), and the device check (rxg_utf8_check) against the
oracle (GPU), including the per-string semantics of the `rxvm match` loop."""
import numpy as np
import pytest

from oracle_bind import Oracle, Ref
from paper_1108_3126_b200 import rx

# byte pools that hit every branch of decode_utf8: ASCII, continuation bytes,
# 2/3/4-byte leads (incl. overlong C0/C1/E0/F0 and out-of-range F4-F7), F8-FF
_POOL = np.array([0x61, 0x0A, 0x20, 0x7F, 0x80, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1, 0xC2, 0xDF, 0xE0, 0xED, 0xEF,
                  0xF0, 0xF4, 0xF5, 0xF7, 0xF8, 0xFF], np.uint8)


def _fuzz_strings(seed, count, max_len=12):
    rng = np.random.default_rng(seed)
    out = []
    valid = ["a", "é", "ߧ", "中", "퟿", "", "￿", "😀", "\U0010ffff", "\n"]
    for _ in range(count):
        mode = rng.integers(0, 3)
        if mode == 0:   # structured: valid scalars with a few corrupted bytes
            s = bytearray("".join(rng.choice(valid) for _ in range(rng.integers(0, 6))).encode())
            for _ in range(rng.integers(0, 3)):
                if s:
                    s[rng.integers(0, len(s))] = int(rng.choice(_POOL))
            out.append(bytes(s))
        elif mode == 1:   # uniform pool bytes
            out.append(bytes(rng.choice(_POOL, size=rng.integers(0, max_len))))
        else:   # fully random bytes
            out.append(bytes(rng.integers(0, 256, size=rng.integers(0, max_len), dtype=np.uint8)))
    return out


KNOWN = [
    (b"", None), (b"abc", None), ("é中😀".encode(), None),
    (b"\x80", 0), (b"a\xbf", 1), (b"\xc3", 0), (b"\xc3a", 1), (b"\xc0\x80", 0), (b"\xc1\xbf", 0),
    (b"\xe0\x80\x80", 0), (b"\xe0\xa0\x80", None), (b"\xed\xa0\x80", 0), (b"\xed\x9f\xbf", None),
    (b"\xf0\x80\x80\x80", 0), (b"\xf4\x90\x80\x80", 0), (b"\xf4\x8f\xbf\xbf", None), (b"\xf8", 0),
    (b"ab\xe4\xb8", 2), (b"ab\xe4\xb8a", 4), (b"\xff\xc3", 0), ("é".encode() + b"\xa9", 2),
]


@pytest.mark.parametrize("b,want", KNOWN)
def test_oracle_known_answers(b, want):
    assert Oracle.decode_utf8_error(b) == want
    if Ref.available():
        assert Ref.decode_utf8_error(b) == want


def test_oracle_matches_reference_decode_utf8_fuzz():
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    bad = [s for s in _fuzz_strings(1, 20000) if Oracle.decode_utf8_error(s) != Ref.decode_utf8_error(s)]
    assert not bad, bad[:5]


def test_oracle_per_string_offsets():
    """first_bad over a buffer = offset of the first failing string + N."""
    strings = [b"ok", b"\xc3", b"x\xff"]
    text = b"\n".join(strings) + b"\n"
    assert Oracle.utf8_first_bad(text, 10) == 3
    # decoded as one string the lead runs into the delimiter: error at the '\n'
    assert Oracle.utf8_first_bad(text, -1, 0) == 4
    assert Oracle.utf8_first_bad(b"ab\xc3\xa9cd", -1, 3) == 2   # stride 3 cuts the 2-byte sequence
    assert Oracle.utf8_first_bad(b"ab\xc3\xa9cd", -1, 2) is None


# ── device ──

def _device_check(text, delimiter=-1, stride=0, offset=0):
    import torch

    buf = torch.zeros(len(text) + 32, dtype=torch.uint8)
    if len(text):
        buf[offset:offset + len(text)] = torch.from_numpy(np.frombuffer(bytes(text), np.uint8).copy())
    d = buf.cuda()
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    rx.utf8_check_device(d.data_ptr() + offset, len(text), out, delimiter, stride)
    torch.cuda.synchronize()
    v = int(out.item())
    return None if v == -1 else v


@pytest.mark.gpu
def test_device_known_answers_and_fuzz():
    for b, want in KNOWN:
        assert rx.utf8_check(b) == want, b
    strings = _fuzz_strings(2, 3000, max_len=40)
    for s in strings[:600]:
        assert rx.utf8_check(s) == Oracle.decode_utf8_error(s), s
    # whole fuzz corpus as one buffer, per line / per stride / as one string, any alignment
    text = b"\n".join(s.replace(b"\n", b"") for s in strings) + b"\n"
    for off in (0, 1, 7, 15):
        assert _device_check(text, 10, 0, off) == Oracle.utf8_first_bad(text, 10), off
        assert _device_check(text, -1, 0, off) == Oracle.utf8_first_bad(text, -1, 0), off
    st = text[: len(text) // 7 * 7]
    assert _device_check(st, -1, 7, 3) == Oracle.utf8_first_bad(st, -1, 7)


@pytest.mark.gpu
def test_device_single_error_positions_in_large_ascii():
    """One bad byte in a 48 MiB valid buffer, at positions around 16-byte
    groups, thread and grid boundaries and the end."""
    rng = np.random.default_rng(5)
    base = rx.synth_input("c", 48 << 20)
    n = len(base)
    assert rx.utf8_check(base, 10) is None
    for pos in [0, 15, 16, 17, 4095, 4096, 1 << 20, n // 2 + 3, n - 17, n - 2, n - 1]:
        for bad in (b"\xc3", b"\x80", b"\xff", b"\xe4\xb8"):
            t = base.copy()
            p = min(pos, n - len(bad))
            t[p:p + len(bad)] = np.frombuffer(bad, np.uint8)
            want = Oracle.utf8_first_bad(t, 10)
            assert rx.utf8_check(t, 10) == want, (pos, bad)
            assert rx.utf8_check(t, -1) == Oracle.utf8_first_bad(t, -1, 0), (pos, bad)
    # valid multi-byte text everywhere: no false positives
    u = ("".join(rng.choice(list("ab é中😀")) for _ in range(20000)) + "\n").encode() * 50
    assert rx.utf8_check(u, 10) is None


@pytest.mark.gpu
def test_device_single_corruptions_in_multibyte_text():
    """Valid mixed 1-4 byte text with one corrupted byte (every class of
    decode_utf8 error) at many offsets: exercises the vectorised group test
    against the per-byte rules, as one string, per line and per stride."""
    rng = np.random.default_rng(9)
    alpha = list("ab é中😀\U0010ffff\ud7ff\ue000")
    base = np.frombuffer(("".join(rng.choice(alpha) for _ in range(30000))).encode(), np.uint8)
    lines = base.copy()
    lines[rng.integers(0, len(lines), 2000)] = 10   # may cut sequences: per-line errors
    assert rx.utf8_check(base) is None
    corrupt = [0x80, 0xBF, 0xC0, 0xC1, 0xC3, 0xE0, 0xED, 0xE4, 0xF0, 0xF4, 0xF5, 0xF8, 0xFF, 0x41, 0xA0, 0x8F, 0x90]
    for t0, delim, stride in [(base, -1, 0), (lines, 10, 0), (base[: len(base) // 13 * 13], -1, 13)]:
        for trial in range(60):
            t = t0.copy()
            pos = int(rng.integers(0, len(t)))
            t[pos] = corrupt[trial % len(corrupt)]
            want = Oracle.utf8_first_bad(t, delim, stride)
            assert rx.utf8_check(t, delim, stride) == want, (delim, stride, pos, hex(t[pos]))


@pytest.mark.gpu
def test_match_batch_with_fused_utf8_check():
    pattern = "(a|é)*中"
    m = rx.Matcher(pattern, device=0)
    lines = ["aé中", "中", "x", "aaé中"] * 5000
    text = np.frombuffer(("\n".join(lines) + "\n").encode(), np.uint8)
    c0, r0 = m.match_batch(text, 10, results=True)
    c, r, bad = m.match_batch_utf8(text, 10, results=True)
    assert bad is None and c == c0 and np.array_equal(r, r0)
    t = text.copy()
    t[-3] = 0xFF   # inside the last line
    c, r, bad = m.match_batch_utf8(t, 10, results=True)
    assert bad == Oracle.utf8_first_bad(t, 10) == len(t) - 3
