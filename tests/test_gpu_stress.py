"""Stress parity of the line kernels at sizes and shapes the synthetic
configs do not reach: long-tailed line lengths (lines spanning many ranges),
no delimiter at all, only delimiters, lines ending exactly on range
boundaries, tiny forced ranges, and both TMA table layouts. Every count is
checked against the CPU oracle (or, at sizes the oracle cannot finish in
seconds, against the independent bitset engine and per-line results)."""
import os

import numpy as np
import pytest

from oracle_bind import Oracle
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu

PATS = {
    "c": None,   # filled lazily: rx.synth_pattern("c") (direct layout)
    "d": None,   # rx.synth_pattern("d") (class layout)
    "abb": "(a|b)*abb",
    "empty_ok": "(a|b| )*",
}


ALPHA = {"c": b"abcdefgh ERORWANFIL", "d": b"abcdefghijklmnopqrstuvwxyz  ", "abb": b"ab ", "empty_ok": b"ab "}


def _pat(k):
    if k in ("c", "d"):
        return rx.synth_pattern(k)
    return PATS[k]


def _dev_count(m, text, engine="auto"):
    import torch

    d = torch.zeros(len(text) + 64, dtype=torch.uint8, device="cuda")
    if len(text):
        d[: len(text)].copy_(torch.from_numpy(np.ascontiguousarray(text)))
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, cnt, nbytes=len(text), engine=engine)
    torch.cuda.synchronize()
    return int(cnt.item())


def _long_tailed(seed, total, alphabet=b"abcdefgh ERORWANFIL", long_every=50, long_len=(20_000, 400_000)):
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(alphabet, np.uint8)
    out, n = [], 0
    while n < total:
        if rng.integers(0, long_every) == 0:
            L = int(rng.integers(*long_len))
        else:
            L = int(rng.integers(0, 200))
        line = alpha[rng.integers(0, len(alpha), L)]
        out.append(line)
        out.append(np.array([10], np.uint8))
        n += L + 1
    return np.concatenate(out)[:total]


@pytest.mark.parametrize("key", ["c", "d", "abb", "empty_ok"])
@pytest.mark.parametrize("chunk", [None, "96", "4096"])
def test_long_tailed_lines_all_range_sizes(key, chunk):
    pat = _pat(key)
    text = _long_tailed(len(key), 3 << 20, ALPHA[key])
    want, _ = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    try:
        rx.set_option("RXG_LINE_CHUNK", chunk)
        m = rx.Matcher(pat, device=0)
        assert _dev_count(m, text) == want
        c, r = m.match_batch(text, 10, results=True)
        assert c == want and int(r.sum()) == want
    finally:
        rx.set_option("RXG_LINE_CHUNK", None)


@pytest.mark.parametrize("key", ["c", "abb", "empty_ok"])
def test_no_delimiter_is_one_string(key):
    pat = _pat(key)
    rng = np.random.default_rng(3)
    text = np.frombuffer(b"ab ", np.uint8)[rng.integers(0, 3, 24 << 20)]
    text[-3:] = np.frombuffer(b"abb", np.uint8)
    m = rx.Matcher(pat, device=0)
    one = m.lockstep_accepts(text.tobytes())
    assert _dev_count(m, text) == int(one)
    assert _dev_count(m, text, "bitset") == int(one)


@pytest.mark.parametrize("key", ["c", "d", "abb", "empty_ok"])
def test_only_delimiters(key):
    pat = _pat(key)
    text = np.full(8 << 20, 10, np.uint8)
    empty = Oracle(rx.compile(rx.parse(pat))).accepts(b"")
    m = rx.Matcher(pat, device=0)
    assert _dev_count(m, text) == (len(text) if empty else 0)
    c, r = m.match_batch(text[: 1 << 20], 10, results=True)
    assert c == ((1 << 20) if empty else 0)


@pytest.mark.parametrize("key", ["c", "d"])
@pytest.mark.parametrize("line_len", [95, 96, 97, 4095, 4096])
def test_lines_on_range_boundaries(key, line_len):
    """Every line exactly line_len bytes including '\\n' with the range size
    forced to 96 / 4096: delimiters land on, before and after every boundary."""
    pat = _pat(key)
    rng = np.random.default_rng(line_len)
    n_lines = (2 << 20) // line_len
    alpha = np.frombuffer(ALPHA[key], np.uint8)
    body = alpha[rng.integers(0, len(alpha), (n_lines, line_len))]
    body[:, -1] = 10
    # a keyword in every third line so the count is not trivial
    kw = np.frombuffer(b"ERROR", np.uint8)
    if line_len > 10:
        body[::3, 2:7] = kw
    text = body.reshape(-1)
    want, _ = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    try:
        for chunk in ("96", "4096"):
            rx.set_option("RXG_LINE_CHUNK", chunk)
            m = rx.Matcher(pat, device=0)
            assert _dev_count(m, text) == want, chunk
    finally:
        rx.set_option("RXG_LINE_CHUNK", None)


def test_full_size_cross_engine_long_tailed():
    """256 MiB of long-tailed lines: the TMA DFA kernel, the generic kernel
    with per-line results and the bitset engine agree (the oracle checks a
    prefix)."""
    pat = _pat("c")
    text = _long_tailed(11, 256 << 20, long_every=200)
    m = rx.Matcher(pat, device=0)
    a = _dev_count(m, text)
    b = _dev_count(m, text, "bitset")
    c, r = m.match_batch(text, 10, results=True)
    assert a == b == c == int(r.sum())
    cut = int(np.flatnonzero(text[: 8 << 20] == 10)[-1]) + 1
    want, wr = Oracle(rx.compile(rx.parse(pat))).match_batch(text[:cut], 10, 0)
    assert np.array_equal(r[: len(wr)], wr)


@pytest.mark.parametrize("key", ["c", "d", "abb"])
def test_generic_line_kernel_results(key):
    """The generic line kernel (k_lines: tables too large for the TMA
    layouts) forced with RXG_NO_LT, per-line results against the oracle and
    the TMA kernel."""
    pat = _pat(key)
    text = _long_tailed(7, 2 << 20, ALPHA[key], long_every=100, long_len=(2_000, 50_000))
    want_c, want_r = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    m = rx.Matcher(pat, device=0)
    c1, r1 = m.match_batch(text, 10, results=True)
    with rx.option("RXG_NO_LT", 1):
        c2, r2 = m.match_batch(text, 10, results=True)
        c3 = _dev_count(m, text)
    assert c1 == c2 == c3 == want_c
    assert np.array_equal(r1, want_r) and np.array_equal(r2, want_r)


@pytest.mark.parametrize("stride", [32, 64, 96, 48, 7, 33])
@pytest.mark.parametrize("n", [1, 95, 96, 97, 20_011])
def test_fixed_stride_kernels(stride, n):
    """Fixed-stride batches: the TMA kernel (stride a multiple of 32), the LDG
    kernel (RXG_NO_FIXED_TMA, and stride 48) and the oracle agree per string."""
    rng = np.random.default_rng(stride * 1000 + n)
    for pat in ["(a|b)*abb", rx.synth_pattern("b"), "(a|())(a|())aa(a|b)*"]:
        text = np.frombuffer(b"ab", np.uint8)[rng.integers(0, 2, n * stride)]
        if "abb" in pat:
            text.reshape(n, stride)[::3, -3:] = np.frombuffer(b"abb", np.uint8)
        want_c, want_r = Oracle(rx.compile(rx.parse(pat))).match_batch(text, -1, stride)
        m = rx.Matcher(pat, device=0)
        c1, r1 = m.match_batch(text, -1, stride, results=True)
        with rx.option("RXG_NO_FIXED_TMA", 1):
            c2, r2 = m.match_batch(text, -1, stride, results=True)
        assert c1 == c2 == want_c, (pat, c1, c2, want_c)
        assert np.array_equal(r1, want_r) and np.array_equal(r2, want_r)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_mid_size_dfas_both_layouts(k):
    """(a|b)*a(a|b)^k needs 2^(k+1) live states: 17 and 33 take the direct layouts
    (33 only with two rows per column word), 65 the class layout."""
    pat = "(a|b)*a" + "(a|b)" * k
    m = rx.Matcher(pat, device=0)
    assert m.info()["dfa_states"] == 2 ** (k + 1) + 1   # + the dead state
    rng = np.random.default_rng(k)
    lines = [bytes(rng.choice([97, 98, 99], size=int(rng.integers(0, 40))).astype(np.uint8)) for _ in range(20000)]
    text = np.frombuffer(b"\n".join(lines) + b"\n", np.uint8)
    o = Oracle(rx.compile(rx.parse(pat)))
    want_c, want_r = o.match_batch(text, 10, 0)
    m.tune(text[: 1 << 18])
    assert _dev_count(m, text) == want_c
    c, r = m.match_batch(text, 10, results=True)
    assert c == want_c and np.array_equal(r, want_r)
    w = np.frombuffer(b"ab" * 300_000 + b"a" + b"b" * k, np.uint8)
    for eng in ("chunked", "dfa_seq"):
        assert m.lockstep_accepts(w.tobytes(), eng) == o.accepts(w.tobytes()), eng


def test_back_to_back_launches_on_streams():
    """The TMA kernels publish counts through a per-stream slot that the last
    CTA re-zeroes (no memset launch): many launches back to back, on two
    streams at once and mixed with the other kernels, all exact."""
    import torch

    pat = _pat("c")
    text = _long_tailed(5, 4 << 20, ALPHA["c"], long_every=500, long_len=(1000, 5000))
    want, _ = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    m = rx.Matcher(pat, device=0)
    d = torch.zeros(len(text) + 64, dtype=torch.uint8, device="cuda")
    d[: len(text)].copy_(torch.from_numpy(text))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c1 = torch.full((50,), -1, dtype=torch.int64, device="cuda")
    c2 = torch.full((50,), -1, dtype=torch.int64, device="cuda")
    for i in range(50):
        m.match_batch_device(d, c1[i:i + 1], nbytes=len(text), stream=s1)
        m.match_batch_device(d, c2[i:i + 1], nbytes=len(text), stream=s2, engine="dfa" if i % 3 else "bitset")
    torch.cuda.synchronize()
    assert (c1 == want).all() and (c2 == want).all()
    # single-string engine on the same streams (its slot holds the ticket and the repair flag)
    w = torch.from_numpy(rx.synth_input("a")).cuda()
    acc = torch.zeros(20, dtype=torch.int32, device="cuda")
    for i in range(20):
        m2 = rx.Matcher(rx.synth_pattern("a"), device=0) if i == 0 else m2
        m2.match_one_device(w, acc[i:i + 1], stream=s1 if i % 2 else s2)
    torch.cuda.synchronize()
    assert acc.all()


@pytest.mark.parametrize("chunk", [0, 128, 256, 96])
def test_chunked_cooperative_path_wrong_guesses(chunk):
    """Strings >= 4 MiB take the cooperative launch (seams checked in-stream by
    the later neighbour, parallel repair rounds). Non-synchronizing automata
    with a 16-byte lookback guess wrong at many seams; the answer must still
    equal the sequential walk's."""
    import torch

    rng = np.random.default_rng(17)
    for p in ["(aa)*", "(aaa)*", "((a|b)(a|b))*", "(ab|ba)*a", "(a|b)*abb"]:
        m = rx.Matcher(p, device=0)
        for n in (4 << 20, (6 << 20) + 5, (12 << 20) + 1):
            if p in ("(aa)*", "(aaa)*"):
                w = np.full(n, 97, np.uint8)
                if rng.integers(0, 2):
                    w[int(rng.integers(0, n))] = 98   # one wrong byte somewhere
            else:
                w = rng.choice([97, 98], size=n).astype(np.uint8)
            d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
            d[:n].copy_(torch.from_numpy(w))
            acc = torch.zeros(1, dtype=torch.int32, device="cuda")
            ref = torch.zeros(1, dtype=torch.int32, device="cuda")
            rep = torch.zeros(1, dtype=torch.int64, device="cuda")
            m.match_one_ex(d, acc, "chunked", nbytes=n, chunk=chunk, lookback=16, d_repairs=rep)
            m.match_one_ex(d, ref, "dfa_seq", nbytes=n)
            torch.cuda.synchronize()
            assert bool(acc.item()) == bool(ref.item()), (p, n, chunk)


@pytest.mark.parametrize("key", ["c", "abb", "empty_ok"])
def test_very_long_lines_warp_cooperative(key):
    """Lines of several MB: the range that owns one hands it to its whole warp
    after 16 KB (kCoopTail), which walks it in 1 KB blocks with checked guesses.
    Counts and per-line results against the oracle; the 24 MB buffer must not
    take seconds (the serial finish ran at ~25 ns/byte)."""
    import time

    pat = _pat(key)
    rng = np.random.default_rng(11)
    alpha = np.frombuffer(ALPHA[key], np.uint8)
    parts = []
    for n in (100, 9_000_000, 30, 0, 5_000_001, 77, 8_000_000, 12):
        parts.append(alpha[rng.integers(0, len(alpha), n)])
        parts.append(np.array([10], np.uint8))
    text = np.concatenate(parts)[:-1]   # unterminated last line
    want_c, want_r = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    m = rx.Matcher(pat, device=0)
    assert _dev_count(m, text) == want_c
    t0 = time.perf_counter()
    assert _dev_count(m, text) == want_c
    dt = time.perf_counter() - t0
    c, r = m.match_batch(text, 10, results=True)
    assert c == want_c and np.array_equal(r, want_r)
    assert dt < 0.25, dt


@pytest.mark.parametrize("key", ["c", "d", "abb", "empty_ok"])
@pytest.mark.parametrize("chunk", [None, "96", "4096"])
def test_short_lines_results_every_offset(key, chunk):
    """Lines of 0-40 bytes: delimiters at every offset of the 32-byte groups the
    per-line walk records from its bit masks, runs of empty lines, and lines
    crossing group and range boundaries. Per-line results against the oracle."""
    pat = _pat(key)
    rng = np.random.default_rng(17)
    alpha = np.frombuffer(ALPHA[key], np.uint8)
    lens = rng.integers(0, 41, 60_000)
    lens[rng.random(len(lens)) < 0.2] = 0
    parts = []
    for n in lens:
        parts.append(alpha[rng.integers(0, len(alpha), n)])
        parts.append(np.array([10], np.uint8))
    text = np.concatenate(parts)
    if key == "c":   # keywords so that lines match
        for p in rng.integers(0, len(text) - 5, 4000):
            text[p:p + 5] = np.frombuffer(b"ERROR", np.uint8)
    want_c, want_r = Oracle(rx.compile(rx.parse(pat))).match_batch(text, 10, 0)
    try:
        rx.set_option("RXG_LINE_CHUNK", chunk)
        m = rx.Matcher(pat, device=0)
        c, r = m.match_batch(text, 10, results=True)
        assert c == want_c and np.array_equal(r, want_r)
    finally:
        rx.set_option("RXG_LINE_CHUNK", None)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_per_line_results_tma_vs_generic_random_mixes(seed):
    """Per-line results of the TMA line kernel (range-local bits, per-tile
    totals, the bit-array scatter with 16-byte stores) against the generic
    kernel (RXG_NO_LT), on buffers mixing empty, short and long lines, at
    sizes that leave ragged remainders and groups with > 64 lines per range."""
    import torch

    rng = np.random.default_rng(seed)
    pat = "(a|b)*a(a|b)"
    m = rx.Matcher(pat, device=0)
    for size in (1, 31, 4097, 65_537, 1 << 20, (3 << 20) + 5, (24 << 20) + 11):
        mode = rng.integers(0, 3)
        if mode == 0:      # short lines (many lines per range: the per-range fallback)
            w = rng.choice(np.frombuffer(b"ab\n", np.uint8), size=size, p=[0.3, 0.3, 0.4])
        elif mode == 1:    # ~100-byte lines
            w = rng.choice(np.frombuffer(b"ab\n", np.uint8), size=size, p=[0.495, 0.495, 0.01])
        else:              # long lines with bursts of empty ones
            w = rng.choice(np.frombuffer(b"ab\n", np.uint8), size=size, p=[0.4985, 0.4985, 0.003])
            k = int(rng.integers(0, max(1, size - 200)))
            w[k:k + 150] = 10
        w = np.ascontiguousarray(w.astype(np.uint8))
        c1, r1 = m.match_batch(w, 10, results=True)
        rx.set_option("RXG_NO_LT", 1)
        try:
            m2 = rx.Matcher(pat, device=0)
            c2, r2 = m2.match_batch(w, 10, results=True)
        finally:
            rx.set_option("RXG_NO_LT", None)
        assert c1 == c2 == int(r1.sum()), (seed, size, mode)
        assert np.array_equal(r1, r2), (seed, size, mode, int(np.argmax(r1 != r2)))
        torch.cuda.synchronize()
