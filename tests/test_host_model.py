"""CPU tests of the host logic behind the kernels: the position-form tables
(SURVEY.md §8(a) restatement), the memoized step table images and the
kernels' range-ownership / SKIP / tail rules, emulated on the host over the
exact images the GPU receives."""
import hashlib
import itertools
import json
from pathlib import Path

import numpy as np
import pytest

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

G = Path(__file__).parent / "golden"


def O(p):
    return Oracle(rx.compile(rx.parse(p)))


def H(p):
    return rx.Matcher(p, device=-1)


def strings(n, alpha="ab"):
    return [""] + ["".join(t) for k in range(1, n + 1) for t in itertools.product(alpha, repeat=k)]


@pytest.mark.parametrize("cfg,nodes,pos,words", [("a", 10, 5, 1), ("b", 191, 64, 3), ("c", 64, 31, 1),
                                                 ("d", 1024, 511, 16), ("e", 4096, 2048, 65)])
def test_config_shapes(cfg, nodes, pos, words):
    # N / |C| / W per config (W here counts the accept bit)
    i = H(rx.synth_pattern(cfg)).info()
    assert (i["nodes"], i["positions"]) == (nodes, pos)
    assert i["words"] == (pos + 1 + 31) // 32
    assert i["dfa_states"] > 0 and i["byte_symbols"] == 1


def test_position_form_equals_lockstep_sets_exhaustive():
    """E_i of the position form == evolve(S_i) of the reference at every step,
    for every regex <= 5 nodes and every string <= 4 over {a,b}."""
    d = json.loads((G / "lockstep_small.json").read_text())
    ws = d["strings"]
    for p, bits in d["accept"].items():
        m = H(p)
        pos_addr, _, _ = m.tables()
        o = O(p)
        for w, bit in zip(ws, bits):
            sets, acc = m.host_walk(w.encode())
            assert acc == (bit == "1"), (p, w)
            s = {0}
            for i, a in enumerate(w):
                e = o.evolve(s)
                row = sets[i]
                got = {int(pos_addr[q]) for q in range(len(pos_addr)) if (row[q >> 5] >> (q & 31)) & 1}
                assert got == e, (p, w, i)
                s = o.step_char(e, ord(a))
                if not s:
                    break


def test_emulated_line_kernels_match_oracle_on_configs():
    for cfg, n in [("c", 1 << 21), ("d", 1 << 20)]:
        pat = rx.synth_pattern(cfg)
        text = rx.synth_input(cfg, n)
        oc, ores = O(pat).match_batch(text, 10, 0)
        m = H(pat)
        for chunk in (16, 48, 1024, 4096):
            c, r = m.emulate_batch(text, 10, 0, chunk)
            assert c == oc and np.array_equal(r, ores), (cfg, chunk)
        if cfg == "c":
            for chunk in (32, 64, 3392, 6752):
                assert m.emulate_lines_tma(text, 10, chunk) == oc
            m.tune(text[: 1 << 18])
            for chunk in (32, 3392):
                assert m.emulate_lines_tma(text, 10, chunk) == oc


@pytest.mark.parametrize("text", [b"", b"\n", b"\n\n\n", b"ab", b"ab\n", b"\nab", b"a\nb\n\nab", b"ab\n" * 40,
                                  (b"abb\n\n" * 50)[:-3], b"x" * 100, b"abb\n" * 7 + b"a" * 70])
@pytest.mark.parametrize("pattern", ["a*", "ab", "()", "(a|b)*abb", "a|()", "(ab)*", "a**b"])
def test_emulated_line_edges(pattern, text):
    a = np.frombuffer(text, np.uint8) if text else np.zeros(0, np.uint8)
    oc, ores = O(pattern).match_batch(a, 10, 0)
    m = H(pattern)
    for chunk in (16, 32, 64):
        c, r = m.emulate_batch(a, 10, 0, chunk)
        assert c == oc and np.array_equal(r, ores)
        assert m.emulate_lines_tma(a, 10, max(chunk, 32)) == oc


def test_emulated_fixed_stride():
    pat = rx.synth_pattern("b")
    text = rx.synth_input("b", 32 * 3000)
    c, r = H(pat).emulate_batch(text, -1, 32)
    assert c == 3000 and r.all()
    rng = np.random.default_rng(0)
    t = rng.choice([97, 98], size=7 * 500).astype(np.uint8)
    for p in ["(a|b)*abb", "a*b*", "(ab|ba)*"]:
        oc, ores = O(p).match_batch(t, -1, 7)
        c, r = H(p).emulate_batch(t, -1, 7)
        assert c == oc and np.array_equal(r, ores)


def test_non_matching_bytes_behave_like_unmatched_scalars():
    """Bytes >= 0x80 (UTF-8 of scalars no ASCII literal matches) kill the set,
    exactly as the decoded scalar would in the reference."""
    m = H("(a|b)*abb")
    for w in ["abb", "aébb", "éabb", "ab中b", "aabb"]:
        _, acc = m.host_walk(w.encode())
        want = w in ("abb", "aabb")   # the reference decodes to scalars; é / 中 match no literal
        assert acc == want
        if Ref.available():
            assert RefHeap(b"(a|b)*abb").accepts(w) == want


def test_non_ascii_literals_match_as_utf8_chains():
    """Literals >= 0x80 become UTF-8 byte chains: same answers as the reference
    on decoded scalars, for valid UTF-8 inputs."""
    import random

    rng = random.Random(3)
    alpha = ["a", "b", "é", "中", "😀"]
    for p in ["é*", "(a|é)*中", "😀(a|b)*é", "a|é|中|😀", "(é中)*😀", "((é|b)*中)*"]:
        m = H(p)
        assert m.info()["byte_symbols"] == 1
        want = RefHeap(p.encode()) if Ref.available() else None
        for _ in range(150):
            w = "".join(rng.choice(alpha) for _ in range(rng.randint(0, 8)))
            _, acc = m.host_walk(w.encode())
            if want is not None:
                assert acc == want.accepts(w), (p, w)
        # the emulated line kernels agree with the host walk on a UTF-8 line buffer
        lines = ["".join(rng.choice(alpha) for _ in range(rng.randint(0, 8))) for _ in range(300)]
        text = np.frombuffer("\n".join(lines).encode() + b"\n", np.uint8)
        c, res = m.emulate_batch(text, 10, 0, 16)
        assert list(res) == [int(m.host_walk(l.encode())[1]) for l in lines]


def test_synth_generators_are_deterministic():
    d = json.loads((G / "configs.json").read_text())
    for cfg, e in d.items():
        assert hashlib.sha1(rx.synth_input(cfg, e["bytes"]).tobytes()).hexdigest() == e["input_sha1"]


def test_shard_bounds_split_on_string_boundaries():
    text = rx.synth_input("c", 1 << 20)
    for n in (1, 2, 3, 8):
        b = rx.shard_bounds(text, n, delimiter=10)
        assert b[0] == 0 and b[-1] == len(text) and all(x <= y for x, y in zip(b, b[1:]))
        for cut in b[1:-1]:
            assert text[cut - 1] == 10
        total = sum(O(rx.synth_pattern("c")).match_batch(text[lo:hi], 10, 0)[0] for lo, hi in zip(b, b[1:]))
        assert total == O(rx.synth_pattern("c")).match_batch(text, 10, 0)[0]
    t = rx.synth_input("b", 32 * 1001)
    b = rx.shard_bounds(t, 4, delimiter=-1, stride=32)
    assert all(x % 32 == 0 for x in b) and b[-1] == len(t)


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_dfa_tables_against_reference_random():
    rng = np.random.default_rng(1)
    for p in Ref.random_regexes(80, 20, seed=5, alphabet="abc"):
        m, r = H(p), RefHeap(p.encode())
        lines = [bytes(rng.choice([97, 98, 99], size=int(rng.integers(0, 12))).astype(np.uint8)) for _ in range(60)]
        text = np.frombuffer(b"\n".join(lines) + b"\n", np.uint8)
        rc, rr = r.match_batch(text, 10, 0)
        c, res = m.emulate_batch(text, 10, 0, 16)
        assert c == rc and np.array_equal(res, rr), p
        if m.info()["dfa_states"] <= 25:
            assert m.emulate_lines_tma(text, 10, 32) == rc


def test_minimised_memoized_step():
    """Moore refinement of the memoized step: the kernels only need each
    string's accept bit, so states with the same accept bit on every
    continuation merge. (e)'s keyword union is absorbed by the star of single
    letters ([a-z ]*abb: 1,209 E sets, 5 states); (d) halves. Per-string
    results of the minimised table equal the oracle's."""
    want = {"a": (5, 5), "c": (14, 14), "d": (624, 309), "e": (1209, 5)}
    for cfg, (sets, states) in want.items():
        i = rx.Matcher(rx.synth_pattern(cfg), device=-1).info()
        assert (i["dfa_sets"], i["dfa_states"]) == (sets, states), cfg
    rng = np.random.default_rng(8)
    for p in ["(a|b|ab|ba|aab)*abb", "((a|b)*a(a|b)|a)*", "(aa|ab|ba|bb)*", "(a|())*(b|())*a*", "((ab)*|(ba)*)*b"]:
        m = rx.Matcher(p, device=-1)
        i = m.info()
        assert 0 < i["dfa_states"] <= i["dfa_sets"]
        lines = [bytes(rng.choice([97, 98], size=int(rng.integers(0, 14))).astype(np.uint8)) for _ in range(3000)]
        text = np.frombuffer(b"\n".join(lines) + b"\n", np.uint8)
        ocount, ores = Oracle(rx.compile(rx.parse(p))).match_batch(text, 10, 0)
        count, res = m.emulate_batch(text, 10, 0, 64)
        assert count == ocount and np.array_equal(res, ores), p
