"""Pins the CPU oracle (oracle/lockstep_oracle.c) to the reference: the golden
vectors of proj/tests/test_lockstep.cpp, the exhaustive small suite
(test_lockstep.cpp:60-72, acceptance criterion 3 shape) recorded from the
reference library in tests/golden/, and (when built) oracle/_ref directly."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

G = Path(__file__).parent / "golden"


def O(p):
    return Oracle(rx.compile(rx.parse(p)))


def test_evolve_goldens():
    # test_lockstep.cpp:15-23
    o = O("a**b")
    assert o.evolve({0}) == {4, 2}
    assert o.evolve({3}) == {4, 2}
    assert o.evolve(set()) == set()
    assert o.evolve({-1}) == set()
    assert o.evolve({2}) == {2}


def test_evolve_is_not_a_closure():
    o = O("ab")
    assert 0 not in o.evolve({0})


def test_eps_reaches_null_goldens():
    # test_lockstep.cpp:34-41
    assert O("a**").eps_reaches_null({0})
    assert not O("ab").eps_reaches_null({0})
    assert O("ab").eps_reaches_null({-1})
    assert not O("a**b").eps_reaches_null({0})
    assert not O("a**b").eps_reaches_null({2})


def test_step_char_goldens():
    # test_lockstep.cpp:43-50
    o = O("a**b")
    assert o.step_char({4, 2}, ord("a")) == {3}
    assert o.step_char({4, 2}, ord("b")) == {-1}
    assert o.step_char(set(), ord("a")) == set()
    assert o.step_char({-1}, ord("a")) == set()
    with pytest.raises(ValueError):
        o.step_char({0}, ord("a"))


def test_acceptance_goldens():
    # test_lockstep.cpp:52-58
    assert O("a**b").accepts(b"aab")
    assert not O("a**b").accepts(b"aa")
    assert O("a**").accepts(b"")
    assert O("()").accepts(b"")
    assert not O("a").accepts(b"")


def test_linear_time_family():
    # test_thompson.cpp:139-146 / acceptance criterion 6: (a*)*b vs a^1000 b
    assert O("(a*)*b").accepts(b"a" * 1000 + b"b")
    assert not O("(a*)*b").accepts(b"a" * 1000)


def test_truth_table():
    # test_regex.cpp:98-104: (a|b)*a over |w| <= 3
    want = {"a", "aa", "ba", "aaa", "aba", "baa", "bba"}
    o = O("(a|b)*a")
    import itertools

    for n in range(4):
        for t in itertools.product("ab", repeat=n):
            w = "".join(t)
            assert o.accepts(w.encode()) == (w in want)


def test_exhaustive_small_suite_golden():
    d = json.loads((G / "lockstep_small.json").read_text())
    ws = d["strings"]
    for p, bits in d["accept"].items():
        o = O(p)
        got = "".join("1" if o.accepts(w.encode()) else "0" for w in ws)
        assert got == bits, p


def test_per_step_evolved_sets_golden():
    for case in json.loads((G / "lockstep_steps.json").read_text()):
        o = O(case["pattern"])
        s = {0}
        for a, want in zip(case["input"], case["evolved"]):
            e = o.evolve(s)
            assert sorted(e) == want
            s = o.step_char(e, ord(a))
        assert o.accepts(case["input"].encode()) == case["accept"]


def test_config_samples_golden():
    import hashlib

    d = json.loads((G / "configs.json").read_text())
    for cfg, e in d.items():
        pat = rx.synth_pattern(cfg)
        assert hashlib.sha1(pat.encode()).hexdigest() == e["pattern_sha1"]
        text = rx.synth_input(cfg, e["bytes"])
        assert hashlib.sha1(text.tobytes()).hexdigest() == e["input_sha1"]
        o = O(pat)
        if "accept" in e:
            assert o.accepts(text.tobytes()) == e["accept"]
        else:
            delim, stride = (-1, 32) if cfg == "b" else (10, 0)
            cnt, res = o.match_batch(text, delim, stride)
            assert cnt == e["count"] and len(res) == e["strings"]
            assert hashlib.sha1(res.tobytes()).hexdigest() == e["results_sha1"]


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_oracle_against_reference_random():
    rng = np.random.default_rng(3)
    for p in Ref.random_regexes(150, 24, seed=11, alphabet="abc"):
        o, r = O(p), RefHeap(p.encode())
        for _ in range(8):
            w = bytes(rng.choice([97, 98, 99], size=int(rng.integers(0, 30))).astype(np.uint8))
            assert o.accepts(w) == r.accepts(w), (p, w)


def test_synth_restatement_equals_product_generator():
    """oracle/synth_oracle.c (the reference arm's inputs, no librxg) emits the
    same bytes as the product's generator for every config (prefixes for the
    big ones), and its mt19937_64 passes the standard's known answer."""
    import oracle_bind as ob
    from paper_1108_3126_b200 import rx

    assert ob.mt64_nth(5489, 10000) == 9981545732273789042   # [rand.predef]
    for c in "aAbcde":
        assert ob.synth_pattern(c) == rx.synth_pattern(c), c
    for c, n in [("a", None), ("A", None), ("b", None), ("c", 4 << 20), ("d", 4 << 20), ("e", 1 << 20)]:
        assert np.array_equal(ob.synth_input(c, n), rx.synth_input(c, n)), c
    assert np.array_equal(ob.synth_input("c", 1 << 20, seed=1003), rx.synth_input("c", 1 << 20, seed=1003))


def test_oracle_decodes_utf8_like_the_reference():
    """The C oracle matches decoded scalars (utf8.cpp:16-46), not bytes: a
    one-scalar literal pattern accepts its 2/3/4-byte encoding, a byte-wise
    reading would not; malformed strings never match (the reference throws)."""
    from oracle_bind import Oracle, Ref, RefHeap
    from paper_1108_3126_b200 import rx

    for pat, good, bad in [("é", "é", "e"), ("(λ|b)*", "λbλ", "λc"), ("😀a", "😀a", "😀")]:
        o = Oracle(rx.compile(rx.parse(pat)))
        assert o.accepts(good.encode()) and not o.accepts(bad.encode())
        if Ref.available():   # the reference on the decoded scalars agrees
            r = RefHeap(pat.encode())
            assert r.accepts(good) and not r.accepts(bad)
    o = Oracle(rx.compile(rx.parse("(a|())*")))
    assert not o.accepts(b"a\xffa") and not o.accepts(b"\xc3")
    cnt, res = o.match_batch(np.frombuffer("é\na\n\xff\n".encode("latin-1"), np.uint8), 10, 0)
    assert list(res) == [0, 1, 0]
