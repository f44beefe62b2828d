"""GPU parity of the single-string engines against the oracle / reference."""
import numpy as np
import pytest

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu

ENGINES = ["dfa_seq", "auto"]


@pytest.mark.parametrize("engine", ENGINES)
def test_worked_examples(engine):
    # test_lockstep.cpp:52-58
    assert rx.Matcher("a**b").lockstep_accepts(b"aab", engine)
    assert not rx.Matcher("a**b").lockstep_accepts(b"aa", engine)
    assert rx.Matcher("a**").lockstep_accepts(b"", engine)
    assert rx.Matcher("()").lockstep_accepts(b"", engine)
    assert not rx.Matcher("a").lockstep_accepts(b"", engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_config_a_full(engine):
    pattern = rx.synth_pattern("a")
    m = rx.Matcher(pattern)
    assert m.lockstep_accepts(rx.synth_input("a").tobytes(), engine) is True
    assert m.lockstep_accepts(rx.synth_input("A").tobytes(), engine) is False


@pytest.mark.parametrize("engine", ENGINES)
def test_random_small(engine):
    rng = np.random.default_rng(5)
    pats = Ref.random_regexes(40, 12, seed=9) if Ref.available() else ["(a|b)*abb", "a**b"]
    for p in pats:
        m = rx.Matcher(p)
        o = Oracle(rx.compile(rx.parse(p)))
        for _ in range(10):
            w = bytes(rng.choice([97, 98], size=int(rng.integers(0, 40))).astype(np.uint8))
            assert m.lockstep_accepts(w, engine) == o.accepts(w), (p, w)
