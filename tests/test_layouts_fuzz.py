"""Random regexes through every line-table layout (direct, class rows with
range-clamped columns, class rows with a class map; RXG_FORCE_CLASS and
RXG_NO_RANGE_LAYOUT force the latter two on small DFAs): the host model of
the TMA line kernel (CPU) and the kernel itself (GPU) against the oracle."""
import os

import numpy as np
import pytest

from oracle_bind import Oracle, Ref
from paper_1108_3126_b200 import rx
from test_gpu_stress import _dev_count

LAYOUT_ID = {"direct": 1, "classmap": 2, "range": 3}
LAYOUTS = {"direct": {}, "range": {"RXG_FORCE_CLASS": "1"},
           "classmap": {"RXG_FORCE_CLASS": "1", "RXG_NO_RANGE_LAYOUT": "1"}}


def _regexes(n, seed):
    if Ref.available():
        return Ref.random_regexes(n, 14, seed, "abc ")
    rng = np.random.default_rng(seed)   # fallback: small hand-made mixes
    atoms = ["a", "b", "c", " ", "()", "(a|b)", "(b|c)*", "a*", "(ab|c)"]
    return ["".join(rng.choice(atoms, size=int(rng.integers(1, 6)))) + "*" * int(rng.integers(0, 2)) for _ in range(n)]


def _lines(seed, n=3000):
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(b"abc ", np.uint8)
    out = [alpha[rng.integers(0, 4, int(rng.integers(0, 30)))].tobytes() for _ in range(n)]
    return np.frombuffer(b"\n".join(out) + b"\n", np.uint8)


class _env:
    """Sets rxg_set_option switches for the block (the library reads no environment)."""

    def __init__(self, kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            rx.set_option(k, v)

    def __exit__(self, *exc):
        for k in self.kv:
            rx.set_option(k, None)


@pytest.mark.parametrize("layout", list(LAYOUTS))
def test_host_model_all_layouts(layout):
    text = _lines(1)
    for p in _regexes(40, 3):
        want, _ = Oracle(rx.compile(rx.parse(p))).match_batch(text, 10, 0)
        with _env(LAYOUTS[layout]):
            m = rx.Matcher(p, device=-1)
            for chunk in (64, 512):
                assert m.emulate_lines_tma(text, 10, chunk) == want, (layout, p, chunk)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", list(LAYOUTS))
def test_kernel_all_layouts(layout):
    text = _lines(2, 20000)
    seen = set()
    for p in _regexes(60, 5):
        want_c, want_r = Oracle(rx.compile(rx.parse(p))).match_batch(text, 10, 0)
        with _env(LAYOUTS[layout]):
            m = rx.Matcher(p, device=0)
            c, r = m.match_batch(text, 10, results=True)
            c2, _ = m.match_batch(text, 10)
            c3 = _dev_count(m, text)
            lay = m.info()["line_tma_layout"]
        assert c == c2 == c3 == want_c and np.array_equal(r, want_r), (layout, p)
        assert lay in (0, LAYOUT_ID[layout]), (layout, p, lay)   # 0: DFA too large for any line table
        seen.add(lay)
    assert LAYOUT_ID[layout] in seen


# ── single-string (chunk) tables: packed per-byte words (<= 6 states), direct, class ──

CHUNK_LAYOUTS = {"default": {}, "nopacked": {"RXG_NO_PACKED": "1"}}


def _strings(seed, n=60):
    rng = np.random.default_rng(seed)
    alpha = np.frombuffer(b"abc ", np.uint8)
    return [alpha[rng.integers(0, 4, int(rng.integers(0, 40)))].tobytes() for _ in range(n)]


@pytest.mark.parametrize("layout", list(CHUNK_LAYOUTS))
def test_chunk_table_host_model(layout):
    seen = set()
    for p in _regexes(60, 11) + ["(a|b)*abb", "a*", "()", "(a|b|c| )*"]:
        o = Oracle(rx.compile(rx.parse(p)))
        with _env(CHUNK_LAYOUTS[layout]):
            m = rx.Matcher(p, device=-1)
            states = m.info()["dfa_states"]
            for w in _strings(hash(p) & 0xFFFF):
                acc, lay = m.emulate_chunk_tma(w)
                assert acc == o.accepts(w), (layout, p, w)
                assert (lay == 4) == (layout == "default" and 0 < states <= 6), (p, states, lay)
                seen.add(lay)
    assert (4 in seen) == (layout == "default")


@pytest.mark.gpu
@pytest.mark.parametrize("layout", list(CHUNK_LAYOUTS))
def test_chunk_kernel_layouts(layout):
    import torch

    rng = np.random.default_rng(7)
    alpha = np.frombuffer(b"abc ", np.uint8)
    for p in _regexes(25, 13) + ["(a|b)*abb", "(a|b|c| )*"]:
        o = Oracle(rx.compile(rx.parse(p)))
        with _env(CHUNK_LAYOUTS[layout]):
            m = rx.Matcher(p, device=0)
            for n in (0, 1, 100, 5000, 300_000, 5 << 20):   # up to the cooperative-launch path
                w = alpha[rng.integers(0, 4, n)]
                if n > 3 and rng.integers(0, 2):
                    w[-3:] = np.frombuffer(b"abb", np.uint8)
                want = o.accepts(w.tobytes()) if n <= 300_000 else None
                d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
                d[:n].copy_(torch.from_numpy(w))
                acc = torch.zeros(1, dtype=torch.int32, device="cuda")
                m.match_one_ex(d, acc, engine="chunked", nbytes=n)
                got = bool(acc.item())
                if want is None:   # long: the sequential DFA engine is the check
                    acc2 = torch.zeros(1, dtype=torch.int32, device="cuda")
                    m.match_one_ex(d, acc2, engine="dfa_seq", nbytes=n)
                    want = bool(acc2.item())
                assert got == want, (layout, p, n)
