"""K2b, the bitset lockstep engine on K2's TMA data path
(csrc/kernels_bits_tma.cu), against the C oracle and the reference library:
line batches and fixed-stride batches, counts and per-string results,
patterns whose memoized step is over the cap ((a|b)*a(a|b)^17: 2^18 DFA
states), many residual groups (Cox), shared-memory rows (8 and 16 words),
and the rxvm-style edge buffers. Also: the instrumentation of the literal
protocol kernel equals the reference's LockstepStats / ParStats."""
import numpy as np
import pytest
import torch

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu


def _o(p):
    return Oracle(rx.compile(rx.parse(p)))


def _dev(m, text, delim, stride=0, results=False):
    n = len(text)
    d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    if n:
        d[:n].copy_(torch.from_numpy(np.ascontiguousarray(text)))
    cnt = torch.full((1,), 777, dtype=torch.int64, device="cuda")
    nstr = rx.count_strings(text, delim, stride) if (delim >= 0 or stride) else 0
    res = torch.zeros(max(nstr, 1) + 1, dtype=torch.uint8, device="cuda") if results else None
    m.match_batch_device(d, cnt, res, delimiter=delim, stride=stride, nbytes=n, engine="bitset")
    torch.cuda.synchronize()
    return int(cnt.item()), (res[:nstr].cpu().numpy() if results else None)


def _lines(rng, alpha, n, maxlen, longs=0):
    a = np.frombuffer(alpha, np.uint8)
    out = [a[rng.integers(0, len(a), int(rng.integers(0, maxlen)))].tobytes() for _ in range(n)]
    for i in rng.integers(0, n, longs):
        out[i] = a[rng.integers(0, len(a), 20_000)].tobytes()
    return np.frombuffer(b"\n".join(out) + b"\n", np.uint8)


PATTERNS = ["(a|b)*abb", "(a|b)*a(a|b)" + "(a|b)" * 16, "a*", "()", "(a|())*b", "((a|b)(a|b))*",
            "(ab|ba|a)*(bb|())"]


@pytest.mark.parametrize("pat", PATTERNS)
def test_lines_random_against_oracle(pat):
    rng = np.random.default_rng(abs(hash(pat)) % 1000)
    text = _lines(rng, b"ab", 40_000, 60, longs=3)
    o = _o(pat)
    want, wres = o.match_batch(text, 10, 0)
    m = rx.Matcher(pat, device=0)
    c, r = _dev(m, text, 10, results=True)
    assert c == want and np.array_equal(r, wres), pat
    c2, _ = _dev(m, text, 10)
    assert c2 == want


@pytest.mark.parametrize("stride", [32, 20, 7, 64, 33])
@pytest.mark.parametrize("pat", ["(a|b)*a(a|b)" + "(a|b)" * 16, rx.synth_pattern("b"), "(a|b)*abb"])
def test_fixed_stride_against_oracle(stride, pat):
    rng = np.random.default_rng(stride)
    n = 20_011
    text = np.frombuffer(b"ab", np.uint8)[rng.integers(0, 2, n * stride)].copy()
    if "(a|())" in pat:   # Cox: mostly all-a strings, some broken
        text[:] = ord("a")
        text[rng.integers(0, n * stride, n // 5)] = ord("b")
    want, wres = _o(pat).match_batch(text, -1, stride)
    m = rx.Matcher(pat, device=0)
    c, r = _dev(m, text, -1, stride, results=True)
    assert c == want and np.array_equal(r, wres), (pat[:20], stride)


def test_over_cap_pattern_runs_auto_in_both_modes():
    """(a|b)*a(a|b)^17 has 2^18 DFA states: the AUTO batch path takes K2b
    for lines and for a fixed stride (no longer RXG_ETOOBIG)."""
    pat = "(a|b)*a" + "(a|b)" * 17
    m = rx.Matcher(pat, device=0)
    assert m.info()["dfa_states"] == 0
    rng = np.random.default_rng(3)
    text = _lines(rng, b"ab", 5000, 40)
    want, wres = _o(pat).match_batch(text, 10, 0)
    c, r = m.match_batch(text, delimiter=10, results=True)
    assert c == want and np.array_equal(r, wres)
    fs = np.frombuffer(b"ab", np.uint8)[rng.integers(0, 2, 24 * 3001)]
    want, wres = _o(pat).match_batch(fs, -1, 24)
    c, r = m.match_batch(fs, delimiter=-1, stride=24, results=True)
    assert c == want and np.array_equal(r, wres)
    if Ref.available():
        rc, rr = RefHeap(pat.encode()).match_batch(fs, -1, 24)
        assert rc == c and np.array_equal(rr, r)


@pytest.mark.parametrize("cfg,nbytes", [("c", 8 << 20), ("d", 4 << 20)])
def test_configs_forced_bitset(cfg, nbytes):
    """(c): one word; (d): 511 positions + A = 16 words (shared-memory rows)."""
    pat = rx.synth_pattern(cfg)
    text = rx.synth_input(cfg, nbytes)
    want, wres = _o(pat).match_batch(text, 10, 0)
    m = rx.Matcher(pat, device=0)
    c, r = _dev(m, text, 10, results=True)
    assert c == want and np.array_equal(r, wres)
    assert _dev(m, text, 10)[0] == want


def test_eight_word_sets():
    """A pattern with 200-odd positions (8 words)."""
    kws = ["".join(chr(97 + (i * 7 + j * 3) % 26) for j in range(3 + i % 5)) for i in range(50)]
    pat = "((" + "|".join(kws) + ")| )*"
    m = rx.Matcher(pat, device=0)
    assert 128 < m.info()["positions"] < 256
    rng = np.random.default_rng(9)
    words = [kws[i] for i in rng.integers(0, 50, 60_000)]
    text = " ".join(words).encode()
    text = np.frombuffer(text.replace(b" ", b"\n", 20_000), np.uint8)
    text = text.copy()
    text[rng.integers(0, len(text), 300)] = ord("z")
    want, wres = _o(pat).match_batch(text, 10, 0)
    c, r = _dev(m, text, 10, results=True)
    assert c == want and np.array_equal(r, wres)


@pytest.mark.parametrize("buf", [b"", b"\n", b"\n\n\n", b"ab", b"abb\n", b"\nabb", b"a\nb\n\nabb", b"x" * 100])
def test_edge_buffers(buf):
    for pat in ["a*", "abb", "()", "(a|b)*abb", "a|()"]:
        m = rx.Matcher(pat, device=0)
        text = np.frombuffer(buf, np.uint8) if buf else np.zeros(0, np.uint8)
        want, wres = _o(pat).match_batch(text, 10, 0)
        c, r = _dev(m, text, 10, results=True)
        assert c == want and list(r) == list(wres), (pat, buf)


def test_lockstep_and_parallel_stats_equal_the_reference():
    """LockstepStats.enqueued and ParStats (claims, launches, macro steps,
    max claims per node per step) of one GPU run of the literal protocol equal
    the reference's own counters (lockstep.hpp:16-18, parallel.hpp:52-58)."""
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(17)
    pats = Ref.random_regexes(120, 10, 5, "ab") + ["a**b", "(a|b)*abb", "()"]
    checked = 0
    for p in pats:
        m = rx.Matcher(p, device=0)
        r = RefHeap(p.encode())
        for _ in range(4):
            w = bytes(rng.choice([97, 98], int(rng.integers(0, 12))).astype(np.uint8))
            acc, st = m.lockstep_stats(w)
            racc, renq = r.accepts_stats(w.decode())
            assert acc == racc and st["enqueued"] == renq, (p, w, st, renq)
            pacc, ps = r.par_accepts(w.decode(), workers=1, seed=0)
            assert pacc == acc
            assert ps["claims"] == st["claims"] and ps["launches"] == st["launches"], (p, w, ps, st)
            assert ps["max_claims"] == st["max_claims_per_node_step"] <= 1
            checked += 1
    assert checked == len(pats) * 4
