"""GPU parity of the single-string engines (K1 thread-per-node, the literal
§8 rounds protocol, the chunk-parallel walk, the sequential table walk)
against the oracle and the reference library."""
import numpy as np
import pytest
import torch

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu

ENGINES = ["dfa_seq", "chunked", "pernode", "rounds", "auto"]


def O(p):
    return Oracle(rx.compile(rx.parse(p)))


@pytest.mark.parametrize("engine", ENGINES)
def test_worked_examples(engine):
    # test_lockstep.cpp:52-58, test_parallel.cpp:84-93
    assert rx.Matcher("a**b").lockstep_accepts(b"aab", engine)
    assert not rx.Matcher("a**b").lockstep_accepts(b"aa", engine)
    assert rx.Matcher("a**").lockstep_accepts(b"", engine)
    assert rx.Matcher("()").lockstep_accepts(b"", engine)
    assert not rx.Matcher("a").lockstep_accepts(b"", engine)
    assert not rx.Matcher("a").lockstep_accepts(b"b", engine)
    assert rx.Matcher("(a*)*b").lockstep_accepts(b"a" * 1000 + b"b", engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_config_a_full(engine):
    m = rx.Matcher(rx.synth_pattern("a"))
    assert m.lockstep_accepts(rx.synth_input("a").tobytes(), engine) is True
    assert m.lockstep_accepts(rx.synth_input("A").tobytes(), engine) is False


@pytest.mark.parametrize("engine", ENGINES)
def test_random_small_against_oracle(engine):
    rng = np.random.default_rng(5)
    pats = Ref.random_regexes(40, 14, seed=9) if Ref.available() else ["(a|b)*abb", "a**b", "(ab|a)*b"]
    for p in pats:
        m = rx.Matcher(p)
        o = O(p)
        for _ in range(6):
            w = bytes(rng.choice([97, 98], size=int(rng.integers(0, 300))).astype(np.uint8))
            assert m.lockstep_accepts(w, engine) == o.accepts(w), (p, w)


@pytest.mark.parametrize("chunk", [256, 96, 288])
def test_chunked_long_strings_with_small_ranges(chunk):
    """Many ranges and repairs: parity on non-synchronizing automata too; range
    sizes that are not multiples of the 256-byte checkpoint period."""
    rng = np.random.default_rng(2)
    for p in ["(a|b)*abb", "(aa)*", "((a|b)(a|b))*", "(ab|ba)*a", "a*b*a*b*"]:
        m = rx.Matcher(p)
        o = O(p)
        for n in (0, 1, 63, 64, 65, 5000, 100_000, 1_000_003):
            w = rng.choice([97, 98], size=n).astype(np.uint8)
            if p == "(aa)*":
                w[:] = 97
            d = torch.from_numpy(w).cuda() if n else torch.zeros(1, dtype=torch.uint8, device="cuda")
            acc = torch.zeros(1, dtype=torch.int32, device="cuda")
            rep = torch.zeros(1, dtype=torch.int64, device="cuda")
            m.match_one_ex(d, acc, "chunked", nbytes=n, chunk=chunk, lookback=16, d_repairs=rep)
            torch.cuda.synchronize()
            assert bool(acc.item()) == o.accepts(w.tobytes()), (p, n)


def test_rounds_instrumentation_like_parallel_cpp():
    """claims once per node per macro step, launches <= steps * N (test_parallel.cpp:95-112)."""
    rng = np.random.default_rng(23)
    pats = Ref.random_regexes(30, 8, seed=23) if Ref.available() else ["a**b", "(a|b)*a"]
    for p in pats:
        m = rx.Matcher(p)
        h = rx.compile(rx.parse(p))
        w = rng.choice([97, 98], size=int(rng.integers(0, 6))).astype(np.uint8)
        d = torch.from_numpy(w).cuda() if len(w) else torch.zeros(1, dtype=torch.uint8, device="cuda")
        acc = torch.zeros(1, dtype=torch.int32, device="cuda")
        stats = torch.zeros(4, dtype=torch.int64, device="cuda")
        m.match_one_ex(d, acc, "rounds", nbytes=len(w), d_stats=stats)
        claims, rounds, steps, maxc = stats.tolist()
        assert bool(acc.item()) == O(p).accepts(w.tobytes())
        assert maxc <= 1
        assert rounds <= steps * h.size()
        if Ref.available():
            ok, rs = RefHeap(p.encode()).par_accepts(w.tobytes(), workers=1, seed=1)
            assert ok == bool(acc.item())
            assert claims == rs["claims"]   # each node claimed once per step it is scheduled in


def test_rounds_macro_boundaries_equal_lockstep_sets():
    """test_parallel.cpp:114-137: the next schedule (null included) equals step_char(evolve(S), a)."""
    rng = np.random.default_rng(31)
    pats = Ref.random_regexes(30, 8, seed=31) if Ref.available() else ["a**b", "(a|b)*a"]
    for p in pats:
        h = rx.compile(rx.parse(p))
        o = O(p)
        m = rx.Matcher(p)
        w = rng.choice([97, 98], size=int(rng.integers(1, 5))).astype(np.uint8)
        words = (h.size() + 1 + 31) // 32
        trace = torch.zeros(len(w) * words, dtype=torch.int32, device="cuda")
        acc = torch.zeros(1, dtype=torch.int32, device="cuda")
        m.match_one_ex(torch.from_numpy(w).cuda(), acc, "rounds", d_trace=trace)
        rows = trace.cpu().numpy().view(np.uint32).reshape(len(w), words)
        s = {0}
        for i, a in enumerate(w):
            s = o.step_char(o.evolve(s), int(a))
            got = {q for q in range(h.size()) if (rows[i][q >> 5] >> (q & 31)) & 1}
            if (rows[i][h.size() >> 5] >> (h.size() & 31)) & 1:
                got.add(-1)
            assert got == s, (p, w, i)
            if not s:
                break


def test_pernode_checkpoints_equal_host_sets():
    p = rx.synth_pattern("e")
    m = rx.Matcher(p)
    w = rx.synth_input("e", 4096)
    W = m.info()["words"]
    every = 256
    ck = torch.zeros((4096 // every) * W, dtype=torch.int32, device="cuda")
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    m.match_one_ex(torch.from_numpy(w).cuda(), acc, "pernode", checkpoint_every=every, d_checkpoints=ck)
    got = ck.cpu().numpy().view(np.uint32).reshape(-1, W)
    sets, hacc = rx.Matcher(p, device=-1).host_walk(w.tobytes())
    for k in range(len(got)):
        assert np.array_equal(got[k], sets[(k + 1) * every]), k
    assert bool(acc.item()) == hacc


@pytest.mark.parametrize("engine", ["chunked", "pernode", "dfa_seq"])
def test_config_e_prefix(engine):
    p = rx.synth_pattern("e")
    m = rx.Matcher(p)
    for n in (1 << 16, 1 << 20):
        w = rx.synth_input("e", n)
        assert m.lockstep_accepts(w.tobytes(), engine) == O(p).accepts(w.tobytes())


def test_config_e_k1_checkpoints_verified_chunk_parallel():
    """SURVEY.md §8(c) parity plan item 2: K1 (thread-per-node) emits its active
    set every 256 KiB of a 4 MiB prefix of config (e); each chunk is re-run by
    the oracle from the previous checkpoint on all host cores."""
    from oracle_bind import verify_checkpoints

    p = rx.synth_pattern("e")
    m = rx.Matcher(p)
    n, every = 4 << 20, 256 << 10
    w = rx.synth_input("e", n)
    W = m.info()["words"]
    ck = torch.zeros((n // every) * W, dtype=torch.int32, device="cuda")
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    m.match_one_ex(torch.from_numpy(w).cuda(), acc, "pernode", checkpoint_every=every, d_checkpoints=ck)
    rows = ck.cpu().numpy().view(np.uint32).reshape(-1, W)
    pos_addr, _, _ = rx.Matcher(p, device=-1).tables()
    assert verify_checkpoints(rx.compile(rx.parse(p)), pos_addr, len(pos_addr), rows, w, every) == n // every
    assert bool(acc.item()) == bool((rows[-1][len(pos_addr) >> 5] >> (len(pos_addr) & 31)) & 1)


def test_chunked_entry_exit_states_chain_segments():
    """A string cut anywhere: the exit state of the first part, used as the
    entry of the second, gives the whole string's answer (including
    non-synchronizing automata), and chaining from the start state equals
    the default run."""
    rng = np.random.default_rng(21)
    for p in ["(a|b)*abb", "(aa)*", "((a|b)(a|b))*", rx.synth_pattern("c")]:
        m = rx.Matcher(p)
        o = O(p)
        alpha = [97, 98] if "ERROR" not in p else list(b"abcdefgh ERORWANFIL")
        w = rng.choice(alpha, size=200_003).astype(np.uint8)
        if p == "(aa)*":
            w[:] = 97
        for cut in (0, 1, 4096, 100_000, 200_003):
            d1 = torch.from_numpy(w[:cut].copy()).cuda() if cut else torch.zeros(16, dtype=torch.uint8, device="cuda")
            d2 = torch.from_numpy(w[cut:].copy()).cuda() if cut < len(w) else torch.zeros(16, dtype=torch.uint8, device="cuda")
            ex = torch.zeros(2, dtype=torch.int32, device="cuda")
            acc = torch.zeros(1, dtype=torch.int32, device="cuda")
            m.match_one_ex(d1, acc, "chunked", nbytes=cut, d_exit_state=ex[0:1])
            torch.cuda.synchronize()
            e1 = int(ex[0].item()) & 0xFFFFFFFF
            m.match_one_ex(d2, acc, "chunked", nbytes=len(w) - cut, flags=1, entry_state=e1, d_exit_state=ex[1:2])
            torch.cuda.synchronize()
            assert bool(acc.item()) == o.accepts(w.tobytes()), (p, cut)


@pytest.mark.parametrize("ndev", [1, 2, 3, 5])
def test_match_one_multi_segments(ndev):
    """rxg_match_one_multi with the one GPU listed several times: segments
    run from guessed entries, wrong guesses are re-run in order; exact."""
    rng = np.random.default_rng(ndev)
    for p, n in [("(a|b)*abb", 3_000_000), ("(aa)*", 1_000_002), (rx.synth_pattern("e"), 2_000_000)]:
        if p == "(aa)*":
            w = np.full(n, 97, np.uint8)
        elif "abb" in p and len(p) < 20:
            w = rng.choice([97, 98], size=n).astype(np.uint8)
            w[-3:] = np.frombuffer(b"abb", np.uint8)
        else:
            w = rx.synth_input("e", n)
        acc, reruns = rx.match_one_multi([0] * ndev, p, w)
        want = rx.Matcher(p).lockstep_accepts(w.tobytes(), "dfa_seq")
        assert acc == want, (p, ndev)
    # (aaa)*: a 64-byte prefix leaves the counter at 64 mod 3, the true state
    # at a 16-aligned cut is (offset mod 3): wrong guesses must be re-run
    w = np.full(3_000_000, 97, np.uint8)
    acc, reruns = rx.match_one_multi([0] * ndev, "(aaa)*", w)
    assert acc is True
    if ndev > 2:
        assert reruns > 0


@pytest.mark.parametrize("layout", ["range", "class"])
def test_chunked_class_tables(layout):
    """Single strings whose minimal DFA exceeds the direct layout: the chunk
    kernel's class rows, with range-clamped columns or the class map, against
    the sequential walk and the oracle."""
    if layout == "class":
        rx.set_option("RXG_NO_RANGE_LAYOUT", 1)
    try:
        rng = np.random.default_rng(5)
        for p, alpha in [("(a|b)*a" + "(a|b)" * 6, b"ab"), (rx.synth_pattern("d"), b"abcdefghijklmnopqrstuvwxyz ")]:
            m = rx.Matcher(p)
            assert m.info()["dfa_states"] > 56
            a = np.frombuffer(alpha, np.uint8)
            for n in (1000, 300_001):
                w = a[rng.integers(0, len(a), n)].tobytes()
                want = m.lockstep_accepts(w, "dfa_seq")
                assert m.lockstep_accepts(w, "chunked") == want, (p[:20], n)
                if n == 1000:
                    assert want == O(p).accepts(w)
    finally:
        rx.set_option("RXG_NO_RANGE_LAYOUT", None)


def test_chunked_sticky_states_parallel_rounds():
    """A keyword seen once keeps (d)'s automaton accepting: on one long string
    of words nearly every range's guessed entry is wrong. Large inputs repair
    in parallel rounds (cooperative launch), small ones in order; both exact,
    including strings where the keyword appears only near the start or end."""
    rng = np.random.default_rng(13)
    p = rx.synth_pattern("d")
    m = rx.Matcher(p)
    words = rx.synth_input("d", 24 << 20).copy()
    words[words == 10] = 32
    for n in (1 << 20, 24 << 20):
        w = words[:n]
        want = m.lockstep_accepts(w.tobytes(), "dfa_seq")
        assert m.lockstep_accepts(w.tobytes(), "chunked") == want, n
    # a string whose only keyword match region is near the end, and one with a
    # byte outside [a-z ] at the end (the sink leaves): the answers flip
    w = words.copy()
    w[-1] = ord("#")
    assert m.lockstep_accepts(w.tobytes(), "chunked") == m.lockstep_accepts(w.tobytes(), "dfa_seq")
    acc_rounds = rx.Matcher("(a|b)*a(a|b)*")   # sticky after the first 'a'
    w = np.full(24 << 20, ord("b"), np.uint8)
    w[int(rng.integers(0, 100))] = ord("a")
    assert acc_rounds.lockstep_accepts(w.tobytes(), "chunked") is True
    w[:] = ord("b")
    assert acc_rounds.lockstep_accepts(w.tobytes(), "chunked") is False


@pytest.mark.parametrize("pat,alpha,n", [("(a|b)*abb", b"ab", 3 << 20), ("(aa)*", b"a", 2 << 20), ("(aaa)*", b"a", (3 << 20) + 7),
                                         ("(a|b)*a(a|b)(a|b)(a|b)", b"ab", 5 << 20), ("(ab|a)*(b|())", b"ab", 2 << 20)])
def test_pernode_segments_across_sms_equal_one_warp(pat, alpha, n):
    """K1 over a long string as segments across SMs (guessed entry sets,
    exact repair rounds) gives the one-warp walk's answer, including
    non-synchronizing automata ((aa)*, (aaa)*) whose guesses are wrong."""
    import torch

    rng = np.random.default_rng(n)
    a = np.frombuffer(alpha, np.uint8)
    w = a[rng.integers(0, len(a), n)].copy()
    m = rx.Matcher(pat)
    d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    d[:n].copy_(torch.from_numpy(w))
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    for tail in (b"", b"abb", b"a", b"aa"):
        if tail:
            d[n - len(tail):n].copy_(torch.frombuffer(bytearray(tail), dtype=torch.uint8))
        m.match_one_ex(d, acc, "pernode", nbytes=n)
        torch.cuda.synchronize()
        seg = bool(acc.item())
        m.match_one_ex(d, acc, "pernode", nbytes=n, flags=2)   # RXG_ONE_SINGLE_WARP
        torch.cuda.synchronize()
        one = bool(acc.item())
        m.match_one_ex(d, acc, "dfa_seq", nbytes=n)
        torch.cuda.synchronize()
        assert seg == one == bool(acc.item()), (pat, tail)


@pytest.mark.parametrize("n", [(64 << 20) + 1, (64 << 20) + 2, 64 << 20, (16 << 20) + 5])
def test_chunked_nonsynchronizing_by_transfer_functions(n):
    """(aaa)* / (aa)* over long strings of a's: every entry guess of the
    chunk-parallel engine is wrong; the packed layout composes the ranges'
    transfer functions in order instead of repairing range by range. Known
    answers (n mod 3, n mod 2) and a broken string."""
    import torch

    d = torch.full((n + 64,), ord("a"), dtype=torch.uint8, device="cuda")
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    for pat, want in (("(aaa)*", n % 3 == 0), ("(aa)*", n % 2 == 0), ("(aaaa|aaaaaa)*", n % 2 == 0 and n != 2)):
        m = rx.Matcher(pat)
        m.match_one_ex(d, acc, "chunked", nbytes=n)
        torch.cuda.synchronize()
        assert bool(acc.item()) == want, (pat, n)
    d[n // 3] = ord("b")
    m = rx.Matcher("(aaa)*")
    m.match_one_ex(d, acc, "chunked", nbytes=n)
    torch.cuda.synchronize()
    assert not bool(acc.item())


@pytest.mark.parametrize("force", ["1", "0"])
def test_chunked_transfer_function_mode(force):
    """Packed tables: the transfer-function mode (every range walked from all
    of its S states on the TMA ring, functions composed in range order) chosen
    for automata with a permuting byte ((aaa)*), forced on here for patterns
    of 1-6 states and forced off for (aaa)* (guess, then the fallback pass).
    Small (last-CTA) and large (cooperative) launches, chained entry/exit
    states; against the sequential walk and the oracle."""
    rng = np.random.default_rng(31)
    rx.set_option("RXG_CHUNK_FN", force)
    try:
        for p in ["(aaa)*", "(aa)*", "(a|b)*abb", "((a|b)(a|b))*", "(ab|ba)*a", "a*b*a*b*", "a*", "(a|b)*(aa|bb)"]:
            m = rx.Matcher(p)
            o = O(p)
            for n in (0, 1, 100, 4097, 300_001, (5 << 20) + 3, (40 << 20) + 1):
                w = (np.full(n, 97, np.uint8) if p in ("(aaa)*", "(aa)*", "a*")
                     else rng.choice([97, 98], size=n).astype(np.uint8))
                if n and p in ("(aaa)*", "(aa)*") and rng.integers(0, 2):
                    w[int(rng.integers(0, n))] = 98
                d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
                if n:
                    d[:n].copy_(torch.from_numpy(w))
                acc = torch.zeros(1, dtype=torch.int32, device="cuda")
                ref = torch.zeros(1, dtype=torch.int32, device="cuda")
                m.match_one_ex(d, acc, "chunked", nbytes=n)
                m.match_one_ex(d, ref, "dfa_seq", nbytes=n)
                torch.cuda.synchronize()
                assert bool(acc.item()) == bool(ref.item()), (p, n, force)
                if n <= 300_001:
                    assert bool(acc.item()) == o.accepts(w.tobytes()), (p, n, force)
            # chained pieces: the exit state of one call is the entry of the next
            w = np.full((3 << 20) + 2, 97, np.uint8) if p in ("(aaa)*", "(aa)*") else rng.choice([97, 98], size=(3 << 20) + 2).astype(np.uint8)
            d = torch.from_numpy(w).cuda()
            acc = torch.zeros(1, dtype=torch.int32, device="cuda")
            ex = torch.zeros(1, dtype=torch.int32, device="cuda")
            cut = len(w) // 3
            m.match_one_ex(d[:cut], acc, "chunked", nbytes=cut, d_exit_state=ex)
            torch.cuda.synchronize()
            m.match_one_ex(d[cut:], acc, "chunked", nbytes=len(w) - cut, flags=1, entry_state=int(ex.item()))
            torch.cuda.synchronize()
            assert bool(acc.item()) == o.accepts(w.tobytes()), (p, "chained", force)
    finally:
        rx.set_option("RXG_CHUNK_FN", None)
