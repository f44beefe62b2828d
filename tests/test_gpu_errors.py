"""Error behaviour of the C ABI on a GPU: bad arguments come back as status
codes with a message (the C++ facade rethrows them, as the reference's
callers expect exceptions, rxvm.cpp:243-249), never as wrong answers."""
import numpy as np
import pytest
import torch

from paper_1108_3126_b200 import _lib as L
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu


def _status(fn, *a, **k):
    with pytest.raises(rx.RxgError) as ei:
        fn(*a, **k)
    return ei.value.status


def test_batch_argument_errors():
    m = rx.Matcher("(a|b)*abb", device=0)
    d = torch.zeros(4096 + 64, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    # misaligned device buffer (the TMA/vector paths need 16-byte alignment)
    assert _status(m.match_batch_device, d[1:], cnt, nbytes=4000) == L.RXG_EINVAL
    # fixed stride that does not divide the buffer
    assert _status(m.match_batch_device, d, cnt, delimiter=-1, stride=7, nbytes=4000) == L.RXG_EINVAL
    # delimiter outside a byte
    assert _status(m.match_batch_device, d, cnt, delimiter=300, nbytes=4000) == L.RXG_EINVAL
    # the call after an error still works
    m.match_batch_device(d, cnt, nbytes=4096)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0   # 4096 zero bytes: one line, no match


def test_single_string_alignment():
    m = rx.Matcher("(a|b)*abb", device=0)
    d = torch.zeros(4096 + 64, dtype=torch.uint8, device="cuda")
    d[4000:4003] = torch.tensor(list(b"abb"), dtype=torch.uint8)
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    for eng in ("auto", "chunked", "dfa_seq", "pernode"):
        assert _status(m.match_one_ex, d[1:], acc, engine=eng, nbytes=4002) == L.RXG_EINVAL
    m.match_one_ex(d[16:], acc, nbytes=4003 - 16)   # aligned: fine, and the context is healthy
    torch.cuda.synchronize()
    assert int(acc.item()) == 0   # zeros before "abb" are outside (a|b)*


def test_utf8_check_argument_errors():
    d = torch.zeros(64, dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    assert _status(rx.utf8_check_device, d, 64, out, delimiter=200) == L.RXG_EINVAL
    assert _status(rx.utf8_check_device, d, 60, out, delimiter=-1, stride=7) == L.RXG_EINVAL


def test_bad_device_and_engine():
    assert _status(rx.Matcher, "(a|b)*abb", device=97) == L.RXG_ECUDA
    m = rx.Matcher("é*", device=0)
    # the literal rounds engine compares bytes with literals: ASCII only
    assert _status(m.lockstep_accepts, "éé".encode(), "rounds") == L.RXG_EUNSUPPORTED
    assert m.lockstep_accepts("éé".encode(), "pernode")


def test_exploding_dfa_single_string_auto_falls_back():
    """Over the memoized-step cap, the default single-string engine is the
    thread-per-node form (still exact), fixed-stride batches run on the bitset
    engine; DFA-only engines report ETOOBIG."""
    pat = "(a|b)*a" + "(a|b)" * 17
    m = rx.Matcher(pat, device=0)
    w = b"ab" * 1000 + b"a" + b"b" * 17
    assert m.lockstep_accepts(w) is True
    assert m.lockstep_accepts(w[:-1] + b"c") is False
    assert _status(m.lockstep_accepts, w, "dfa_seq") == L.RXG_ETOOBIG
    # fixed stride over the cap: the bitset engine (K2b) answers instead of RXG_ETOOBIG
    from oracle_bind import Oracle

    fs = np.frombuffer(w[: len(w) // 2 * 2], np.uint8)
    got, _ = m.match_batch(fs, -1, 2)
    want, _ = Oracle(rx.compile(rx.parse(pat))).match_batch(fs, -1, 2, results=False)
    assert got == want
