"""Full-size parity of the batch configs in the driver's GPU suite
(SURVEY.md §8(c) parity plan item 1).

  (c) all 10,000,000 lines of the 1.02 GB job: per-line results of the host
      path and the count of the count-only kernel on the resident buffer,
      against the C oracle on every line (all host cores); the first >= 64 MB
      of lines also against the reference library itself (oracle/_ref).
  (b) all 1,000,000 strings at stride 32 with negatives mixed in (one byte in
      every seventh string replaced), per string against the oracle and the
      first 50,000 against the reference library.
"""
import numpy as np
import pytest
import torch

from oracle_bind import Oracle, Ref, RefHeap
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu


def test_config_c_all_lines():
    pattern = rx.synth_pattern("c")
    text = rx.synth_input("c")
    assert len(text) == 1_020_819_674
    m = rx.Matcher(pattern, device=0)
    m.tune(text[: 1 << 20])
    count, res = m.match_batch(text, delimiter=10, results=True)
    assert len(res) == 10_000_000
    d = torch.empty(len(text) + 64, dtype=torch.uint8, device="cuda")
    d[: len(text)].copy_(torch.from_numpy(text))
    dc = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, dc, delimiter=10, nbytes=len(text))
    torch.cuda.synchronize()
    ocount, ores = Oracle(rx.compile(rx.parse(pattern))).match_batch(text, 10, 0)
    assert count == ocount == int(dc.item()) == 2_499_760
    assert np.array_equal(res, ores)
    if Ref.available():   # the reference itself on a >= 64 MB prefix of whole lines
        cut = int(np.flatnonzero(text[: 64 << 20] == 10)[-1]) + 1
        rc, rr = RefHeap(pattern.encode()).match_batch(text[:cut], 10, 0)
        assert rc == int(res[: len(rr)].sum()) and np.array_equal(res[: len(rr)], rr)


def test_config_b_all_strings_with_negatives():
    pattern = rx.synth_pattern("b")
    text = rx.synth_input("b").copy()
    rng = np.random.default_rng(7)
    idx = np.arange(0, 1_000_000, 7)
    pos = rng.integers(0, 32, len(idx))
    text[idx * 32 + pos] = rng.choice(np.frombuffer(b"bcA\n\x00", np.uint8), len(idx))
    m = rx.Matcher(pattern, device=0)
    count, res = m.match_batch(text, delimiter=-1, stride=32, results=True)
    d = torch.from_numpy(text).cuda()
    dc = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, dc, delimiter=-1, stride=32)
    torch.cuda.synchronize()
    ocount, ores = Oracle(rx.compile(rx.parse(pattern))).match_batch(text, -1, 32)
    assert count == ocount == int(dc.item()) == 1_000_000 - len(idx)
    assert np.array_equal(res, ores)
    if Ref.available():
        rc, rr = RefHeap(pattern.encode()).match_batch(text[: 32 * 50_000], -1, 32)
        assert np.array_equal(res[:50_000], rr)
