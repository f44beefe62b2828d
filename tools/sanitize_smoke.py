"""Dev tool: every kernel once on small inputs, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_smoke.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1108_3126_b200 import rx

text_c = rx.synth_input("c", 1 << 20)
text_d = rx.synth_input("d", 1 << 20)
for cfg, text in (("c", text_c), ("d", text_d)):
    m = rx.Matcher(rx.synth_pattern(cfg), device=0)
    m.tune(text[: 1 << 18])
    c1, _ = m.match_batch(text, 10)                      # k_lines_tma (count)
    c2, r = m.match_batch(text, 10, results=True)        # k_lines_tma RES + delimiter counts + scan
    d = torch.from_numpy(text.copy()).cuda()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, cnt, engine="bitset")        # k_lines_bitset
    torch.cuda.synchronize()
    assert c1 == c2 == int(r.sum()) == int(cnt.item()), cfg
# one 300 KB line: the range that owns it hands it to its whole warp (kCoopTail)
mc = rx.Matcher(rx.synth_pattern("c"), device=0)
long_text = np.concatenate([text_c[:4096], np.full(300_000, ord("a"), np.uint8), text_c[4096:8192]])
long_text[4096 + 150_000] = 10
cl1, _ = mc.match_batch(long_text, 10)
cl2, rl = mc.match_batch(long_text, 10, results=True)
assert cl1 == cl2 == int(rl.sum())
m = rx.Matcher(rx.synth_pattern("c"), device=0)
with rx.option("RXG_NO_LT", 1):
    c3, _ = m.match_batch(text_c, 10, results=True)      # k_lines (generic) + k_count_delims
assert c3 == c1
tb = rx.synth_input("b", 1000 * 32)
mb = rx.Matcher(rx.synth_pattern("b"), device=0)
cb, rb = mb.match_batch(tb, -1, 32, results=True)        # k_fixed_tma
assert cb == 1000 and rb.all()
cb2, _ = mb.match_batch(np.frombuffer(bytes(tb[: 48 * 100]), np.uint8), -1, 48)   # k_fixed_abs
for cfg in ("a", "e"):
    ms = rx.Matcher(rx.synth_pattern(cfg), device=0)
    w = rx.synth_input(cfg, 1 << 18).tobytes()
    for eng in ("chunked", "dfa_seq", "pernode"):
        ms.lockstep_accepts(w[: 1 << 14] if eng == "pernode" else w, eng)
ma = rx.Matcher(rx.synth_pattern("a"), device=0)
ma.lockstep_accepts(b"abababb", "rounds")                # k_rounds
rx.utf8_check(("aé中😀\n" * 1000).encode(), 10)           # k_utf8_check
rx.match_many(["(a|b)*abb", "a*"], b"ab\nabb\n\n", 10, device=0) if hasattr(rx, "match_many") else None
print("sanitize smoke done")
