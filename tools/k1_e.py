"""Dev tool: K1 (the paper's thread-per-node scheme, engine=pernode) over the
full config (e) string, segmented across SMs, against the chunked engine;
ns/symbol. usage: python tools/k1_e.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "e"
pat, w = rx.synth_pattern(cfg), rx.synth_input(cfg)
m = rx.Matcher(pat, device=0)
n = len(w)
d = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
d[:n].copy_(torch.from_numpy(w))
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
for twin in ("pos", "neg"):
    if twin == "neg":
        d[n - 1] = ord("a")
    res = {}
    for eng in ("pernode", "chunked"):
        m.match_one_ex(d, acc, eng, nbytes=n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        m.match_one_ex(d, acc, eng, nbytes=n)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[eng] = (bool(acc.item()), ms)
        print(f"({cfg}) {twin} {eng}: accept={res[eng][0]} {ms:.3f} ms = {ms * 1e6 / n:.3f} ns/symbol = {n / ms / 1e6:.1f} GB/s")
    assert res["pernode"][0] == res["chunked"][0]
print("k1 ok")
