"""Dev tool: device-time A/B of the line kernels on a synthetic config.
usage: python tools/ab_lines.py CFG VARIANT... where VARIANT is tune|notune|res|res_tune|bitset[:chunk]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx

cfg = sys.argv[1]
pat = rx.synth_pattern(cfg)
text = rx.synth_input(cfg)
d = torch.empty(len(text) + 64, dtype=torch.uint8, device=0)
d[: len(text)].copy_(torch.from_numpy(text))
cnt = torch.zeros(1, dtype=torch.int64, device=0)
for v in sys.argv[2:]:
    name, _, ch = v.partition(":")
    if ch:
        os.environ["RXG_LINE_CHUNK"] = ch
    m = rx.Matcher(pat, device=0)
    if name == "tune":
        m.tune(text[: 1 << 20])
    eng = "bitset" if name == "bitset" else "auto"
    res = None
    if name.startswith("res"):   # per-line results (TMA results path)
        res = torch.zeros(rx.count_strings(text, 10, 0) + 1, dtype=torch.uint8, device=0)
        if name == "res_tune":
            m.tune(text[: 1 << 20])
    for _ in range(3):
        m.match_batch_device(d, cnt, res, nbytes=len(text), engine=eng)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        m.match_batch_device(d, cnt, res, nbytes=len(text), engine=eng)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{v:16s} {ms*1e3:8.1f} us  {len(text)/ms/1e6:8.1f} GB/s  count={int(cnt.item())}", flush=True)
    m.close()
