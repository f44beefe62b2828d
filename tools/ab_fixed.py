"""Dev tool: device time of the fixed-stride batch kernels on config (b), with
the input hot in L2 and after an L2 flush. usage: python tools/ab_fixed.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx

pat = rx.synth_pattern("b")
text = rx.synth_input("b")
d = torch.empty(len(text) + 64, dtype=torch.uint8, device=0)
d[: len(text)].copy_(torch.from_numpy(text))
cnt = torch.zeros(1, dtype=torch.int64, device=0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=0)
clean = torch.ones(256 << 20, dtype=torch.uint8, device=0)
for variant in ("tma", "ldg"):
    if variant == "ldg":
        rx.set_option("RXG_NO_FIXED_TMA", 1)
    m = rx.Matcher(pat, device=0)
    for _ in range(3):
        m.match_batch_device(d, cnt, delimiter=-1, stride=32, nbytes=len(text))
    torch.cuda.synchronize()
    for mode in ("hot", "cold"):
        ts = []
        for _ in range(20):
            if mode == "cold":
                flush.zero_()
                clean.sum(dtype=torch.int64)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            m.match_batch_device(d, cnt, delimiter=-1, stride=32, nbytes=len(text))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{variant:4s} {mode:5s} median {ts[len(ts)//2]:7.2f} us  min {ts[0]:7.2f} us  count={int(cnt.item())}", flush=True)
    rx.set_option("RXG_NO_FIXED_TMA", None)
