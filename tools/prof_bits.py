"""Dev tool: one forced-bitset (K2b) launch per config on a resident buffer,
for ncu captures. usage: python tools/prof_bits.py c d"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

for cfg in sys.argv[1:] or ["c"]:
    pat, text = rx.synth_pattern(cfg), rx.synth_input(cfg)
    m = rx.Matcher(pat, device=0)
    d = torch.empty(len(text) + 64, dtype=torch.uint8, device="cuda")
    d[: len(text)].copy_(torch.from_numpy(text))
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        m.match_batch_device(d, cnt, delimiter=10, nbytes=len(text), engine="bitset")
    torch.cuda.synchronize()
    print(cfg, int(cnt.item()))
