"""Dev tool: device time of per-line results on the TMA line kernel (one
pass: range-local result bits + counts, scan, scatter) against the count-only
launch, on the full config buffers. usage: python tools/res_lines.py c d"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

for cfg in sys.argv[1:] or ["c"]:
    pat, text = rx.synth_pattern(cfg), rx.synth_input(cfg)
    m = rx.Matcher(pat, device=0)
    m.tune(text[: 1 << 20])
    n = len(text)
    d = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    d[:n].copy_(torch.from_numpy(text))
    nl = rx.count_strings(text, 10)
    res = torch.zeros(nl + 1, dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = {}
    for mode in ("count", "results"):
        r = res if mode == "results" else None
        for _ in range(3):
            m.match_batch_device(d, cnt, r, delimiter=10, nbytes=n)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            m.match_batch_device(d, cnt, r, delimiter=10, nbytes=n)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        out[mode] = (int(cnt.item()), ts[len(ts) // 2])
    assert out["count"][0] == out["results"][0] == int(res[:nl].sum().item())
    print(f"({cfg}) {n} B {nl} lines: count-only {out['count'][1]:.1f} us, per-line results {out['results'][1]:.1f} us "
          f"({n / out['results'][1] / 1e3:.0f} GB/s); matches {out['count'][0]}")
