"""Dev tool: device-time of the single-string engines on a config (optionally a prefix).
usage: python tools/ab_single.py CFG NBYTES ENGINE[:reps]..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx

cfg, nbytes = sys.argv[1], int(sys.argv[2])
pat = rx.synth_pattern(cfg)
text = rx.synth_input(cfg, nbytes if nbytes > 0 else None)
d = torch.from_numpy(text).cuda()
m = rx.Matcher(pat, device=0)
acc = torch.zeros(1, dtype=torch.int32, device=0)
rep = torch.zeros(1, dtype=torch.int64, device=0)
for v in sys.argv[3:]:
    if v == "tune":   # bank placement of the single-string table from a 1 MiB sample
        m.tune(text[: 1 << 20], delimiter=-1)
        continue
    eng, _, reps = v.partition(":")
    reps = int(reps or 3)
    kw = {"d_repairs": rep} if eng in ("chunked", "auto") else {}
    m.match_one_ex(d, acc, eng, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        m.match_one_ex(d, acc, eng, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{cfg} {len(text):>10d} B {eng:8s} {ms:10.3f} ms {len(text)/ms/1e6:9.2f} GB/s {len(text)/ms/1e3:9.1f} Msym/s "
          f"{ms*1e6/len(text):8.3f} ns/sym accept={int(acc.item())} repairs={int(rep.item())}", flush=True)
