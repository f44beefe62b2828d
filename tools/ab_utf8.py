"""Throughput of the device UTF-8 check (rxg_utf8_check) on config (c)'s
1 GB line buffer (ASCII fast path) and on a multi-byte UTF-8 buffer."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1108_3126_b200 import rx


def timeit(d, n, delim, reps=20):
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        rx.utf8_check_device(d, n, out, delim)
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rx.utf8_check_device(d, n, out, delim)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return n / float(np.median(ts)) / 1e9, int(out.item())


text = rx.synth_input("c")
d = torch.from_numpy(text).cuda()
gbs, bad = timeit(d, len(text), 10)
rng = np.random.default_rng(1)
u = ("".join(rng.choice(list("abcdé中😀 ")) for _ in range(1 << 16)) + "\n").encode() * 4096
du = torch.from_numpy(np.frombuffer(u, np.uint8).copy()).cuda()
gbu, badu = timeit(du, len(u), 10)
print(json.dumps({"ascii_GBps": round(gbs, 1), "ascii_bytes": len(text), "ascii_first_bad": bad,
                  "utf8_GBps": round(gbu, 1), "utf8_bytes": len(u), "utf8_first_bad": badu}))
