"""Dev tool: the chunk-parallel engine on config (d)'s pattern over one long
string of words (config (d)'s input with newlines turned into spaces)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1108_3126_b200 import rx

w = rx.synth_input("d", 256 << 20).copy()
w[w == 10] = 32
m = rx.Matcher(rx.synth_pattern("d"), device=0)
m.tune(w[: 1 << 20], delimiter=-1)
d = torch.from_numpy(w).cuda()
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
rep = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    m.match_one_ex(d, acc, "chunked", d_repairs=rep)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10):
    m.match_one_ex(d, acc, "chunked", d_repairs=rep)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"(d) words as one string: {len(w) / ms / 1e6:.1f} GB/s accept={int(acc.item())} repairs={int(rep.item())}")
