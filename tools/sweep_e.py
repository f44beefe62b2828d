"""Dev tool: config (e) device time vs input size (fixed cost vs per-byte rate) for the chunk kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx


def t_us(step, n=30):
    for _ in range(5): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): step()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


m = rx.Matcher(rx.synth_pattern("e"), device=0)
full = rx.synth_input("e", 1 << 30)
m.tune(full[: 4 << 20], -1)
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
d = torch.from_numpy(full).cuda()
rep = torch.zeros(1, dtype=torch.int64, device="cuda")
for n in (16 << 20, 64 << 20, 256 << 20, 1 << 30):
    us = t_us(lambda: m.match_one_ex(d, acc, engine="chunked", nbytes=n))
    m.match_one_ex(d, acc, engine="chunked", nbytes=n, d_repairs=rep); torch.cuda.synchronize()
    print(os.environ.get("TAG", ""), n >> 20, "MB %.1f us  %.0f GB/s  repairs %d" % (us, n / us / 1e3, int(rep.item())), flush=True)
