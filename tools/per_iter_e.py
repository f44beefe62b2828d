import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1108_3126_b200 import rx
m = rx.Matcher(rx.synth_pattern("e"), device=0)
t = rx.synth_input("e")
m.tune(t[: 1 << 20], -1)
d = torch.empty(len(t) + 64, dtype=torch.uint8, device="cuda"); d[: len(t)].copy_(torch.from_numpy(t))
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for rep in range(3):
    for _ in range(3): m.match_one_device(d[: len(t)], acc, stream=st)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(13)]
    ev[0].record(st)
    for i in range(12):
        m.match_one_device(d[: len(t)], acc, stream=st)
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i + 1]) * 1e3, 1) for i in range(12)])
