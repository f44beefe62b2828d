import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1108_3126_b200 import rx
for cfg in ("a", "b"):
    m = rx.Matcher(rx.synth_pattern(cfg), device=0)
    t = rx.synth_input(cfg)
    d = torch.from_numpy(t).cuda()
    acc = torch.zeros(1, dtype=torch.int32, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    def step():
        if cfg == "a": m.match_one_device(d, acc)
        else: m.match_batch_device(d, cnt, delimiter=-1, stride=32)
    for _ in range(10): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(200): step()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(cfg, "host us/call", (t1 - t0) / 200 * 1e6, "gpu us/step", e0.elapsed_time(e1) / 200 * 1e3)
