"""Dev tool: host (CPU) time per async call vs device time per step, per config."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_1108_3126_b200 import rx

acc = torch.zeros(1, dtype=torch.int32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for cfg in ("a", "b", "e"):
    m = rx.Matcher(rx.synth_pattern(cfg), device=0)
    t = rx.synth_input(cfg)
    if cfg in "ae":
        m.tune(t[: 1 << 20], -1)
    d = torch.from_numpy(t).cuda()

    def step():
        if cfg == "b":
            m.match_batch_device(d, cnt, delimiter=-1, stride=32)
        else:
            m.match_one_device(d, acc)
    for _ in range(10): step()
    torch.cuda.synchronize()
    hs = []
    for _ in range(20):   # one call after an idle GPU: host time of the call alone
        torch.cuda.synchronize()
        t0 = time.perf_counter(); step(); hs.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(200): step()
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(cfg, "host us/call (idle GPU) median %.1f min %.1f" % (sorted(hs)[10], min(hs)), "loop host us/call %.1f" % ((t1 - t0) / 200 * 1e6),
          "gpu us/step %.1f" % (e0.elapsed_time(e1) / 200 * 1e3), flush=True)
