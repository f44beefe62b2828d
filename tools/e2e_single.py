"""Dev tool: host-buffer (e2e) timing of single-string matching."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx
cfg = sys.argv[1]
text = rx.synth_input(cfg)
host = torch.from_numpy(text).pin_memory().numpy()
m = rx.Matcher(rx.synth_pattern(cfg), device=0)
for eng in sys.argv[2:] or ["auto"]:
    m.lockstep_accepts(host, eng)
    t0 = time.perf_counter()
    for _ in range(5):
        r = m.lockstep_accepts(host, eng)
    dt = (time.perf_counter() - t0) / 5
    print(cfg, eng, f"{dt*1e3:.3f} ms", f"{len(text)/dt/1e9:.2f} GB/s", r)
