"""Dev tool: one very long line in line mode (the warp-cooperative finish)."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch
from paper_1108_3126_b200 import rx
m = rx.Matcher(rx.synth_pattern("c"), device=0)
for n in (1 << 20, 16 << 20, 100 << 20):
    t = np.frombuffer(b"abcdefgh ERROR", np.uint8)[np.random.default_rng(1).integers(0, 14, n)]
    d = torch.from_numpy(t).cuda(); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, cnt); torch.cuda.synchronize()
    t0 = time.perf_counter(); m.match_batch_device(d, cnt); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print("one line of", n >> 20, "MiB:", round(dt * 1e3, 2), "ms", round(n / dt / 1e9, 3), "GB/s", int(cnt.item()), flush=True)
