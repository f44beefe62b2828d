"""Dev tool: device time per call vs input size (hot, back to back) for the
single-string and fixed-stride paths, to expose the fixed per-call cost."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_1108_3126_b200 import rx

def t_us(step, n=200):
    for _ in range(10): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): step()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3

ma = rx.Matcher(rx.synth_pattern("a"), device=0)
mb = rx.Matcher(rx.synth_pattern("b"), device=0)
mc = rx.Matcher(rx.synth_pattern("c"), device=0)
acc = torch.zeros(1, dtype=torch.int32, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
for n in (4096, 65536, 1 << 20, 4 << 20, 16 << 20):
    da = torch.from_numpy(rx.synth_input("a", n)).cuda()
    db = torch.from_numpy(rx.synth_input("b", n // 32 * 32)).cuda()
    dc = torch.from_numpy(rx.synth_input("c", n)).cuda()
    print(n, "single %.1f" % t_us(lambda: ma.match_one_device(da, acc)),
          "fixed %.1f" % t_us(lambda: mb.match_batch_device(db, cnt, delimiter=-1, stride=32)),
          "lines %.1f us" % t_us(lambda: mc.match_batch_device(dc, cnt)), flush=True)
