"""Dev tool: one chunk-parallel launch of (aaa)* over 256 MiB of a's (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

n = 256 << 20
d = torch.full((n + 64,), ord("a"), dtype=torch.uint8, device="cuda")
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
m = rx.Matcher("(aaa)*")
for _ in range(2):
    m.match_one_ex(d, acc, "chunked", nbytes=n)
torch.cuda.synchronize()
print(bool(acc.item()))
