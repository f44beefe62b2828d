"""Dev tool: the chunk-parallel engine on non-synchronising automata
((aaa)*, (aa)*) over a 256 MiB string of a's, against config (e)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

n = 256 << 20
d = torch.full((n + 64,), ord("a"), dtype=torch.uint8, device="cuda")
acc = torch.zeros(1, dtype=torch.int32, device="cuda")
e = rx.synth_input("e")
de = torch.empty(len(e) + 64, dtype=torch.uint8, device="cuda")
de[: len(e)].copy_(torch.from_numpy(e))
for pat, buf, nb in (("(aaa)*", d, n), ("(aa)*", d, n), (rx.synth_pattern("e"), de, len(e))):
    m = rx.Matcher(pat)
    for _ in range(2):
        m.match_one_ex(buf, acc, "chunked", nbytes=nb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        m.match_one_ex(buf, acc, "chunked", nbytes=nb)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{pat[:24]:24s} {nb} B: {ts[2] * 1e3:.1f} us  accept={bool(acc.item())}")
