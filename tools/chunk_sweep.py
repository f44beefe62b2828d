"""Dev tool: K2 lines kernel time on the N-GPU shard of config (c) for several
range widths (RXG_LINE_CHUNK). usage: python tools/chunk_sweep.py 8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

n_gpus = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = sys.argv[2] if len(sys.argv) > 2 else "c"
pat, text = rx.synth_pattern(cfg), rx.synth_input(cfg)
lo, hi = rx.shard(text, n_gpus, 0, delimiter=10)
nb = hi - lo
m = rx.Matcher(pat, device=0)
m.tune(text[: 1 << 20], delimiter=10)
d = torch.empty(nb + 64, dtype=torch.uint8, device="cuda")
d[:nb].copy_(torch.from_numpy(text[lo:hi]))
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
dirty = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
want = None
for chunk in (None, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096, 8192):
    rx.set_option("RXG_LINE_CHUNK", chunk)
    for _ in range(3):
        m.match_batch_device(d, cnt, delimiter=10, nbytes=nb)
    torch.cuda.synchronize()
    c = int(cnt.item())
    want = want if want is not None else c
    assert c == want, (chunk, c, want)
    ts = []
    for _ in range(10):
        dirty.zero_()
        clean.sum(dtype=torch.int64)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        m.match_batch_device(d, cnt, delimiter=10, nbytes=nb)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"N={n_gpus} shard {nb} B chunk {chunk}: {ts[5]:.1f} us ({nb / ts[5] / 1e3:.0f} GB/s)")
rx.set_option("RXG_LINE_CHUNK", None)
