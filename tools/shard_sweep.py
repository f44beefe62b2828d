"""Per-GPU kernel span of a strong-scaled batch job on ONE GPU: the shard rank
0 of N would match (rx.shard, the product's rxg_shard_bounds) for N = 1, 2,
4, 8, timed like bench.py (L2 flushed below 256 MiB). This is the kernel part
of the N-GPU step; the 8-byte NCCL all-reduce comes on top and is not
measurable with one GPU. usage: python tools/shard_sweep.py c d b"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1108_3126_b200 import rx  # noqa: E402

CFG = {"b": (-1, 32), "c": (10, 0), "d": (10, 0)}
dirty = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for cfg in sys.argv[1:] or ["c"]:
    delim, stride = CFG[cfg]
    pat, text = rx.synth_pattern(cfg), rx.synth_input(cfg)
    m = rx.Matcher(pat, device=0)
    if delim >= 0:
        m.tune(text[: 1 << 20], delimiter=delim)
    rows = {}
    for n in (1, 2, 4, 8):
        lo, hi = rx.shard(text, n, 0, delimiter=delim, stride=stride)
        nb = hi - lo
        d = torch.empty(nb + 64, dtype=torch.uint8, device="cuda")
        d[:nb].copy_(torch.from_numpy(text[lo:hi]))
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        for _ in range(3):
            m.match_batch_device(d, cnt, delimiter=delim, stride=stride, nbytes=nb)
        ts = []
        for _ in range(10):
            if nb < 256 << 20:
                dirty.zero_()
                clean.sum(dtype=torch.int64)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            m.match_batch_device(d, cnt, delimiter=delim, stride=stride, nbytes=nb)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        us = ts[len(ts) // 2]
        rows[n] = {"shard_bytes": nb, "kernel_us": us, "per_gpu_gbs": nb / us / 1e3,
                   "job_gbs_if_all_gpus_alike": len(text) / us / 1e3}
        print(f"({cfg}) N={n}: shard {nb} B, kernel {us:.1f} us, {nb / us / 1e3:.0f} GB/s per GPU, "
              f"job {len(text) / us / 1e3:.0f} GB/s (kernel span, no all-reduce)")
        del d
    out[cfg] = rows
print(json.dumps(out))
