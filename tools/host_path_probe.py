"""Host-buffer path cost on the full config (c) file: which part of the
`rxvm match` call (results, UTF-8 check, mapped vs malloc'd source) costs
what. Diagnostic for tools/rxgmatch_e2e.sh; not a bench."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1108_3126_b200 import rx

text = rx.synth_input("c")
text.tofile("/tmp/c.txt")
pat = rx.synth_pattern("c")
m = rx.Matcher(pat)
mapped = np.memmap("/tmp/c.txt", dtype=np.uint8, mode="r")
_ = int(mapped[::4096].sum())   # fault the mapping in


def t(name, f, reps=3):
    f()
    best = 1e9
    for _ in range(reps):
        s = time.perf_counter()
        f()
        best = min(best, time.perf_counter() - s)
    print(f"{name:36s} {best * 1e3:8.1f} ms  {text.size / best / 1e9:6.2f} GB/s", flush=True)


for src_name, src in [("malloc", text), ("mmap", mapped)]:
    t(f"{src_name} count", lambda: m.match_batch(src))
    t(f"{src_name} count+results", lambda: m.match_batch(src, results=True))
    t(f"{src_name} count+utf8", lambda: m.match_batch_utf8(src))
    t(f"{src_name} count+results+utf8", lambda: m.match_batch_utf8(src, results=True))
