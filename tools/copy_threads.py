"""Dev tool: pageable host-buffer throughput of config (c) (count only and
with per-line results) against the number of staging copy threads
(RXG_COPY_THREADS). usage: python tools/copy_threads.py 4 8 16"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_3126_b200 import rx  # noqa: E402

text = rx.synth_input("c")
pat = rx.synth_pattern("c")
print("host cores", os.cpu_count(), flush=True)
for n in sys.argv[1:] or ["8"]:
    rx.set_option("RXG_COPY_THREADS", n)
    m = rx.Matcher(pat)   # a new handle: a new copy pool
    for results in (False, True):
        m.match_batch(text, results=results)
        best = 1e9
        for _ in range(4):
            s = time.perf_counter()
            m.match_batch(text, results=results)
            best = min(best, time.perf_counter() - s)
        print(f"threads {n:>3s} results {results!s:5s} {best * 1e3:7.1f} ms {len(text) / best / 1e9:6.1f} GB/s", flush=True)
    m.close()
