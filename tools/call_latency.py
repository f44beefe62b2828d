"""Dev tool: per-call latency of the synchronous single-string host path
(rxg_match_one: H2D of the string, one launch, D2H of the answer) for the
short strings the reference's callers pass (crosscheck, run_engine, tests),
per engine, and of the instrumented call (rxg_match_one_stats)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_3126_b200 import rx  # noqa: E402

m = rx.Matcher("(a|b)*abb", device=0)
for n in (8, 64, 1024):
    w = (b"ab" * n)[:n - 3] + b"abb"
    for eng in ("auto", "dfa_seq", "pernode", "rounds"):
        for _ in range(50):
            m.lockstep_accepts(w, eng)
        k = 2000
        t0 = time.perf_counter()
        for _ in range(k):
            m.lockstep_accepts(w, eng)
        print(f"{n:5d} B {eng:8s}: {(time.perf_counter() - t0) / k * 1e6:7.1f} us per call")
    for _ in range(50):
        m.lockstep_stats(w)
    t0 = time.perf_counter()
    for _ in range(1000):
        m.lockstep_stats(w)
    print(f"{n:5d} B stats   : {(time.perf_counter() - t0) / 1000 * 1e6:7.1f} us per call")
