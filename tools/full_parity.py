"""Full-size parity of every config on the GPU box.

  (b), (c), (d): per-string results of the GPU batch path (rxg_match_batch,
                 results mode) against the C oracle over ALL strings, all host cores.
  (a):           full string, both twins, every single-string engine vs the oracle.
  (e):           256 MiB string: K1 (thread-per-node) with checkpoints every
                 4 MiB, every chunk re-run by the oracle from the previous
                 checkpoint on all cores; the chunked engine's answer compared too.

usage: python tools/full_parity.py [a b c d e]   (writes a log line per config)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle_bind import Oracle, verify_checkpoints  # noqa: E402
from paper_1108_3126_b200 import rx  # noqa: E402


def log(*a):
    print(*a, flush=True)


def batch(cfg, delim, stride):
    pat = rx.synth_pattern(cfg)
    text = rx.synth_input(cfg)
    m = rx.Matcher(pat, device=0)
    t0 = time.time()
    cnt, res = m.match_batch(text, delimiter=delim, stride=stride, results=True)
    tg = time.time() - t0
    d = torch.from_numpy(text).cuda()
    dc = torch.zeros(1, dtype=torch.int64, device="cuda")
    m.match_batch_device(d, dc, delimiter=delim, stride=stride)
    torch.cuda.synchronize()
    t0 = time.time()
    ocnt, ores = Oracle(rx.compile(rx.parse(pat))).match_batch(text, delim, stride)
    to = time.time() - t0
    ok = cnt == ocnt == int(dc.item()) and np.array_equal(res, ores)
    log(f"({cfg}) strings={len(ores)} gpu_count={cnt} count_only_kernel={int(dc.item())} oracle_count={ocnt} "
        f"per_string_equal={np.array_equal(res, ores)} -> {'PASS' if ok else 'FAIL'} "
        f"(gpu host-path {tg:.2f}s, oracle {to:.1f}s on {os.cpu_count()} threads)")
    return ok


def single_a():
    pat = rx.synth_pattern("a")
    m = rx.Matcher(pat, device=0)
    o = Oracle(rx.compile(rx.parse(pat)))
    ok = True
    for cfg in ("a", "A"):
        w = rx.synth_input(cfg).tobytes()
        want = o.accepts(w)
        got = {e: m.lockstep_accepts(w, e) for e in ("chunked", "dfa_seq", "pernode", "rounds")}
        ok &= all(v == want for v in got.values())
        log(f"({cfg}) 1 MiB oracle={want} engines={got}")
    log(f"(a) -> {'PASS' if ok else 'FAIL'}")
    return ok


def single_e():
    pat = rx.synth_pattern("e")
    m = rx.Matcher(pat, device=0)
    w = rx.synth_input("e")
    n = len(w)
    every = 4 << 20
    W = m.info()["words"]
    d = torch.from_numpy(w).cuda()
    ck = torch.zeros((n // every) * W, dtype=torch.int32, device="cuda")
    acc = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.time()
    m.match_one_ex(d, acc, "pernode", checkpoint_every=every, d_checkpoints=ck)
    torch.cuda.synchronize()
    tk = time.time() - t0
    rows = ck.cpu().numpy().view(np.uint32).reshape(-1, W)
    pos, _, _ = rx.Matcher(pat, device=-1).tables()
    t0 = time.time()
    nchunks = verify_checkpoints(rx.compile(rx.parse(pat)), pos, len(pos), rows, w, every)
    tv = time.time() - t0
    k1 = bool(acc.item())
    final = bool((rows[-1][len(pos) >> 5] >> (len(pos) & 31)) & 1)
    m.match_one_ex(d, acc, "chunked")
    torch.cuda.synchronize()
    ch = bool(acc.item())
    ok = k1 == final == ch
    log(f"(e) 256 MiB: K1 {tk:.1f}s accept={k1}; {nchunks} chunks of 4 MiB verified by the oracle in {tv:.0f}s; "
        f"chunked engine accept={ch} -> {'PASS' if ok else 'FAIL'}")
    # negative twin (last byte 'a'): the chunk-parallel engine against the
    # sequential walk of the same memoized table over the full string
    d[-1] = ord("a")
    res = {}
    for e in ("chunked", "dfa_seq"):
        m.match_one_ex(d, acc, e)
        torch.cuda.synchronize()
        res[e] = bool(acc.item())
    ok2 = res["chunked"] == res["dfa_seq"] is False
    log(f"(E) 256 MiB negative twin: {res} -> {'PASS' if ok2 else 'FAIL'}")
    return ok and ok2


def main():
    which = sys.argv[1:] or list("abcde")
    ok = True
    for c in which:
        if c == "a":
            ok &= single_a()
        elif c == "b":
            ok &= batch("b", -1, 32)
        elif c in "cd":
            ok &= batch(c, 10, 0)
        elif c == "e":
            ok &= single_e()
    log("ALL PASS" if ok else "SOME FAILED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
