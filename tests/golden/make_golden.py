#!/usr/bin/env python3
"""Regenerates tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref/librxref.so, built from /root/reference/proj/src by
oracle/Makefile). Run here, where /root/reference exists; the fixtures are
committed so the GPU box (no /root/reference) can check against them.

  python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import itertools
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from oracle_bind import Ref, RefHeap, build_oracle  # noqa: E402


def strings(max_len: int, alphabet: str = "ab") -> list[str]:
    out = [""]
    for n in range(1, max_len + 1):
        out += ["".join(t) for t in itertools.product(alphabet, repeat=n)]
    return out


def main():
    if not Ref.available():
        build_oracle(with_ref=True)

    # ── front end: heap dumps, canonical prints, parse errors ──
    pats = ["a**b", "()", "a|b", "(ab)|(ac)", "a|bc*", "abc", "a|b|c", "\\*", "\\\\", "\\a", "(a|b)*abb",
            "((a|b|c|d|e|f|g|h| )*(ERROR|WARN|FAIL)(a|b|c|d|e|f|g|h| )*)*", "()*", "(a*)*b", "a(bc)", "a|(b|c)",
            "(a|b)*a", "\\(*(\\\\|\\|\\))", "α*", "a|()"]
    front = {"dump": {}, "print": {}, "errors": {}}
    for p in pats:
        b = p.encode()
        front["dump"][p] = Ref.dump(b)
        front["print"][p] = Ref.print_regex(b)
    for p in ["(((", "(a", "a)", "*a", "a|", "|a", "a||b", "ab\\", "", "(()", "a(*)", ")", "a**|", "((a)|b))"]:
        try:
            Ref.parse_compile(p.encode())
            front["errors"][p] = None
        except ValueError as e:
            front["errors"][p] = [e.args[0], e.args[1]]
    (HERE / "frontend.json").write_text(json.dumps(front, indent=1, ensure_ascii=False))

    # ── lockstep acceptance: every regex <= 5 nodes x every string <= 4 over {a,b} ──
    regs = Ref.enumerate_regexes(5, "ab")
    ws = strings(4)
    table = {}
    for p in regs:
        h = RefHeap(p.encode())
        table[p] = "".join("1" if h.accepts(w) else "0" for w in ws)
    (HERE / "lockstep_small.json").write_text(json.dumps({"strings": ws, "accept": table}, indent=0))

    # ── per-step evolved sets (evolve(S_i) per symbol) on random cases ──
    rnd = Ref.random_regexes(60, 10, seed=31)
    steps = []
    import random

    rng = random.Random(7)
    for p in rnd:
        h = RefHeap(p.encode())
        w = "".join(rng.choice("ab") for _ in range(rng.randint(0, 6)))
        s = {0}
        sets = []
        for a in w:
            e = h.evolve(s)
            sets.append(sorted(e))
            s = h.step_char(e, ord(a))
            if not s:
                break
        steps.append({"pattern": p, "input": w, "evolved": sets, "accept": h.accepts(w),
                      "trace": h.trace(w)})
    (HERE / "lockstep_steps.json").write_text(json.dumps(steps, indent=0))

    # ── config samples: counts + result digests from the reference itself ──
    from paper_1108_3126_b200 import rx

    cfgs = {}
    for cfg, nbytes, delim, stride in [("a", 1 << 20, -2, 0), ("A", 1 << 20, -2, 0), ("b", 32 * 4096, -1, 32),
                                       ("c", 2 << 20, 10, 0), ("d", 1 << 20, 10, 0), ("e", 1 << 16, -2, 0)]:
        pat = rx.synth_pattern(cfg)
        text = rx.synth_input(cfg, nbytes)
        h = RefHeap(pat.encode())
        entry = {"pattern_sha1": hashlib.sha1(pat.encode()).hexdigest(), "bytes": int(len(text)),
                 "input_sha1": hashlib.sha1(text.tobytes()).hexdigest()}
        if delim == -2:
            entry["accept"] = h.accepts(text.tobytes())
        else:
            cnt, res = h.match_batch(text, delim, stride)
            entry["count"] = cnt
            entry["strings"] = int(len(res))
            entry["results_sha1"] = hashlib.sha1(res.tobytes()).hexdigest()
        cfgs[cfg] = entry
    (HERE / "configs.json").write_text(json.dumps(cfgs, indent=1))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
