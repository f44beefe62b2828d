"""The N>1 path on CPU (world_size 2, gloo), driving the same sharding code as
bench.py's strong-scaled run: every rank builds the whole job, takes its shard
with rx.shard (rxg_shard_bounds: byte-balanced, cut at string boundaries),
matches it with the host emulation of the line kernel (same table image,
tuned from the head of the job, same ownership rules as the GPU), and the
8-byte count is all-reduced — the only collective. The total must equal the
oracle on the whole job; fixed-stride jobs shard at stride multiples."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1108_3126_b200 import rx

    try:
        out = {}
        for cfg, nbytes in (("c", 1 << 20), ("d", 1 << 20)):
            pat = rx.synth_pattern(cfg)
            text = rx.synth_input(cfg, nbytes)
            lo, hi = rx.shard(text, world, rank, delimiter=10)
            m = rx.Matcher(pat, device=-1)
            m.tune(text[: 1 << 16])   # the job's head, as bench.py: identical tables on every rank
            local = m.emulate_lines_tma(text[lo:hi], 10, 64)
            cnt = torch.tensor([local], dtype=torch.int64)
            dist.all_reduce(cnt)
            out[cfg] = (int(cnt.item()), lo, hi)
        # fixed stride: shards at stride multiples
        pat = rx.synth_pattern("b")
        text = rx.synth_input("b", 32 * 1000)
        lo, hi = rx.shard(text, world, rank, delimiter=-1, stride=32)
        assert lo % 32 == 0 and hi % 32 == 0
        m = rx.Matcher(pat, device=-1)
        local, _ = m.emulate_batch(text[lo:hi], delimiter=-1, stride=32)
        cnt = torch.tensor([local], dtype=torch.int64)
        dist.all_reduce(cnt)
        out["b"] = (int(cnt.item()), lo, hi)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_strong_shards_count_allreduce():
    from oracle_bind import Oracle
    from paper_1108_3126_b200 import rx

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for cfg, nbytes, delim, stride in (("c", 1 << 20, 10, 0), ("d", 1 << 20, 10, 0), ("b", 32 * 1000, -1, 32)):
        text = rx.synth_input(cfg, nbytes)
        o = Oracle(rx.compile(rx.parse(rx.synth_pattern(cfg))))
        want, _ = o.match_batch(text, delim, stride, results=False)
        # shards tile the job, in rank order, and split no string
        assert out[0][cfg][1] == 0 and out[0][cfg][2] == out[1][cfg][1] and out[1][cfg][2] == len(text)
        if delim >= 0:
            assert text[out[0][cfg][2] - 1] == delim
        for r in range(world):
            assert out[r][cfg][0] == want, (cfg, r)


def test_shard_bounds_edge_cases():
    from paper_1108_3126_b200 import rx

    # more shards than strings, empty job, no delimiter at all, long lines
    assert rx.shard_bounds(b"ab\ncd\n", 4, 10) [-1] == 6
    b = rx.shard_bounds(b"ab\ncd\n", 4, 10)
    assert b == sorted(b) and all(x in (0, 3, 6) for x in b)
    assert rx.shard_bounds(b"", 3, 10) == [0, 0, 0, 0]
    assert rx.shard_bounds(b"abcdef", 3, 10) == [0, 6, 6, 6]
    t = np.frombuffer(b"x" * 1000 + b"\n" + b"y\n", np.uint8)
    b = rx.shard_bounds(t, 2, 10)
    assert b == [0, 1001, 1003]
    assert rx.shard_bounds(b"a" * 96, 2, -1, 32) == [0, 32, 96]
