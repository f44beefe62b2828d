"""The N>1 path on CPU (world_size 2, gloo): shard a batch at string
boundaries, match each shard with the host emulation of the line kernel
(same table image and ownership rules as the GPU), all-reduce the 8-byte
count — the only collective — and compare with the oracle on the whole
buffer. Also checks the weak-scaling layout bench.py uses (per-rank seeds)."""
import os
import socket

import numpy as np
import pytest
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
        # strong split of one buffer
        pat = rx.synth_pattern("c")
        text = rx.synth_input("c", 1 << 20)
        b = rx.shard_bounds(text, world, delimiter=10)
        shard = text[b[rank]:b[rank + 1]]
        m = rx.Matcher(pat, device=-1)
        m.tune(shard[: 1 << 16])
        local = m.emulate_lines_tma(shard, 10, 64)
        cnt = torch.tensor([local], dtype=torch.int64)
        dist.all_reduce(cnt)
        # weak scaling: every rank its own shard of the config's shape
        own = rx.synth_input("c", 1 << 18, seed=0 if rank == 0 else 1000 + rank)
        wcnt = torch.tensor([m.emulate_lines_tma(own, 10, 64)], dtype=torch.int64)
        dist.all_reduce(wcnt)
        q.put((rank, int(cnt.item()), int(wcnt.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_count_allreduce():
    from oracle_bind import Oracle
    from paper_1108_3126_b200 import rx

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pat = rx.synth_pattern("c")
    o = Oracle(rx.compile(rx.parse(pat)))
    want, _ = o.match_batch(rx.synth_input("c", 1 << 20), 10, 0, results=False)
    wweak = sum(o.match_batch(rx.synth_input("c", 1 << 18, seed=0 if r == 0 else 1000 + r), 10, 0, results=False)[0]
                for r in range(world))
    for rank, c, wc in out:
        assert c == want
        assert wc == wweak
