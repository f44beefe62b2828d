"""Multi-GPU batch path through the C ABI.

On one GPU: the NCCL communicator path with a single rank (rxg_comm +
rxg_match_batch_allreduce: kernel, then ncclAllReduce on the same stream),
and the persistent multi-device handle with the device listed once and
several times (worker threads, shard placement of per-string results, host
sum of the counts). With two or more GPUs (skipped otherwise): the same
handle over distinct devices (ncclCommInitAll, all-reduced count) and two
torchrun ranks, each matching its shard of one job."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle_bind import Oracle
from paper_1108_3126_b200 import rx

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _oracle(pattern):
    return Oracle(rx.compile(rx.parse(pattern)))


CASES = [("c", 8 << 20, 10, 0), ("d", 4 << 20, 10, 0), ("b", 32 * 100_003, -1, 32)]


@pytest.mark.parametrize("cfg,nbytes,delim,stride", CASES)
def test_single_rank_communicator_allreduce(cfg, nbytes, delim, stride):
    pattern = rx.synth_pattern(cfg)
    text = rx.synth_input(cfg, nbytes)
    if cfg == "b":   # negatives mixed in: a^31 b and a^32 with one byte changed
        text = text.copy()
        text[32 * 7 + 31] = ord("b")
        text[32 * 5000 + 3] = ord("c")
    comm = rx.Comm(rx.Comm.unique_id(), 1, 0, 0)
    m = rx.Matcher(pattern, device=0)
    d_text = torch.empty(len(text) + 64, dtype=torch.uint8, device="cuda")
    d_text[: len(text)].copy_(torch.from_numpy(text))
    d_count = torch.full((1,), 12345, dtype=torch.int64, device="cuda")
    for _ in range(3):   # the count is overwritten every call, never accumulated
        rx.match_batch_allreduce(m, comm, d_text, d_count, delimiter=delim, stride=stride, nbytes=len(text))
    torch.cuda.synchronize()
    want, _ = _oracle(pattern).match_batch(text, delim, stride, results=False)
    assert int(d_count.item()) == want
    comm.close()


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("cfg,nbytes,delim,stride", CASES)
def test_multi_handle_shards_on_listed_devices(devices, cfg, nbytes, delim, stride):
    pattern = rx.synth_pattern(cfg)
    text = rx.synth_input(cfg, nbytes)
    mm = rx.MultiMatcher(devices, pattern)
    assert mm.info() == {"devices": len(devices), "nccl": False}
    count, res = mm.match_batch(text, delimiter=delim, stride=stride, results=True)
    ocount, ores = _oracle(pattern).match_batch(text, delim, stride)
    assert count == ocount and np.array_equal(res, ores)
    # persistent: a second job on the same handle (tables, threads reused)
    t2 = text[: len(text) // 2]
    if delim >= 0:
        t2 = t2[: int(np.flatnonzero(t2 == delim)[-1]) + 1]
    else:
        t2 = t2[: len(t2) - len(t2) % stride]
    c2, _ = mm.match_batch(t2, delimiter=delim, stride=stride)
    assert c2 == _oracle(pattern).match_batch(t2, delim, stride, results=False)[0]
    mm.close()


def test_multi_handle_more_shards_than_lines():
    mm = rx.MultiMatcher([0, 0, 0, 0], "(a|b)*abb")
    for text in [b"", b"abb", b"abb\n", b"x\nabb\n", b"ab\nabb"]:
        c, r = mm.match_batch(text, delimiter=10, results=True)
        oc, orr = _oracle("(a|b)*abb").match_batch(np.frombuffer(text, np.uint8), 10, 0)
        assert c == oc and list(r) == list(orr), text


def test_one_shot_multi_matches_oracle():
    pattern = rx.synth_pattern("c")
    text = rx.synth_input("c", 4 << 20)
    c, r = rx.match_batch_multi([0, 0], pattern, text, delimiter=10, results=True)
    oc, orr = _oracle(pattern).match_batch(text, 10, 0)
    assert c == oc and np.array_equal(r, orr)


two_gpus = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")


@two_gpus
@pytest.mark.parametrize("cfg,nbytes,delim,stride", CASES)
def test_multi_handle_nccl_over_distinct_gpus(cfg, nbytes, delim, stride):
    n = min(torch.cuda.device_count(), 8)
    pattern = rx.synth_pattern(cfg)
    text = rx.synth_input(cfg, nbytes)
    mm = rx.MultiMatcher(list(range(n)), pattern)
    assert mm.info() == {"devices": n, "nccl": True}
    count, res = mm.match_batch(text, delimiter=delim, stride=stride, results=True)
    ocount, ores = _oracle(pattern).match_batch(text, delim, stride)
    assert count == ocount and np.array_equal(res, ores)


@two_gpus
def test_torchrun_ranks_allreduce_the_job_count():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(ROOT / "tests" / "rank_worker.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "rank_worker ok" in p.stdout
