"""One rank of a torchrun job (tests/test_gpu_multi.py): the strong-scaled
batch path of bench.py — the same job on every rank, rx.shard for this
rank's piece, the product's rxg_match_batch_allreduce over a rxg_comm whose
id is broadcast with torch.distributed — checked against the oracle."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle_bind import Oracle  # noqa: E402
from paper_1108_3126_b200 import rx  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [rx.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = rx.Comm(uid[0], world, rank, local)
    for cfg, nbytes, delim, stride in [("c", 8 << 20, 10, 0), ("b", 32 * 100_003, -1, 32)]:
        pattern, text = rx.synth_pattern(cfg), rx.synth_input(cfg, nbytes)
        lo, hi = rx.shard(text, world, rank, delimiter=delim, stride=stride)
        m = rx.Matcher(pattern, device=local)
        d = torch.empty(hi - lo + 64, dtype=torch.uint8, device="cuda")
        d[: hi - lo].copy_(torch.from_numpy(text[lo:hi]))
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        rx.match_batch_allreduce(m, comm, d, cnt, delimiter=delim, stride=stride, nbytes=hi - lo)
        torch.cuda.synchronize()
        want, _ = Oracle(rx.compile(rx.parse(pattern))).match_batch(text, delim, stride, results=False)
        assert int(cnt.item()) == want, (cfg, rank, int(cnt.item()), want)
    comm.close()
    dist.destroy_process_group()
    if rank == 0:
        print("rank_worker ok")


if __name__ == "__main__":
    main()
