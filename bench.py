#!/usr/bin/env python3
"""Benchmark harness: input GB/s matched, bit-exact lockstep regex matching.

Metric (BASELINE.json): input GB/s matched at 1/2/4/8 B200 and % of the
binding roofline, beside the reference's CPU lockstep matcher.

Default workload: config (c) of SURVEY.md §8(d) — the 64-node
alternation/star log regex over 10M synthetic '\\n'-terminated lines
(~1.03 GB) — the configuration BASELINE.json names "sharded at 1/2/4/8
GPUs". A "step" is one pass of the batch matcher (K2) over the whole
resident buffer. Other configs: --config a|b|c|d|e.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c] [--impl b200|reference]

Under torchrun (N > 1) every rank matches its own shard of the same shape
(weak scaling; rank r uses generator seed canonical+r) and the only
collective is one all-reduce of the 8-byte match count per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (delimiter, stride, description)
    "a": (-2, 0, "(a|b)*abb over one 1 MiB {a,b} string"),
    "b": (-1, 32, "Cox (a?)^32 a^32, 1M strings a^32 at stride 32"),
    "c": (10, 0, "64-node alternation/star log regex over 10M lines (~100 B)"),
    "d": (10, 0, "1024-node keyword union over 1 GiB of ~1 KiB lines"),
    "e": (-2, 0, "4096-node keyword-star regex over one 256 MiB string"),
}
W_WORDS = {"a": 1, "b": 3, "c": 1, "d": 16, "e": 65}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every ~0.25 ms, plus one sample at
    the start) while the enqueued timed steps run."""

    REASONS = {  # nvmlClocksEventReasons bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
    }

    def __init__(self, device: int):
        self.device = device
        self.period = float(os.environ.get("RXG_CLOCK_PERIOD_S", "0.00025"))
        self.off = os.environ.get("RXG_NO_CLOCKS") is not None   # A/B of the sampler's own cost
        self.rows = []
        self.stop = threading.Event()
        self.h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _sample(self):
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            try:
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except AttributeError:
                bits = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.rows.append((mhz, bits))
        except Exception:
            pass

    def _loop(self):
        while not self.stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.h is not None and not self.off:
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.h is not None and not self.off:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted({n for _, b in self.rows for n, m in self.REASONS.items() if b & m})
        return {"sm_mhz": float(np.median([m for m, _ in self.rows])), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.rows)}


def make_input(cfg: str, seed: int, nbytes: int | None = None):
    from paper_1108_3126_b200 import rx

    return rx.synth_pattern(cfg), rx.synth_input(cfg, nbytes, seed=seed)


def count_units(text: np.ndarray, delim: int, stride: int) -> int:
    if delim == -2:
        return 1
    if delim < 0:
        return len(text) // stride
    n = int(np.count_nonzero(text == delim))
    return n + (1 if len(text) and text[-1] != delim else 0)


# ── CPU legs (reference library compiled from /root/reference sources) ─────

def cpu_reference(cfg: str, pattern: str, text: np.ndarray, target_s: float = 12.0, threads: int | None = None):
    """Time rx::lockstep_accepts (oracle/_ref) on a bounded sample of the
    workload with all host threads. Returns (GB/s, sample description, cores, kind)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bind import REF_SO, Oracle, RefHeap
    from paper_1108_3126_b200 import rx

    threads = threads or os.cpu_count() or 1
    delim, stride, _ = CONFIGS[cfg]
    kind = "reference" if REF_SO.exists() else "port"
    if kind == "reference":
        h = RefHeap(pattern.encode())
    else:
        h = Oracle(rx.compile(rx.parse(pattern)))

    def run(sample: np.ndarray, nthreads: int):
        if delim == -2:   # one string: one core
            t0 = time.perf_counter()
            ok = h.accepts(sample.tobytes())
            return time.perf_counter() - t0, int(ok)
        if kind == "reference":
            # decode_utf8 happens in ref_prepare; time only lockstep_accepts
            import ctypes as C
            a = np.ascontiguousarray(sample)
            prep = h.l.ref_prepare(a.ctypes.data, a.nbytes, delim, stride)
            t0 = time.perf_counter()
            cnt = h.l.ref_run(h.p, prep, None, nthreads)
            dt = time.perf_counter() - t0
            h.l.ref_prepared_free(prep)
            return dt, int(cnt)
        t0 = time.perf_counter()
        cnt, _ = h.match_batch(sample, delim, stride, results=False, threads=nthreads)
        return time.perf_counter() - t0, cnt

    def cut(nb: int) -> np.ndarray:
        nb = min(nb, len(text))
        if delim >= 0:
            j = int(np.flatnonzero(text[:nb] == delim)[-1]) + 1 if np.any(text[:nb] == delim) else nb
            return text[:j]
        if delim == -1:
            return text[: nb - nb % stride]
        return text[:nb]

    cores = 1 if delim == -2 else threads
    probe = cut(1 << 16)
    dt, _ = run(probe, cores)
    rate = len(probe) / max(dt, 1e-6)
    nb = int(min(len(text), max(len(probe), rate * target_s)))
    sample = cut(nb)
    dt, cnt = run(sample, cores)
    desc = (f"first {len(sample)} B of config ({cfg}) ({count_units(sample, delim, stride)} strings), "
            f"rx::lockstep_accepts on {cores} thread(s), decode excluded")
    if delim == -2:
        desc = f"first {len(sample)} B prefix of the config ({cfg}) string, 1 core (single string), extrapolation is linear"
    return len(sample) / dt / 1e9, desc, cores, kind, dt


# ── reference arm ──────────────────────────────────────────────────────────

def run_reference_arm(args):
    """The reference's own CPU lockstep matcher (oracle/_ref = proj/src compiled
    from source) on a bounded sample of the same workload, all host threads.
    The sample is sized once (~args.ref_step_s per step) and decoded once;
    each step times rx::lockstep_accepts over all of its strings."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bind import REF_SO, Oracle, RefHeap
    from paper_1108_3126_b200 import rx

    cfg = args.config
    delim, stride, _ = CONFIGS[cfg]
    pattern, text = make_input(cfg, 0)
    threads = os.cpu_count() or 1
    # size the sample with one calibration run of the shared helper
    _, desc, cores, kind, _ = cpu_reference(cfg, pattern, text, target_s=args.ref_step_s, threads=threads)
    nbytes = int(desc.split()[1])
    sample = text[:nbytes]
    if kind == "reference":
        h = RefHeap(pattern.encode())
        if delim == -2:
            w = sample.tobytes()
            run = lambda: h.accepts(w)  # noqa: E731
        else:
            a = np.ascontiguousarray(sample)
            prep = h.l.ref_prepare(a.ctypes.data, a.nbytes, delim, stride)
            run = lambda: h.l.ref_run(h.p, prep, None, cores)  # noqa: E731
    else:
        o = Oracle(rx.compile(rx.parse(pattern)))
        run = (lambda: o.accepts(sample.tobytes())) if delim == -2 else \
            (lambda: o.match_batch(sample, delim, stride, results=False, threads=cores))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    v = len(sample) / float(np.median(times)) / 1e9
    line = {
        "metric": "input GB/s matched", "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(times)) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config ({cfg}): {CONFIGS[cfg][2]}", "input_bytes": int(len(text)),
                   "sample_bytes": int(len(sample))},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": kind, "sample": desc},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ── B200 arm ───────────────────────────────────────────────────────────────

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--engine", default="auto")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--cpu-target-s", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_1108_3126_b200 import rx
    from paper_1108_3126_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    torch.cuda.set_device(dev)
    cfg = args.config
    delim, stride, desc = CONFIGS[cfg]
    single = delim == -2

    pattern, text_np = make_input(cfg, seed=0 if rank == 0 else 1000 + rank)
    nbytes = len(text_np)
    units = count_units(text_np, delim, stride)
    m = rx.Matcher(pattern, device=dev)
    # planner: table bank placement from a 1 MiB sample (lines, or the single-string table)
    if delim >= 0 or single:
        m.tune(text_np[: 1 << 20], delimiter=delim if delim >= 0 else -1)
    info = m.info()

    host = torch.from_numpy(text_np).pin_memory()
    d_text = torch.empty(nbytes + 64, dtype=torch.uint8, device=dev)
    d_text[:nbytes].copy_(host, non_blocking=False)
    d_count = torch.zeros(1, dtype=torch.int64, device=dev)
    d_acc = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    l2_flush = None
    if nbytes < 256 << 20:
        l2_flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        l2_clean = torch.ones(256 << 20, dtype=torch.uint8, device=dev)

    def flush_l2():
        # write a buffer larger than L2, then read another one so the lines the
        # timed kernel finds in L2 are clean (no write-back during the step)
        l2_flush.zero_()
        l2_clean.sum(dtype=torch.int64)

    def step():
        if single:
            m.match_one_device(d_text[:nbytes], d_acc, engine=args.engine, stream=stream)
        else:
            m.match_batch_device(d_text, d_count, delimiter=delim, stride=stride, stream=stream, nbytes=nbytes)

    clk = ClockSampler(dev)   # NVML initialised before the warm-up, not inside the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    launches_per_step = _lib.lib().rxg_last_launch_count()

    # parity of the timed configuration against the resident result
    result = int(d_acc.item()) if single else int(d_count.item())

    # Every timed step is enqueued first (L2 flush + events + step, no host
    # sync in between), so no host-side stall (NVML sampling, launch latency)
    # can open a gap inside a timed interval; the clock sampler runs while the
    # queue drains. (Sampling during the enqueue measured +7 us/step on (e).)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # A device-side spin (outside the timed interval) holds the stream while the
    # host enqueues the K steps: the first call's host latency (measured 10-65 us
    # in a fresh process) then never shows up as an idle gap between ev0 and the
    # first kernel. Host costs per call are what e2e measures.
    torch.cuda._sleep(int(2.0e6 * (0.3 + 0.02 * args.steps)))   # ~2 GHz: 0.3 ms + 20 us per step
    if l2_flush is None:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))]
        dbg = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if os.environ.get("RXG_BENCH_STEPS") else None
        ev[0][0].record(stream)
        for i in range(args.steps):
            step()
            if world > 1:
                dist.all_reduce(d_count)   # the match-count gather (8 bytes)
            if dbg:
                dbg[i].record(stream)
        ev[0][1].record(stream)
    else:
        ev = []
        for _ in range(args.steps):
            flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            if world > 1:
                dist.all_reduce(d_count)
            e1.record(stream)
            ev.append((e0, e1))
    with clk:
        torch.cuda.synchronize(dev)
    if l2_flush is None:
        total_ms = ev[0][0].elapsed_time(ev[0][1])
        if dbg:
            log("per-step us:", [round(a.elapsed_time(b) * 1e3, 1) for a, b in zip([ev[0][0]] + dbg[:-1], dbg)])
        times = [total_ms / args.steps] * args.steps
    else:
        times = [e0.elapsed_time(e1) for e0, e1 in ev]
        total_ms = float(sum(times))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    total_bytes = nbytes * world
    value = total_bytes / (ms_per_step / 1e3) / 1e9

    # kernel-only roofline figure (1 rank's dominant kernel, events around the launch)
    hbm, peak_src = peaks()
    kern_ms = float(np.median(times)) if l2_flush is not None else ms_per_step
    achieved = nbytes / (kern_ms / 1e3) / 1e9

    # end-to-end through the C ABI with host buffers (H2D inside the timed region)
    e2e = None
    if not args.no_e2e:
        host_np = host.numpy()
        if single:
            m.lockstep_accepts(host_np)   # warm
            t0 = time.perf_counter()
            for _ in range(max(1, args.steps // 2)):
                m.lockstep_accepts(host_np)
            e2e_s = (time.perf_counter() - t0) / max(1, args.steps // 2)
            d2h = 4
        else:
            m.match_batch(host_np, delimiter=delim, stride=stride)
            t0 = time.perf_counter()
            for _ in range(max(1, args.steps // 2)):
                cnt, _ = m.match_batch(host_np, delimiter=delim, stride=stride)
            e2e_s = (time.perf_counter() - t0) / max(1, args.steps // 2)
            d2h = 8
        e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": total_bytes / float(e2e_t.item()) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": d2h}

    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(cfg)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            gbs, sdesc, cores, kind, _ = cpu_reference(cfg, pattern, text_np, target_s=args.cpu_target_s)
            cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sdesc}
        except Exception as e:  # the baseline is reported, never the product path
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": None, "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "input GB/s matched",
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic",
            "config": {
                "workload": f"config ({cfg}): {desc}",
                "pattern_nodes": info["nodes"], "positions": info["positions"], "words": info["words"],
                "dfa_states": info["dfa_states"], "line_col_bytes": m.info()["line_col_bytes"], "chunk_lookback": m.info()["chunk_lookback"], "input_bytes_per_gpu": nbytes, "strings_per_gpu": units,
                "matches_rank0": result,
                "l2": "inputs larger than L2 (126 MB)" if l2_flush is None else "L2 flushed between timed steps (512 MiB write, then 256 MiB read)",
                "parallelism": f"dp{world} (string shards, count all-reduce)" if world > 1 else "dp1",
                "engine": args.engine if single else "k2_lines" if delim >= 0 else "k2_fixed",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": nbytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
