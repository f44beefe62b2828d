#!/usr/bin/env python3
"""Benchmark harness: input GB/s matched, bit-exact lockstep regex matching.

Metric (BASELINE.json): input GB/s matched at 1/2/4/8 B200 and % of the
binding roofline, beside the reference's CPU lockstep matcher.

Headline workload: config (c) of SURVEY.md §8(d) — the 64-node
alternation/star log regex over 10M synthetic '\\n'-terminated lines
(~1.02 GB), the configuration BASELINE.json names "sharded at 1/2/4/8 GPUs".
A "step" is one pass of the batch matcher (K2) over the whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c] [--impl b200|reference]

Multi-GPU (torchrun, one process per GPU) is STRONG scaling for the batch
configs (b, c, d): every rank builds the same job, cuts it with the product's
rxg_shard_bounds (byte-balanced at string boundaries), matches only its shard,
and the product's rxg_match_batch_allreduce sums the 8-byte count over NCCL —
the only inter-GPU traffic. `value` = whole-job bytes / (max over ranks of the
step time including that all-reduce); the kernel-only span is reported next
to it. Single-string configs (a, e) run as replicas (one string has a
sequential dependency chain).

At N=1 the line also carries sub-records for the other four configs, each
with its own roofline and CPU reference sample.
"""
from __future__ import annotations

import argparse
import json
import os
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
NOMINAL_INT32_TOPS = 148 * 128 * 1.965e9 / 1e12   # all lanes issuing one 32-bit op per clock


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


_INT32 = None


def int32_peak(dev: int):
    """Measured INT32 lane-instruction peak (tools/peaks/int32_peak.cu): best of
    LOP3, IADD3 and LOP3+IMAD, in Tops/s; falls back to the nominal figure."""
    global _INT32
    if _INT32 is None:
        import ctypes as C

        so = ROOT / "tools" / "peaks" / "libint32peak.so"
        try:
            lib = C.CDLL(str(so))
            out = (C.c_double * 3)()
            rc = lib.int32_peak(dev, 3, out)
            if rc != 0:
                raise RuntimeError(f"int32_peak rc={rc}")
            mix = {"lop3": out[0], "iadd3": out[1], "lop3_imad": out[2]}
            _INT32 = (max(mix.values()), "measured live (tools/peaks/int32_peak.cu)", mix)
        except Exception as e:  # noqa: BLE001 - report, do not fail the bench
            _INT32 = (NOMINAL_INT32_TOPS, f"nominal (measurement unavailable: {e})", {})
    return _INT32


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every ~0.25 ms, plus one sample at
    the start) while the enqueued timed steps run."""

    REASONS = {  # nvmlClocksEventReasons bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
    }

    def __init__(self, device: int):
        self.device = device
        self.period = float(os.environ.get("RXG_CLOCK_PERIOD_S", "0.00025"))
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
        if self.h is not None:
            self.stop.clear()
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.h is not None:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted({n for _, b in self.rows for n, m in self.REASONS.items() if b & m})
        return {"sm_mhz": float(np.median([m for m, _ in self.rows])), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.rows)}


def count_units(text: np.ndarray, delim: int, stride: int) -> int:
    if delim == -2:
        return 1
    if delim < 0:
        return len(text) // stride
    n = int(np.count_nonzero(text == delim))
    return n + (1 if len(text) and text[-1] != delim else 0)


def roofline(nbytes: int, words: int, kern_ms: float, traffic, cfg: str, dev: int, bitset: bool = False) -> dict:
    """The dominant kernel against the roofline that binds its algorithm.

    SURVEY.md §8(d) models a BITSET lockstep step: t_roof = max(B / BW_HBM,
    B·W / INT32_peak), W 32-bit state-word updates per input byte. The
    memoized-step (DFA) kernels do O(1) work per byte whatever W is, so their
    binding roofline is HBM (every input byte read once); the survey model is
    reported beside it (`survey_model`) and binds only the bitset kernels."""
    bw, bw_src = hbm_peak()
    i32, i32_src, mix = int32_peak(dev)
    t = kern_ms / 1e3
    t_hbm = nbytes / (bw * 1e9)
    t_int = nbytes * words / (i32 * 1e12)
    achieved_gbs = nbytes / t / 1e9
    survey = {"bound": "hbm" if t_hbm >= t_int else "int32", "t_roof_ms": max(t_hbm, t_int) * 1e3,
              "frac": max(t_hbm, t_int) / t, "int32_t_roof_ms": t_int * 1e3, "int32_peak_tops": i32,
              "int32_peak_source": i32_src, "int32_mix_tops": mix, "state_words": words,
              "model": "max(B/BW_HBM, B*W/INT32_peak)"}
    if bitset and t_int > t_hbm:
        r = {"bound": "int32", "achieved": nbytes * words / t / 1e12, "peak": i32,
             "unit": "Tops/s (32-bit state-word updates, B*W)", "frac": t_int / t}
    else:
        r = {"bound": "hbm", "achieved": achieved_gbs, "peak": bw, "unit": "GB/s", "frac": achieved_gbs / bw}
    r.update({
        "traffic": traffic,
        "traffic_source": (f"dram__bytes_read.sum+dram__bytes_write.sum per launch from an earlier ncu --set full "
                           f"capture of config ({cfg}) (profiles/traffic.json), not measured in this run")
        if traffic else None,
        "algorithmic_bytes_per_launch": nbytes,
        "peak_source": bw_src if r["bound"] == "hbm" else i32_src,
        "survey_model": survey,
    })
    return r


# ── CPU legs (reference library compiled from /root/reference sources) ─────

def cpu_reference(cfg: str, pattern: str, text: np.ndarray, target_s: float = 12.0, threads: int | None = None):
    """Time rx::lockstep_accepts (oracle/_ref) on a bounded sample of the
    workload with all host threads. Returns (GB/s, sample description, cores, kind, seconds)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_bind import REF_SO, Oracle, RefHeap

    threads = threads or os.cpu_count() or 1
    delim, stride, _ = CONFIGS[cfg]
    kind = "reference" if REF_SO.exists() else "port"
    if kind == "reference":
        h = RefHeap(pattern.encode())
    else:
        from paper_1108_3126_b200 import rx   # front end only: the port needs the heap table

        h = Oracle(rx.compile(rx.parse(pattern)))

    def run(sample: np.ndarray, nthreads: int):
        if delim == -2:   # one string: one core
            t0 = time.perf_counter()
            ok = h.accepts(sample.tobytes())
            return time.perf_counter() - t0, int(ok)
        if kind == "reference":
            # decode_utf8 happens in ref_prepare; time only lockstep_accepts
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


def cpu_record(cfg, pattern, text, target_s):
    try:
        gbs, sdesc, cores, kind, _ = cpu_reference(cfg, pattern, text, target_s=target_s)
        return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind, "sample": sdesc, "cpu_model": cpu_model()}
    except Exception as e:  # noqa: BLE001 - the baseline is reported, never the product path
        return {"value": None, "unit": "GB/s", "cores": None, "kind": None, "sample": f"unavailable: {e}",
                "cpu_model": cpu_model()}


# ── reference arm ──────────────────────────────────────────────────────────

def run_reference_arm(args):
    """The reference's own CPU lockstep matcher (oracle/_ref = proj/src compiled
    from source) on a bounded sample of the same workload, all host threads.
    The inputs come from the C restatement of the generators (oracle/), so
    this arm never loads the product library. The sample is sized once
    (~args.ref_step_s per step, so --steps 20 --warmup 5 ends in a few
    minutes; the full (c) job takes ~60 s per pass on 16 cores) and decoded
    once; each step times rx::lockstep_accepts over all of its strings."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bind as ob

    cfg = args.config
    delim, stride, _ = CONFIGS[cfg]
    pattern, text = ob.synth_pattern(cfg), ob.synth_input(cfg)
    threads = os.cpu_count() or 1
    _, desc, cores, kind, _ = cpu_reference(cfg, pattern, text, target_s=args.ref_step_s, threads=threads)
    nbytes = int(desc.split()[1])
    sample = text[:nbytes]
    if kind == "reference":
        h = ob.RefHeap(pattern.encode())
        if delim == -2:
            w = sample.tobytes()
            run = lambda: h.accepts(w)  # noqa: E731
        else:
            a = np.ascontiguousarray(sample)
            prep = h.l.ref_prepare(a.ctypes.data, a.nbytes, delim, stride)
            run = lambda: h.l.ref_run(h.p, prep, None, cores)  # noqa: E731
    else:
        from paper_1108_3126_b200 import rx

        o = ob.Oracle(rx.compile(rx.parse(pattern)))
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
        "higher_is_better": True, "scaling": "strong" if delim != -2 else "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"config ({cfg}): {CONFIGS[cfg][2]}", "input_bytes": int(len(text)),
                   "sample_bytes": int(len(sample))},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": kind, "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ── B200 arm ───────────────────────────────────────────────────────────────

class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.args = args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dev = self.local
        torch.cuda.set_device(self.dev)
        self.comm = None
        if self.world > 1:
            from paper_1108_3126_b200 import rx

            uid = [rx.Comm.unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            self.comm = rx.Comm(uid[0], self.world, self.rank, self.dev)
        self.clk = ClockSampler(self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def timed(ctx, step, steps: int, flush, clocks: bool):
    """K steps on the device, events on the launching stream. Inputs larger
    than L2: one interval around all K steps; otherwise L2 is flushed before
    every step (outside the interval) and the intervals are summed.
    Returns (ms per step on this rank, max over ranks)."""
    torch = ctx.torch
    stream = torch.cuda.current_stream(ctx.dev)
    ctx.barrier()
    # A device-side spin (outside the timed interval) holds the stream while the
    # host enqueues the K steps, so first-call host latency never shows up as an
    # idle gap inside an interval. Host costs per call are what e2e measures.
    torch.cuda._sleep(int(2.0e6 * (0.3 + 0.02 * steps)))
    if flush is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        ev = [(e0, e1)]
    else:
        ev = []
        for _ in range(steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            ev.append((e0, e1))
    if clocks:
        with ctx.clk:
            torch.cuda.synchronize(ctx.dev)
    else:
        torch.cuda.synchronize(ctx.dev)
    total = float(sum(a.elapsed_time(b) for a, b in ev))
    ctx.barrier()
    return total / steps, ctx.max_over_ranks(total) / steps


def make_flush(ctx, nbytes: int):
    torch = ctx.torch
    if nbytes >= 256 << 20:
        return None, "inputs larger than L2 (126 MB)"
    dirty = torch.empty(512 << 20, dtype=torch.uint8, device=ctx.dev)
    clean = torch.ones(256 << 20, dtype=torch.uint8, device=ctx.dev)

    def flush():
        # write a buffer larger than L2, then read another one so the lines the
        # timed kernel finds in L2 are clean (no write-back during the step)
        dirty.zero_()
        clean.sum(dtype=torch.int64)

    return flush, "L2 flushed between timed steps (512 MiB write, then 256 MiB read)"


def bench_batch(ctx, cfg: str, steps: int, warmup: int, headline: bool, engine: str = "auto") -> dict:
    """Strong scaling: the job is the config's whole buffer; rank r matches its shard.
    engine: "auto" (memoized step, K2) or "bitset" (K2b, SURVEY.md §8(d)'s bitset step)."""
    from paper_1108_3126_b200 import _lib, rx

    torch = ctx.torch
    delim, stride, desc = CONFIGS[cfg]
    pattern, text = rx.synth_pattern(cfg), rx.synth_input(cfg, seed=0)
    job_bytes = len(text)
    bounds = rx.shard_bounds(text, ctx.world, delimiter=delim if delim >= 0 else -1, stride=stride)
    lo, hi = rx.shard(text, ctx.world, ctx.rank, delimiter=delim if delim >= 0 else -1, stride=stride)
    shard = text[lo:hi]
    nb = len(shard)
    m = rx.Matcher(pattern, device=ctx.dev)
    if delim >= 0:   # planner: bank placement from the head of the JOB (identical tables on every rank)
        m.tune(text[: 1 << 20], delimiter=delim)
    info = m.info()
    host = torch.from_numpy(shard).pin_memory()
    d_text = torch.empty(nb + 64, dtype=torch.uint8, device=ctx.dev)
    d_text[:nb].copy_(host)
    d_count = torch.zeros(1, dtype=torch.int64, device=ctx.dev)
    stream = torch.cuda.current_stream(ctx.dev)
    flush, l2 = make_flush(ctx, nb)

    def kernel_step():
        m.match_batch_device(d_text, d_count, delimiter=delim, stride=stride, stream=stream, nbytes=nb, engine=engine)

    def job_step():
        if ctx.comm is None or engine != "auto":
            kernel_step()
        else:
            rx.match_batch_allreduce(m, ctx.comm, d_text, d_count, delimiter=delim, stride=stride, stream=stream,
                                     nbytes=nb)

    for _ in range(warmup):
        job_step()
    torch.cuda.synchronize(ctx.dev)
    launches = _lib.lib().rxg_last_launch_count()
    matches = int(d_count.item())   # the job's total (all-reduced when N > 1)
    _, ms_step = timed(ctx, job_step, steps, flush, clocks=headline)
    if ctx.world > 1:
        for _ in range(2):
            kernel_step()
        kern_local, kern_max = timed(ctx, kernel_step, steps, flush, clocks=False)
    else:
        kern_local, kern_max = ms_step, ms_step
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and ctx.world == 1:
        traffic = json.loads(tf.read_text()).get(cfg)
    rec = {
        "metric": "input GB/s matched",
        "value": job_bytes / (ms_step / 1e3) / 1e9,
        "unit": "GB/s",
        "ms_per_step": ms_step,
        "scaling": "strong",
        "config": {
            "workload": f"config ({cfg}): {desc}",
            "pattern_nodes": info["nodes"], "positions": info["positions"], "words": info["words"],
            "dfa_states": info["dfa_states"], "line_col_bytes": m.info()["line_col_bytes"],
            "job_bytes": job_bytes, "job_strings": count_units(text, delim, stride),
            "shard_bytes_rank0": int(bounds[1] - bounds[0]), "shards": [int(x) for x in bounds],
            "matches": matches, "l2": l2,
            "parallelism": f"dp{ctx.world} (string shards, count all-reduce over NCCL)" if ctx.world > 1 else "dp1",
            "engine": ("k2b_bitset_" if engine == "bitset" else "k2_") + ("lines" if delim >= 0 else "fixed"),
        },
        "roofline": roofline(nb, info["words"], kern_local, traffic if engine == "auto" else None, cfg, ctx.dev,
                             bitset=engine == "bitset"),
        "gpu_launches": launches * steps,
    }
    if ctx.world > 1:
        rec["spans"] = {"kernel_ms_per_step": kern_max, "kernel_plus_allreduce_ms_per_step": ms_step,
                        "kernel_value": job_bytes / (kern_max / 1e3) / 1e9,
                        "note": "max over ranks; kernel = this rank's shard only, no collective"}
    # end to end through the C ABI with host buffers: this rank's shard, H2D
    # inside the call (pipelined 64 MiB pieces), the count read back, then the
    # 8-byte count all-reduce across ranks
    if not ctx.args.no_e2e and engine == "auto":
        def e2e_time(buf):
            m.match_batch(buf, delimiter=delim, stride=stride)   # warm
            ctx.barrier()
            k = max(1, steps // 2)
            t0 = time.perf_counter()
            for _ in range(k):
                cnt, _ = m.match_batch(buf, delimiter=delim, stride=stride)
                if ctx.world > 1:
                    c = torch.tensor([cnt], dtype=torch.int64, device=ctx.dev)
                    ctx.dist.all_reduce(c)
                    c.item()
            return ctx.max_over_ranks((time.perf_counter() - t0) / k)

        t_pin = e2e_time(host.numpy())
        t_page = e2e_time(shard)
        rec["e2e"] = {"value": job_bytes / t_pin / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nb,
                      "d2h_bytes_per_step": 8, "host_buffer": "pinned",
                      "pageable": {"value": job_bytes / t_page / 1e9, "unit": "GB/s"}}
    if ctx.world > 1 and engine == "auto":   # secondary: weak scaling (every rank the whole job)
        d_full = torch.empty(job_bytes + 64, dtype=torch.uint8, device=ctx.dev)
        d_full[:job_bytes].copy_(torch.from_numpy(text))

        def weak_step():
            rx.match_batch_allreduce(m, ctx.comm, d_full, d_count, delimiter=delim, stride=stride, stream=stream,
                                     nbytes=job_bytes)

        for _ in range(2):
            weak_step()
        _, wms = timed(ctx, weak_step, steps, make_flush(ctx, job_bytes)[0], clocks=False)
        rec["weak"] = {"value": ctx.world * job_bytes / (wms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": wms,
                       "note": "every rank matches the whole job, count all-reduce"}
        del d_full
    if ctx.rank == 0 and ctx.world == 1 and not ctx.args.no_cpu and engine == "auto":
        rec["cpu_baseline"] = cpu_record(cfg, pattern, text, ctx.args.cpu_target_s if headline else ctx.args.sub_cpu_s)
    return rec


def bench_single(ctx, cfg: str, steps: int, warmup: int, headline: bool, engine: str | None = None) -> dict:
    """One long string (replicas only when N > 1). engine: single-string engine
    ("auto" = the chunk-parallel memoized step; "pernode" = K1, the paper's
    thread-per-node scheme, segmented across SMs)."""
    from paper_1108_3126_b200 import _lib, rx

    torch = ctx.torch
    pattern, text = rx.synth_pattern(cfg), rx.synth_input(cfg, seed=0)
    nb = len(text)
    m = rx.Matcher(pattern, device=ctx.dev)
    m.tune(text[: 1 << 20], delimiter=-1)
    info = m.info()
    host = torch.from_numpy(text).pin_memory()
    d_text = torch.empty(nb + 64, dtype=torch.uint8, device=ctx.dev)
    d_text[:nb].copy_(host)
    d_acc = torch.zeros(1, dtype=torch.int32, device=ctx.dev)
    stream = torch.cuda.current_stream(ctx.dev)
    flush, l2 = make_flush(ctx, nb)
    engine = engine or ctx.args.engine

    def step():
        m.match_one_device(d_text[:nb], d_acc, engine=engine, stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(ctx.dev)
    launches = _lib.lib().rxg_last_launch_count()
    accept = int(d_acc.item())
    local, ms_step = timed(ctx, step, steps, flush, clocks=headline)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(cfg)
    rec = {
        "metric": "input GB/s matched",
        "value": ctx.world * nb / (ms_step / 1e3) / 1e9,
        "unit": "GB/s",
        "ms_per_step": ms_step,
        "scaling": "weak",
        "config": {
            "workload": f"config ({cfg}): {CONFIGS[cfg][2]}",
            "pattern_nodes": info["nodes"], "positions": info["positions"], "words": info["words"],
            "dfa_states": info["dfa_states"], "chunk_lookback": m.info()["chunk_lookback"], "input_bytes": nb,
            "accept": accept, "l2": l2,
            "parallelism": f"{ctx.world} replicas (one string is a sequential chain)" if ctx.world > 1 else "dp1",
            "engine": engine,
            "ns_per_symbol": ms_step * 1e6 / nb,
        },
        "roofline": roofline(nb, info["words"], local, traffic, cfg, ctx.dev),
        "gpu_launches": launches * steps,
    }
    if not ctx.args.no_e2e and engine == "auto":
        def e2e_time(w):
            m.lockstep_accepts(w)   # warm
            k = max(1, steps // 2)
            t0 = time.perf_counter()
            for _ in range(k):
                m.lockstep_accepts(w)
            return ctx.max_over_ranks((time.perf_counter() - t0) / k)

        t = e2e_time(host.numpy())
        tp = e2e_time(text)
        rec["e2e"] = {"value": ctx.world * nb / t / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nb,
                      "d2h_bytes_per_step": 4, "host_buffer": "pinned",
                      "pageable": {"value": ctx.world * nb / tp / 1e9, "unit": "GB/s"}}
    if ctx.rank == 0 and ctx.world == 1 and not ctx.args.no_cpu and engine == "auto":
        rec["cpu_baseline"] = cpu_record(cfg, pattern, text, ctx.args.cpu_target_s if headline else ctx.args.sub_cpu_s)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--engine", default="auto", help="single-string engine (a, e)")
    ap.add_argument("--batch-engine", default="auto", choices=["auto", "bitset"], help="batch engine (b, c, d)")
    ap.add_argument("--bitset-subs", default="cd", help="forced-bitset (K2b) sub-records at N=1 ('' = none)")
    ap.add_argument("--k1-subs", default="e", help="K1 (engine=pernode) sub-records at N=1 ('' = none)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="headline config only (no sub-records)")
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--cpu-target-s", type=float, default=12.0)
    ap.add_argument("--sub-cpu-s", type=float, default=6.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    args.warmup = max(args.warmup, 3)

    ctx = Ctx(args)
    cfg = args.config

    def run(c, headline, engine=None):
        if CONFIGS[c][0] == -2:
            return bench_single(ctx, c, args.steps, args.warmup, headline)
        return bench_batch(ctx, c, args.steps, args.warmup, headline, engine or args.batch_engine)

    rec = run(cfg, True)
    subs = {}
    if ctx.world == 1 and not args.no_sub:
        for c in sorted(CONFIGS):
            if c != cfg:
                try:
                    subs[c] = run(c, False)
                except Exception as e:  # noqa: BLE001 - a failing sub-record must not hide the headline
                    subs[c] = {"error": repr(e)}
                ctx.torch.cuda.empty_cache()
        for c in args.bitset_subs:
            try:
                subs[c + "_bitset"] = run(c, False, "bitset")
            except Exception as e:  # noqa: BLE001
                subs[c + "_bitset"] = {"error": repr(e)}
            ctx.torch.cuda.empty_cache()
        for c in args.k1_subs:   # the paper's thread-per-node scheme on the single-string configs
            try:
                subs[c + "_k1"] = bench_single(ctx, c, max(2, args.steps // 4), 2, False, engine="pernode")
            except Exception as e:  # noqa: BLE001
                subs[c + "_k1"] = {"error": repr(e)}
            ctx.torch.cuda.empty_cache()
    if ctx.rank == 0:
        line = {
            "metric": "input GB/s matched",
            "value": rec["value"],
            "unit": "GB/s",
            "n_gpus": ctx.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": rec["ms_per_step"],
            "higher_is_better": True,
            "scaling": rec["scaling"],
            "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic",
            "config": rec["config"],
            "roofline": rec["roofline"],
            "cpu_baseline": rec.get("cpu_baseline"),
            "e2e": rec.get("e2e"),
            "gpu_launches": rec["gpu_launches"],
            "clocks": ctx.clk.summary(),
        }
        for k in ("spans", "weak"):
            if k in rec:
                line[k] = rec[k]
        if subs:
            line["configs"] = subs
        print(json.dumps(line), flush=True)
    if ctx.comm is not None:
        ctx.comm.close()
    if ctx.world > 1:
        ctx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
