"""Host-side mirror of the reference matcher API (proj/include/rx), backed by
librxg.so. Names, argument meaning and error behaviour follow the reference:

  parse(text)              rx::parse            regex.hpp:60    raises ParseError(pos) / Utf8Error
  compile(e)               rx::compile          heap.hpp:43     -> Heap {nodes, knodes}, root 0
  dump(h) / parse_dump(t)  rx::dump/parse_dump  heap.hpp:68-69
  check_knode(h)           rx::check_knode      heap.hpp:52
  print_regex(e)           rx::print            regex.hpp:65
  lockstep_accepts(h, w)   rx::lockstep_accepts lockstep.hpp:43 (runs on the GPU)
  par_accepts(h, w)        rx::par_accepts      parallel.hpp:102 (paper §8 scheme on the GPU)

The GPU-facing object is ``Matcher`` (one compiled heap resident on one
device). Inputs are bytes; str inputs are UTF-8 encoded.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

NODE_EPS, NODE_CHR, NODE_ALT, NODE_SEQ, NODE_STAR = range(5)
NULL_ADDR = -1
_KIND_NAMES = {NODE_EPS: "Eps", NODE_CHR: "Chr", NODE_ALT: "Alt", NODE_SEQ: "Seq", NODE_STAR: "Star"}


class RxgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} [{L.lib().rxg_strerror(status).decode()}]")
        self.status = status


class ParseError(ValueError):
    """rx::ParseError (regex.hpp:50-54): `pos` is the offset in Unicode scalars."""

    def __init__(self, pos: int, msg: str):
        super().__init__(msg)
        self.pos = pos


class Utf8Error(ValueError):
    def __init__(self, at: int, msg: str):
        super().__init__(msg)
        self.at = at


def _check(rc: int):
    if rc != L.RXG_OK:
        raise RxgError(rc, L.lib().rxg_last_error().decode(errors="replace"))


def _b(x) -> bytes:
    if isinstance(x, str):
        return x.encode("utf-8")
    return bytes(x)


@dataclass(frozen=True)
class Node:
    kind: int
    sym: int
    left: int
    right: int


class Regex:
    """A validated pattern (the reference's RegexPtr is only consumed by compile/print here)."""

    def __init__(self, text: bytes):
        self.text = text

    def __repr__(self):
        return f"Regex({self.text!r})"


class Heap:
    """rx::Heap (heap.hpp:28-37): address-indexed nodes plus the continuation map."""

    def __init__(self, nodes: list[Node], knodes: list[int]):
        self.nodes = nodes
        self.knodes = knodes

    def root(self) -> int:
        return 0

    def size(self) -> int:
        return len(self.nodes)

    def node(self, p: int) -> Node:
        return self.nodes[p]

    def knode(self, p: int) -> int:
        return self.knodes[p]

    def _c(self):
        n = len(self.nodes)
        arr = (L.rxg_node * n)()
        for i, x in enumerate(self.nodes):
            arr[i].kind, arr[i].sym, arr[i].left, arr[i].right = x.kind, x.sym, x.left, x.right
        kn = (C.c_int32 * n)(*self.knodes)
        return arr, kn, n

    def __eq__(self, other):
        return isinstance(other, Heap) and self.nodes == other.nodes and self.knodes == other.knodes


def _heap_from_c(arr, kn, n) -> Heap:
    return Heap([Node(arr[i].kind, arr[i].sym, arr[i].left, arr[i].right) for i in range(n)], list(kn[:n]))


def parse(text) -> Regex:
    """rx::parse: raises ParseError / Utf8Error like the reference."""
    t = _b(text)
    n = C.c_int32(0)
    pos = C.c_size_t(0)
    rc = L.lib().rxg_parse_compile(t, len(t), None, None, 0, C.byref(n), C.byref(pos))
    if rc == L.RXG_EPARSE:
        raise ParseError(pos.value, L.lib().rxg_last_error().decode())
    if rc == L.RXG_EUTF8:
        raise Utf8Error(pos.value, L.lib().rxg_last_error().decode())
    _check(rc)
    return Regex(t)


def compile(e: Regex) -> Heap:  # noqa: A001 - mirrors rx::compile
    t = e.text
    n = C.c_int32(0)
    pos = C.c_size_t(0)
    _check(L.lib().rxg_parse_compile(t, len(t), None, None, 0, C.byref(n), C.byref(pos)))
    arr = (L.rxg_node * n.value)()
    kn = (C.c_int32 * n.value)()
    _check(L.lib().rxg_parse_compile(t, len(t), arr, kn, n.value, C.byref(n), C.byref(pos)))
    return _heap_from_c(arr, kn, n.value)


def print_regex(e: Regex) -> str:
    ln = C.c_size_t(0)
    _check(L.lib().rxg_print(e.text, len(e.text), None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _check(L.lib().rxg_print(e.text, len(e.text), buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode("utf-8")


def dump(h: Heap) -> str:
    arr, kn, n = h._c()
    ln = C.c_size_t(0)
    _check(L.lib().rxg_dump(arr, kn, n, None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _check(L.lib().rxg_dump(arr, kn, n, buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode("utf-8")


def parse_dump(text: str) -> Heap:
    t = _b(text)
    n = C.c_int32(0)
    rc = L.lib().rxg_parse_dump(t, len(t), None, None, 0, C.byref(n))
    if rc != L.RXG_OK:
        raise RuntimeError(L.lib().rxg_last_error().decode())
    arr = (L.rxg_node * n.value)()
    kn = (C.c_int32 * n.value)()
    _check(L.lib().rxg_parse_dump(t, len(t), arr, kn, n.value, C.byref(n)))
    return _heap_from_c(arr, kn, n.value)


def check_knode(h: Heap) -> bool:
    arr, kn, n = h._c()
    ok = C.c_int32(0)
    _check(L.lib().rxg_check_knode(arr, kn, n, C.byref(ok)))
    return bool(ok.value)


def _ptr(buf) -> tuple[int, int, object]:
    """(address, nbytes, keepalive) of a bytes-like / numpy / torch buffer."""
    try:
        import torch

        if isinstance(buf, torch.Tensor):
            assert buf.dtype == torch.uint8 and buf.is_contiguous()
            return buf.data_ptr(), buf.numel(), buf
    except ImportError:  # pragma: no cover
        pass
    if isinstance(buf, np.ndarray):
        a = np.ascontiguousarray(buf, dtype=np.uint8)
        return a.ctypes.data, a.nbytes, a
    b = _b(buf)
    cbuf = C.create_string_buffer(b, len(b)) if b else C.create_string_buffer(1)
    return C.addressof(cbuf), len(b), cbuf


class Matcher:
    """A compiled heap with its derived tables resident on one GPU (rxg_heap).

    device < 0 builds a host-only handle (tables and the host model of the
    step, no kernels).
    """

    def __init__(self, pattern_or_heap, device: int = 0):
        self._h = C.c_void_p()
        if isinstance(pattern_or_heap, Heap):
            arr, kn, n = pattern_or_heap._c()
            _check(L.lib().rxg_heap_create(arr, kn, n, device, C.byref(self._h)))
        else:
            t = pattern_or_heap.text if isinstance(pattern_or_heap, Regex) else _b(pattern_or_heap)
            rc = L.lib().rxg_heap_create_pattern(t, len(t), device, C.byref(self._h))
            if rc == L.RXG_EPARSE:
                raise ParseError(-1, L.lib().rxg_last_error().decode())
            _check(rc)
        self.device = device

    def close(self):
        if self._h:
            L.lib().rxg_heap_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        i = L.rxg_heap_info()
        _check(L.lib().rxg_heap_info_get(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in L.rxg_heap_info._fields_}

    def tune(self, sample, delimiter: int = 10):
        """Planner hint: place table rows for the state/byte mix of `sample` (speed only)."""
        p, n, keep = _ptr(sample)
        _check(L.lib().rxg_heap_tune(self._h, p, n, delimiter))

    def tables(self):
        """(pos_addr, follow[(|C|+1) x W], init[W]) of the position form."""
        inf = self.info()
        npos, W = inf["positions"], inf["words"]
        pos = np.zeros(npos, np.int32)
        fol = np.zeros((npos + 1, W), np.uint32)
        ini = np.zeros(W, np.uint32)
        _check(L.lib().rxg_heap_tables(self._h, pos.ctypes.data, fol.ctypes.data, ini.ctypes.data))
        return pos, fol, ini

    def host_walk(self, w):
        """Host model of the kernels' step: (E sets per step [(len+1) x W], accept)."""
        p, n, keep = _ptr(w)
        W = self.info()["words"]
        sets = np.zeros((n + 1, W), np.uint32)
        acc = C.c_int32(0)
        _check(L.lib().rxg_host_walk(self._h, p, n, sets.ctypes.data, C.byref(acc)))
        return sets, bool(acc.value)

    def emulate_batch(self, text, delimiter: int = 10, stride: int = 0, chunk: int = 0):
        """Host emulation of the batch kernels over the same table image -> (count, results)."""
        p, n, keep = _ptr(text)
        nstr = count_strings(text, delimiter, stride)
        res = np.zeros(max(nstr, 1) + 1, np.uint8)
        cnt = C.c_uint64(0)
        _check(L.lib().rxg_host_emulate_batch(self._h, p, n, delimiter, stride, chunk, C.byref(cnt),
                                              res.ctypes.data))
        return cnt.value, res[:nstr]

    def emulate_chunk_tma(self, text) -> tuple[bool, int]:
        """Host walk of the single-string TMA table -> (accepted, layout id) (tests)."""
        p, n, keep = _ptr(text)
        acc, lay = C.c_int32(0), C.c_int32(0)
        _check(L.lib().rxg_host_emulate_chunk_tma(self._h, p, n, C.byref(acc), C.byref(lay)))
        return bool(acc.value), lay.value

    def emulate_lines_tma(self, text, delimiter: int = 10, chunk: int = 256) -> int:
        """Host emulation of the TMA line kernel's table layout and partition -> count."""
        p, n, keep = _ptr(text)
        cnt = C.c_uint64(0)
        _check(L.lib().rxg_host_emulate_lines_tma(self._h, p, n, delimiter, chunk, C.byref(cnt)))
        return cnt.value

    def lockstep_accepts(self, w, engine: str = "auto") -> bool:
        p, n, keep = _ptr(w)
        acc = C.c_int32(0)
        _check(L.lib().rxg_match_one(self._h, p, n, L.ENGINES[engine], C.byref(acc)))
        return bool(acc.value)

    def lockstep_stats(self, w):
        """One string through the literal §8 protocol kernel with the reference's
        instrumentation -> (accepted, {enqueued, claims, launches, macro_steps,
        max_claims_per_node_step, schedule_sizes})."""
        p, n, keep = _ptr(w)
        sched = (C.c_uint32 * (n + 1))()
        st = L.rxg_match_stats()
        st.schedule = C.cast(sched, C.POINTER(C.c_uint32))
        acc = C.c_int32(0)
        _check(L.lib().rxg_match_one_stats(self._h, p, n, C.byref(acc), C.byref(st)))
        return bool(acc.value), {"enqueued": st.enqueued, "claims": st.claims, "launches": st.launches,
                                 "macro_steps": st.macro_steps, "max_claims_per_node_step": st.max_claims_per_node_step,
                                 "schedule_sizes": list(sched[: st.schedule_len])}

    def match_one_ex(self, d_text, d_accept, engine: str = "auto", stream=None, nbytes: int | None = None, **opts):
        """Async single-string match with engine options / instrumentation (device tensors):
        checkpoint_every + d_checkpoints (pernode), d_stats / d_trace (rounds), chunk / lookback / d_repairs (chunked)."""
        o = L.rxg_one_opts()
        for k, v in opts.items():
            setattr(o, k, v.data_ptr() if hasattr(v, "data_ptr") else v)
        n = d_text.numel() if nbytes is None else nbytes
        _check(L.lib().rxg_match_one_ex(self._h, d_text.data_ptr(), n, L.ENGINES[engine], d_accept.data_ptr(),
                                        C.byref(o), _stream_ptr(stream)))

    def match_one_device(self, d_text, d_accept, engine: str = "auto", stream=None):
        """Async single-string match on device tensors (d_accept: int32 cuda tensor)."""
        _check(L.lib().rxg_match_one_device(self._h, d_text.data_ptr(), d_text.numel(), L.ENGINES[engine],
                                            d_accept.data_ptr(), _stream_ptr(stream)))

    def match_batch_device(self, d_text, d_count, d_results=None, delimiter: int = 10, stride: int = 0,
                           stream=None, nbytes: int | None = None, engine: str = "auto"):
        """Async batch match on device tensors (d_count: int64 cuda tensor of 1)."""
        n = d_text.numel() if nbytes is None else nbytes
        _check(L.lib().rxg_match_batch_ex(self._h, d_text.data_ptr(), n, delimiter, stride, L.BATCH_ENGINES[engine],
                                          d_count.data_ptr(), d_results.data_ptr() if d_results is not None else None,
                                          _stream_ptr(stream)))

    def match_batch(self, text, delimiter: int = 10, stride: int = 0, results: bool = False):
        """Synchronous batch match of a host buffer -> (count, results|None)."""
        p, n, keep = _ptr(text)
        res = None
        if results:
            nstr = count_strings(text, delimiter, stride)
            res = np.zeros(max(nstr, 1) + 1, np.uint8)
        cnt = C.c_uint64(0)
        _check(L.lib().rxg_match_batch_host(self._h, p, n, delimiter, stride, C.byref(cnt),
                                            res.ctypes.data if res is not None else None))
        return cnt.value, (res[:nstr] if res is not None else None)

    def match_batch_utf8(self, text, delimiter: int = 10, stride: int = 0, results: bool = False):
        """match_batch plus the fused device UTF-8 check of every string (the
        `rxvm match` loop: getline, decode_utf8, lockstep_accepts) ->
        (count, results|None, first_bad) with first_bad the byte offset
        rx::decode_utf8 would name, or None when every string decodes."""
        p, n, keep = _ptr(text)
        res = None
        if results:
            nstr = count_strings(text, delimiter, stride)
            res = np.zeros(max(nstr, 1) + 1, np.uint8)
        cnt = C.c_uint64(0)
        bad = C.c_uint64(0)
        _check(L.lib().rxg_match_batch_host_ex(self._h, p, n, delimiter, stride, C.byref(cnt),
                                               res.ctypes.data if res is not None else None, C.byref(bad)))
        return cnt.value, (res[:nstr] if res is not None else None), (None if bad.value == 2**64 - 1 else bad.value)


def set_option(name: str, value=None):
    """rxg_set_option: process-wide tuning / test switch (speed only; None unsets)."""
    _check(L.lib().rxg_set_option(name.encode(), None if value is None else str(value).encode()))


class option:
    """Context manager: `with rx.option("RXG_NO_LT", 1): ...` sets a switch and restores it (unset) after."""

    def __init__(self, name: str, value):
        self.name, self.value = name, value

    def __enter__(self):
        set_option(self.name, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.name, None)


def _stream_ptr(stream):
    if stream is None:
        return None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def utf8_check(text, delimiter: int = -1, stride: int = 0, device: int = 0):
    """Device check of a host buffer against rx::decode_utf8 (utf8.cpp:16-46),
    each string decoded separately (delimiter/stride as match_batch; -1/0 =
    one string) -> None when valid, else the offset of the byte decode_utf8
    names in its "invalid UTF-8 at byte N" error (plus the string's offset)."""
    p, n, keep = _ptr(text)
    bad = C.c_uint64(0)
    _check(L.lib().rxg_utf8_check_host(device, p, n, delimiter, stride, C.byref(bad)))
    return None if bad.value == 2**64 - 1 else bad.value


def utf8_check_device(d_text, nbytes: int, d_first_bad, delimiter: int = -1, stride: int = 0, device: int = 0,
                      stream=None):
    """Asynchronous device variant: d_text / d_first_bad are device pointers
    (ints) or tensors; *d_first_bad = offset or 2**64-1 (int64 -1)."""
    tp = d_text.data_ptr() if hasattr(d_text, "data_ptr") else d_text
    bp = d_first_bad.data_ptr() if hasattr(d_first_bad, "data_ptr") else d_first_bad
    _check(L.lib().rxg_utf8_check(device, C.c_void_p(tp), nbytes, delimiter, stride, C.c_void_p(bp),
                                  _stream_ptr(stream)))


def count_strings(text, delimiter: int = 10, stride: int = 0) -> int:
    """Strings in a host buffer as the batch calls split it (rxg_count_strings)."""
    p, n, keep = _ptr(text)
    out = C.c_uint64(0)
    _check(L.lib().rxg_count_strings(p, n, delimiter, stride, C.byref(out)))
    return out.value


class Comm:
    """A NCCL communicator over one-process-per-GPU ranks (rxg_comm).

    Rank 0 calls ``Comm.unique_id()``; the host plumbing (torch.distributed,
    MPI, a file) broadcasts the 128 bytes; every rank then constructs
    ``Comm(uid, nranks, rank, device)`` (collective)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(L.lib().rxg_comm_unique_id(buf, 128))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        assert len(uid) == 128
        self._c = C.c_void_p()
        ub = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(L.lib().rxg_comm_init_rank(ub, 128, nranks, rank, device, C.byref(self._c)))
        self.nranks, self.rank, self.device = nranks, rank, device

    def close(self):
        if self._c:
            L.lib().rxg_comm_destroy(self._c)
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def match_batch_allreduce(m: "Matcher", comm: Comm, d_text, d_count, d_results=None, delimiter: int = 10,
                          stride: int = 0, stream=None, nbytes: int | None = None):
    """This rank's shard through K2, then the NCCL sum of d_count over the ranks, on `stream`."""
    n = d_text.numel() if nbytes is None else nbytes
    _check(L.lib().rxg_match_batch_allreduce(m.handle, comm._c, d_text.data_ptr(), n, delimiter, stride,
                                             d_count.data_ptr(),
                                             d_results.data_ptr() if d_results is not None else None,
                                             _stream_ptr(stream)))


class MultiMatcher:
    """One pattern resident on several GPUs (rxg_multi): tables built once and
    uploaded per device, one worker thread per device, communicators created
    once. A device may be listed twice (the counts are then summed on the host)."""

    def __init__(self, devices, pattern):
        devs = (C.c_int * len(devices))(*devices)
        pat = _b(pattern)
        self._m = C.c_void_p()
        _check(L.lib().rxg_multi_create(devs, len(devices), pat, len(pat), C.byref(self._m)))
        self.devices = list(devices)

    def close(self):
        if self._m:
            L.lib().rxg_multi_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        n, u = C.c_int32(0), C.c_int32(0)
        _check(L.lib().rxg_multi_info(self._m, C.byref(n), C.byref(u)))
        return {"devices": n.value, "nccl": bool(u.value)}

    def tune(self, sample, delimiter: int = 10):
        p, n, keep = _ptr(sample)
        _check(L.lib().rxg_multi_tune(self._m, p, n, delimiter))

    def match_batch(self, text, delimiter: int = 10, stride: int = 0, results: bool = False):
        """Shard a host buffer over the devices -> (count, results|None)."""
        p, n, keep = _ptr(text)
        res = None
        if results:
            nstr = count_strings(text, delimiter, stride)
            res = np.zeros(max(nstr, 1) + 1, np.uint8)
        cnt = C.c_uint64(0)
        _check(L.lib().rxg_multi_match_batch(self._m, p, n, delimiter, stride, C.byref(cnt),
                                             res.ctypes.data if res is not None else None))
        return cnt.value, (res[:nstr] if res is not None else None)


def match_batch_multi(devices, pattern, text, delimiter: int = 10, stride: int = 0, results: bool = False):
    """One-shot: shard a host buffer over several GPUs; one NCCL all-reduce of the count."""
    devs = (C.c_int * len(devices))(*devices)
    pat = _b(pattern)
    p, n, keep = _ptr(text)
    res = None
    if results:
        nstr = count_strings(text, delimiter, stride)
        res = np.zeros(max(nstr, 1) + 1, np.uint8)
    cnt = C.c_uint64(0)
    _check(L.lib().rxg_match_batch_multi(devs, len(devices), pat, len(pat), p, n, delimiter, stride, C.byref(cnt),
                                         res.ctypes.data if res is not None else None))
    return cnt.value, (res[:nstr] if res is not None else None)


def match_many(patterns, text, delimiter: int = 10, stride: int = 0, device: int = 0) -> np.ndarray:
    """Every pattern against every string (the crosscheck sweep shape) -> [n_patterns, n_strings] 0/1."""
    blob = b"".join(_b(p) + b"\0" for p in patterns)
    p, n, keep = _ptr(text)
    nstr = count_strings(text, delimiter, stride) if delimiter >= 0 else n // stride
    res = np.zeros(max(len(patterns) * nstr, 1), np.uint8)
    ns = C.c_uint64(0)
    bad = C.c_int32(-1)
    _check(L.lib().rxg_match_many(device, blob, len(patterns), p, n, delimiter, stride, res.ctypes.data,
                                  C.byref(ns), C.byref(bad)))
    return res[: len(patterns) * ns.value].reshape(len(patterns), ns.value)


def match_one_multi(devices, pattern, text):
    """One long string split over several GPUs (chunk-speculative across
    devices, exact) -> (accept, segments re-run)."""
    devs = (C.c_int * len(devices))(*devices)
    pat = _b(pattern)
    p, n, keep = _ptr(text)
    acc = C.c_int32(0)
    rer = C.c_int32(0)
    _check(L.lib().rxg_match_one_multi(devs, len(devices), pat, len(pat), p, n, C.byref(acc), C.byref(rer)))
    return bool(acc.value), rer.value


def shard(text, nshards: int, index: int, delimiter: int = 10, stride: int = 0) -> tuple[int, int]:
    """[lo, hi) of shard `index` of a job cut into `nshards` byte-balanced shards at
    string boundaries (rxg_shard_bounds): what rank `index` of a strong-scaled run matches."""
    b = shard_bounds(text, nshards, delimiter, stride)
    return b[index], b[index + 1]


def shard_bounds(text, ndev: int, delimiter: int = 10, stride: int = 0) -> list[int]:
    p, n, keep = _ptr(text)
    off = (C.c_uint64 * (ndev + 1))()
    _check(L.lib().rxg_shard_bounds(p, n, delimiter, stride, ndev, off))
    return list(off)


_matchers: dict = {}


def lockstep_accepts(h: Heap, w, device: int = 0) -> bool:
    """rx::lockstep_accepts(const Heap&, InputView) on the GPU."""
    key = (id(h), device)
    m = _matchers.get(key)
    if m is None or m[0] is not h:
        m = (h, Matcher(h, device))
        _matchers[key] = m
    return m[1].lockstep_accepts(w)


def synth_pattern(config: str) -> str:
    ln = C.c_size_t(0)
    _check(L.lib().rxg_synth_pattern(config.encode(), None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _check(L.lib().rxg_synth_pattern(config.encode(), buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode()


def synth_input(config: str, nbytes: int | None = None, seed: int = 0, out=None) -> np.ndarray:
    """Synthetic input of a SURVEY §8(d) config (first `nbytes`, default the full size)."""
    cap = nbytes if nbytes is not None else int(L.lib().rxg_synth_input_size(config.encode()))
    buf = out if out is not None else np.empty(cap, np.uint8)
    written = C.c_uint64(0)
    _check(L.lib().rxg_synth_input(config.encode(), seed, buf.ctypes.data, cap, C.byref(written)))
    return buf[: written.value]
