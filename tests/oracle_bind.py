"""TEST INFRASTRUCTURE: ctypes bindings of the CPU checkers under oracle/.

  Oracle   oracle/liboracle.so      plain-C restatement (oracle/lockstep_oracle.c)
  Ref      oracle/_ref/librxref.so  the unmodified reference library + shim

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "librxref.so"


class _Node(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("pad", C.c_uint8 * 3), ("sym", C.c_uint32),
                ("left", C.c_int32), ("right", C.c_int32)]


class _Heap(C.Structure):
    _fields_ = [("nodes", C.POINTER(_Node)), ("knodes", C.POINTER(C.c_int32)), ("n", C.c_int32)]


def build_oracle(with_ref: bool | None = None) -> None:
    """make -C oracle (the reference part only when its sources are present)."""
    import subprocess

    targets = ["liboracle.so"]
    if with_ref is None:
        with_ref = Path("/root/reference/proj/src").exists()
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")] + targets, check=True)


class Oracle:
    """Plain-C restatement of rx::lockstep_accepts over a heap table."""

    @staticmethod
    def _raw():
        if not ORACLE_SO.exists():
            build_oracle(with_ref=False)
        l = C.CDLL(str(ORACLE_SO))
        l.oracle_decode_utf8_error.restype = C.c_int64
        l.oracle_decode_utf8_error.argtypes = [C.c_void_p, C.c_uint64]
        l.oracle_utf8_first_bad.restype = C.c_uint64
        l.oracle_utf8_first_bad.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_uint32]
        return l

    @staticmethod
    def decode_utf8_error(b: bytes):
        """decode_utf8 restated: None or the byte index it throws at."""
        a = np.frombuffer(bytes(b), np.uint8)
        r = Oracle._raw().oracle_decode_utf8_error(a.ctypes.data if len(a) else None, len(a))
        return None if r < 0 else int(r)

    @staticmethod
    def utf8_first_bad(text, delimiter=-1, stride=0):
        a = np.ascontiguousarray(np.frombuffer(bytes(text), np.uint8) if not isinstance(text, np.ndarray) else text)
        r = Oracle._raw().oracle_utf8_first_bad(a.ctypes.data if len(a) else None, len(a), delimiter, stride)
        return None if r == 2**64 - 1 else int(r)

    def __init__(self, heap):
        if not ORACLE_SO.exists():
            build_oracle(with_ref=False)
        self.lib = C.CDLL(str(ORACLE_SO))
        self.lib.oracle_match_batch.restype = C.c_uint64
        self.lib.oracle_match_batch.argtypes = [C.POINTER(_Heap), C.c_void_p, C.c_uint64, C.c_int32, C.c_uint32,
                                                C.c_void_p, C.c_int]
        self.lib.oracle_accepts_bytes.restype = C.c_int
        self.lib.oracle_accepts_bytes.argtypes = [C.POINTER(_Heap), C.c_void_p, C.c_uint64]
        P = C.c_void_p
        for fn, res, args in [("oracle_ws_init", None, [P, C.c_int32]), ("oracle_ws_free", None, [P]),
                              ("oracle_evolve", C.c_int32, [C.POINTER(_Heap), P, P, C.c_int32, P, P]),
                              ("oracle_step_char", C.c_int32, [C.POINTER(_Heap), P, P, C.c_int32, C.c_uint32, P]),
                              ("oracle_eps_reaches_null", C.c_int, [C.POINTER(_Heap), P, P, C.c_int32])]:
            getattr(self.lib, fn).restype = res
            getattr(self.lib, fn).argtypes = args
        n = heap.size()
        self._nodes = (_Node * n)()
        for i, x in enumerate(heap.nodes):
            self._nodes[i].kind, self._nodes[i].sym = x.kind, x.sym
            self._nodes[i].left, self._nodes[i].right = x.left, x.right
        self._knodes = (C.c_int32 * n)(*heap.knodes)
        self.h = _Heap(self._nodes, self._knodes, n)

    def accepts(self, w: bytes) -> bool:
        buf = C.create_string_buffer(bytes(w), max(len(w), 1))
        return bool(self.lib.oracle_accepts_bytes(C.byref(self.h), buf, len(w)))

    def walk_from(self, s, w: bytes) -> set:
        """S after stepping through w from start set s (lockstep.cpp:77-80)."""
        self.lib.oracle_walk_from.restype = C.c_int32
        self.lib.oracle_walk_from.argtypes = [C.POINTER(_Heap), C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64]
        io = np.zeros(self.h.n + 2, np.int32)
        arr = sorted(s)
        io[: len(arr)] = arr
        buf = C.create_string_buffer(bytes(w), max(len(w), 1))
        k = self.lib.oracle_walk_from(C.byref(self.h), io.ctypes.data, len(arr), buf, len(w))
        return set(io[:k].tolist())

    # set-level functions (lockstep.cpp:10-73), sets as Python sets of addresses (-1 = null)
    def _ws(self):
        class WS(C.Structure):
            _fields_ = [("n", C.c_int32), ("seen", C.c_void_p), ("queue", C.c_void_p), ("epoch", C.c_uint32)]
        ws = WS()
        self.lib.oracle_ws_init(C.byref(ws), self.h.n)
        return ws

    def evolve(self, s) -> set:
        k, out = self._evolve(s)
        return set(out[:k].tolist())

    def _evolve(self, s):
        ws = self._ws()
        a = np.array(sorted(s), np.int32)
        out = np.zeros(2 * self.h.n + len(a) + 2, np.int32)
        k = self.lib.oracle_evolve(C.byref(self.h), C.byref(ws), a.ctypes.data, len(a), out.ctypes.data, None)
        self.lib.oracle_ws_free(C.byref(ws))
        return k, out

    def step_char(self, s, a: int) -> set:
        ws = self._ws()
        arr = np.array(sorted(s), np.int32)
        out = np.zeros(2 * self.h.n + len(arr) + 2, np.int32)
        k = self.lib.oracle_step_char(C.byref(self.h), C.byref(ws), arr.ctypes.data, len(arr), a, out.ctypes.data)
        self.lib.oracle_ws_free(C.byref(ws))
        if k < 0:
            raise ValueError("step_char: unevolved member")
        return set(out[:k].tolist())

    def eps_reaches_null(self, s) -> bool:
        ws = self._ws()
        arr = np.array(sorted(s), np.int32)
        r = self.lib.oracle_eps_reaches_null(C.byref(self.h), C.byref(ws), arr.ctypes.data, len(arr))
        self.lib.oracle_ws_free(C.byref(ws))
        return bool(r)

    def match_batch(self, text: np.ndarray, delimiter=10, stride=0, results=True, threads=None):
        a = np.ascontiguousarray(text, np.uint8)
        nstr = _count_strings(a, delimiter, stride)
        res = np.zeros(max(nstr, 1), np.uint8) if results else None
        threads = threads or os.cpu_count() or 1
        cnt = self.lib.oracle_match_batch(C.byref(self.h), a.ctypes.data, a.nbytes, delimiter, stride,
                                          res.ctypes.data if res is not None else None, threads)
        return int(cnt), (res[:nstr] if res is not None else None)


def _raw_synth():
    l = Oracle._raw()
    l.oracle_synth_pattern.restype = C.c_size_t
    l.oracle_synth_pattern.argtypes = [C.c_char, C.c_char_p, C.c_size_t]
    l.oracle_synth_input.restype = C.c_uint64
    l.oracle_synth_input.argtypes = [C.c_char, C.c_uint64, C.c_void_p, C.c_uint64]
    l.oracle_synth_input_size.restype = C.c_uint64
    l.oracle_synth_input_size.argtypes = [C.c_char]
    l.oracle_mt64_nth.restype = C.c_uint64
    l.oracle_mt64_nth.argtypes = [C.c_uint64, C.c_uint64]
    return l


def synth_pattern(cfg: str) -> str:
    """SURVEY.md §8(d) pattern of a config, from the C restatement (no librxg)."""
    l = _raw_synth()
    n = l.oracle_synth_pattern(cfg.encode(), None, 0)
    buf = C.create_string_buffer(n + 1)
    l.oracle_synth_pattern(cfg.encode(), buf, n + 1)
    return buf.value.decode()


def synth_input(cfg: str, nbytes: int | None = None, seed: int = 0) -> np.ndarray:
    """SURVEY.md §8(d) input of a config (first nbytes; c: whole lines), from the C restatement."""
    l = _raw_synth()
    cap = nbytes if nbytes is not None else int(l.oracle_synth_input_size(cfg.encode()))
    buf = np.empty(max(cap, 1), np.uint8)
    n = l.oracle_synth_input(cfg.encode(), seed, buf.ctypes.data, cap)
    return buf[:n]


def mt64_nth(seed: int, n: int) -> int:
    return int(_raw_synth().oracle_mt64_nth(seed, n))


def verify_checkpoints(heap, pos_addr, n_pos, checkpoints, text, every, threads=None):
    """Chunk-parallel check of a long single-string run.
    checkpoints[k] is the position-form set E after (k+1)*every symbols: the
    Chr addresses of evolve(S) plus the accept bit n_pos. Chunk k is re-run by
    the oracle from the Chr addresses of checkpoint k-1 (evolve(E) = E for Chr
    sets; {root} for k = 0) and must end in a set S with evolve(S) equal to
    checkpoint k's Chr addresses and accepts(S) equal to its accept bit.
    Returns the number of chunks verified; raises AssertionError on a mismatch."""
    from concurrent.futures import ThreadPoolExecutor

    o = Oracle(heap)

    def chr_set(row):
        return {int(pos_addr[q]) for q in range(n_pos) if (row[q >> 5] >> (q & 31)) & 1}

    def acc_bit(row):
        return bool((row[n_pos >> 5] >> (n_pos & 31)) & 1)

    def check(k):
        start = {0} if k == 0 else chr_set(checkpoints[k - 1])
        s = o.walk_from(start, bytes(text[k * every:(k + 1) * every]))
        assert o.evolve(s) == chr_set(checkpoints[k]), f"chunk {k}: evolved set differs"
        assert (-1 in s or o.eps_reaches_null(s)) == acc_bit(checkpoints[k]), f"chunk {k}: accept differs"
        return True

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        return sum(ex.map(check, range(len(checkpoints))))


def _count_strings(a, delimiter, stride):
    if delimiter < 0:
        return len(a) // stride
    n = int(np.count_nonzero(a == delimiter))
    if len(a) and a[-1] != delimiter:
        n += 1
    return n


class Ref:
    """The reference library itself (oracle/_ref/librxref.so)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return REF_SO.exists()

    @classmethod
    def lib(cls):
        if cls._lib is None:
            l = C.CDLL(str(REF_SO))
            P = C.c_void_p
            sig = {
                "ref_parse_compile": (C.c_int, [C.c_char_p, C.c_size_t, P, P, C.c_int32, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
                "ref_print": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]),
                "ref_dump": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]),
                "ref_compile": (P, [C.c_char_p, C.c_size_t]),
                "ref_free": (None, [P]),
                "ref_accepts": (C.c_int, [P, P, C.c_size_t, C.POINTER(C.c_uint64)]),
                "ref_par_accepts": (C.c_int, [P, P, C.c_size_t, C.c_uint, C.c_uint64, C.POINTER(C.c_uint64),
                                              C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]),
                "ref_evolve": (C.c_int, [P, P, C.c_int, P]),
                "ref_step_char": (C.c_int, [P, P, C.c_int, C.c_uint32, P]),
                "ref_eps_reaches_null": (C.c_int, [P, P, C.c_int]),
                "ref_trace": (C.c_int, [P, P, C.c_size_t, C.c_char_p, C.c_size_t]),
                "ref_prepare": (P, [P, C.c_uint64, C.c_int32, C.c_uint32]),
                "ref_prepared_count": (C.c_uint64, [P]),
                "ref_prepared_free": (None, [P]),
                "ref_run": (C.c_uint64, [P, P, P, C.c_int]),
                "ref_enumerate": (C.c_int, [C.c_int, C.c_char_p, C.c_char_p, C.c_size_t]),
                "ref_random_regexes": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_uint64, C.c_char_p, C.c_size_t]),
                "ref_decode_utf8_error": (C.c_int64, [P, C.c_size_t]),
            }
            for k, (r, a) in sig.items():
                f = getattr(l, k)
                f.restype, f.argtypes = r, a
            cls._lib = l
        return cls._lib

    @classmethod
    def decode_utf8_error(cls, b: bytes):
        """rx::decode_utf8 itself: None or N of its "invalid UTF-8 at byte N"."""
        a = np.frombuffer(bytes(b), np.uint8)
        r = cls.lib().ref_decode_utf8_error(a.ctypes.data if len(a) else None, len(a))
        assert r != -2
        return None if r < 0 else int(r)

    # ── front end ──
    @classmethod
    def parse_compile(cls, pattern: bytes):
        """-> (nodes [(kind,sym,left,right)], knodes) or raises ValueError(pos, msg)."""
        l = cls.lib()
        n = C.c_int32(0)
        pos = C.c_size_t(0)
        msg = C.create_string_buffer(256)
        rc = l.ref_parse_compile(pattern, len(pattern), None, None, 0, C.byref(n), C.byref(pos), msg, 256)
        if rc == 1:
            raise ValueError(pos.value, msg.value.decode())
        if rc == 2:
            raise RuntimeError(msg.value.decode())
        nodes = (_Node * n.value)()
        kn = (C.c_int32 * n.value)()
        l.ref_parse_compile(pattern, len(pattern), nodes, kn, n.value, C.byref(n), C.byref(pos), msg, 256)
        return [(x.kind, x.sym, x.left, x.right) for x in nodes], list(kn)

    @classmethod
    def _str(cls, fn, *args):
        l = cls.lib()
        n = getattr(l, fn)(*args, None, 0)
        if n < 0:
            raise ValueError("reference call failed")
        buf = C.create_string_buffer(n + 1)
        getattr(l, fn)(*args, buf, n + 1)
        return buf.value.decode("utf-8")

    @classmethod
    def print_regex(cls, pattern: bytes) -> str:
        return cls._str("ref_print", pattern, len(pattern))

    @classmethod
    def dump(cls, pattern: bytes) -> str:
        return cls._str("ref_dump", pattern, len(pattern))

    @classmethod
    def enumerate_regexes(cls, max_nodes: int, alphabet: str = "ab") -> list[str]:
        return cls._str("ref_enumerate", max_nodes, alphabet.encode()).splitlines()

    @classmethod
    def random_regexes(cls, count: int, max_nodes: int, seed: int, alphabet: str = "ab") -> list[str]:
        return cls._str("ref_random_regexes", count, max_nodes, alphabet.encode(), seed).splitlines()


class RefHeap:
    """A reference rx::Heap compiled by the reference itself."""

    def __init__(self, pattern: bytes):
        self.l = Ref.lib()
        self.p = self.l.ref_compile(pattern, len(pattern))
        if not self.p:
            raise ValueError("reference failed to compile pattern")

    def __del__(self):
        try:
            self.l.ref_free(self.p)
        except Exception:
            pass

    @staticmethod
    def _u32(w) -> np.ndarray:
        if isinstance(w, str):
            return np.array([ord(c) for c in w], np.uint32)
        return np.frombuffer(bytes(w), np.uint8).astype(np.uint32)

    def accepts(self, w) -> bool:
        a = self._u32(w)
        return bool(self.l.ref_accepts(self.p, a.ctypes.data if len(a) else None, len(a), None))

    def accepts_stats(self, w):
        a = self._u32(w)
        enq = C.c_uint64(0)
        r = self.l.ref_accepts(self.p, a.ctypes.data if len(a) else None, len(a), C.byref(enq))
        return bool(r), enq.value

    def par_accepts(self, w, workers=1, seed=0):
        a = self._u32(w)
        c, ln, mc = C.c_uint64(0), C.c_uint64(0), C.c_uint32(0)
        r = self.l.ref_par_accepts(self.p, a.ctypes.data if len(a) else None, len(a), workers, seed, C.byref(c),
                                   C.byref(ln), C.byref(mc))
        return bool(r), {"claims": c.value, "launches": ln.value, "max_claims": mc.value}

    def _set_call(self, fn, s, *extra):
        a = np.array(sorted(s), np.int32)
        out = np.zeros(4096 * 4 + len(a) + 2, np.int32)
        k = getattr(self.l, fn)(self.p, a.ctypes.data, len(a), *extra, out.ctypes.data)
        if k < 0:
            raise ValueError("reference threw")
        return set(out[:k].tolist())

    def evolve(self, s) -> set:
        return self._set_call("ref_evolve", s)

    def step_char(self, s, a: int) -> set:
        return self._set_call("ref_step_char", s, a)

    def eps_reaches_null(self, s) -> bool:
        a = np.array(sorted(s), np.int32)
        return bool(self.l.ref_eps_reaches_null(self.p, a.ctypes.data, len(a)))

    def trace(self, w) -> str:
        a = self._u32(w)
        n = self.l.ref_trace(self.p, a.ctypes.data if len(a) else None, len(a), None, 0)
        buf = C.create_string_buffer(n + 1)
        self.l.ref_trace(self.p, a.ctypes.data if len(a) else None, len(a), buf, n + 1)
        return buf.value.decode()

    def match_batch(self, text: np.ndarray, delimiter=10, stride=0, threads=None, results=True):
        """rx::lockstep_accepts over every string (decoded with decode_utf8 first)."""
        a = np.ascontiguousarray(text, np.uint8)
        prep = self.l.ref_prepare(a.ctypes.data, a.nbytes, delimiter, stride)
        if not prep:
            raise ValueError("invalid UTF-8 input")
        try:
            n = self.l.ref_prepared_count(prep)
            res = np.zeros(max(n, 1), np.uint8) if results else None
            cnt = self.l.ref_run(self.p, prep, res.ctypes.data if res is not None else None,
                                 threads or os.cpu_count() or 1)
        finally:
            self.l.ref_prepared_free(prep)
        return int(cnt), (res[:n] if res is not None else None)
