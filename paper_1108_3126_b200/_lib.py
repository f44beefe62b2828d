"""ctypes binding of the product library librxg.so (include/rxg.h).

The library is built in-tree by ``paper_1108_3126_b200/build.py`` (or
``__graft_entry__.build()``). There is no fallback: importing the binding
without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# RXG_LIB: load another build (A/B timing of two builds in one process tree; tools only)
LIB_PATH = Path(os.environ["RXG_LIB"]) if os.environ.get("RXG_LIB") else Path(__file__).resolve().parent / "librxg.so"

RXG_OK = 0
RXG_EINVAL = 1
RXG_EPARSE = 2
RXG_EUTF8 = 3
RXG_EUNSUPPORTED = 4
RXG_ECUDA = 5
RXG_ENOMEM = 6
RXG_ETOOBIG = 7
RXG_ENCCL = 8
RXG_EHEAP = 9
RXG_ENODEV = 10

ENGINES = {"auto": 0, "dfa_seq": 1, "pernode": 2, "rounds": 3, "chunked": 4}
BATCH_ENGINES = {"auto": 0, "dfa": 1, "bitset": 2}


class rxg_node(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("pad", C.c_uint8 * 3), ("sym", C.c_uint32),
                ("left", C.c_int32), ("right", C.c_int32)]


class rxg_heap_info(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("positions", C.c_int32), ("words", C.c_int32),
                ("classes", C.c_int32), ("dfa_states", C.c_int32), ("byte_symbols", C.c_int32),
                ("device", C.c_int32), ("nullable", C.c_int32),
                ("line_table_bytes", C.c_uint32), ("plain_table_bytes", C.c_uint32), ("dfa_sets", C.c_int32),
                ("line_tma_layout", C.c_int32), ("line_col_bytes", C.c_int32), ("chunk_lookback", C.c_int32)]


class rxg_match_stats(C.Structure):
    _fields_ = [("enqueued", C.c_uint64), ("claims", C.c_uint64), ("launches", C.c_uint64),
                ("macro_steps", C.c_uint64), ("max_claims_per_node_step", C.c_uint32),
                ("schedule", C.POINTER(C.c_uint32)), ("schedule_len", C.c_uint64)]


class rxg_one_opts(C.Structure):
    _fields_ = [("checkpoint_every", C.c_uint32), ("d_checkpoints", C.c_void_p), ("d_stats", C.c_void_p),
                ("d_trace", C.c_void_p), ("chunk", C.c_uint32), ("lookback", C.c_uint32), ("d_repairs", C.c_void_p),
                ("flags", C.c_uint32), ("entry_state", C.c_uint32), ("d_exit_state", C.c_void_p),
                ("d_enqueued", C.c_void_p), ("d_schedule", C.c_void_p)]


# name -> (restype, argtypes). Every symbol declared in include/rxg.h.
_P = C.c_void_p
_SIG = {
    "rxg_strerror": (C.c_char_p, [C.c_int]),
    "rxg_last_error": (C.c_char_p, []),
    "rxg_version": (C.c_char_p, []),
    "rxg_parse_compile": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(rxg_node), C.POINTER(C.c_int32),
                                    C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_size_t)]),
    "rxg_print": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rxg_dump": (C.c_int, [C.POINTER(rxg_node), C.POINTER(C.c_int32), C.c_int32, C.c_char_p, C.c_size_t,
                           C.POINTER(C.c_size_t)]),
    "rxg_parse_dump": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(rxg_node), C.POINTER(C.c_int32), C.c_int32,
                                 C.POINTER(C.c_int32)]),
    "rxg_check_knode": (C.c_int, [C.POINTER(rxg_node), C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]),
    "rxg_heap_create": (C.c_int, [C.POINTER(rxg_node), C.POINTER(C.c_int32), C.c_int32, C.c_int, C.POINTER(_P)]),
    "rxg_heap_create_pattern": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(_P)]),
    "rxg_heap_destroy": (None, [_P]),
    "rxg_heap_info_get": (C.c_int, [_P, C.POINTER(rxg_heap_info)]),
    "rxg_heap_tune": (C.c_int, [_P, _P, C.c_uint64, C.c_int32]),
    "rxg_heap_tables": (C.c_int, [_P, _P, _P, _P]),
    "rxg_host_walk": (C.c_int, [_P, _P, C.c_uint64, _P, C.POINTER(C.c_int32)]),
    "rxg_host_emulate_batch": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.c_uint32,
                                         C.POINTER(C.c_uint64), _P]),
    "rxg_host_emulate_lines_tma": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "rxg_host_emulate_chunk_tma": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "rxg_match_one": (C.c_int, [_P, _P, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]),
    "rxg_match_one_ex": (C.c_int, [_P, _P, C.c_uint64, C.c_int, _P, C.POINTER(rxg_one_opts), _P]),
    "rxg_match_one_device": (C.c_int, [_P, _P, C.c_uint64, C.c_int, _P, _P]),
    "rxg_match_batch": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, _P, _P, _P]),
    "rxg_match_batch_ex": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.c_int, _P, _P, _P]),
    "rxg_match_batch_host": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64), _P]),
    "rxg_match_batch_host_ex": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64), _P,
                                          C.POINTER(C.c_uint64)]),
    "rxg_utf8_check": (C.c_int, [C.c_int, _P, C.c_uint64, C.c_int32, C.c_uint32, _P, _P]),
    "rxg_utf8_check_host": (C.c_int, [C.c_int, _P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "rxg_match_batch_multi": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_char_p, C.c_size_t, _P, C.c_uint64,
                                        C.c_int32, C.c_uint32, C.POINTER(C.c_uint64), _P]),
    "rxg_comm_unique_id": (C.c_int, [_P, C.c_size_t]),
    "rxg_comm_init_rank": (C.c_int, [_P, C.c_size_t, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "rxg_comm_destroy": (None, [_P]),
    "rxg_match_batch_allreduce": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int32, C.c_uint32, _P, _P, _P]),
    "rxg_multi_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_char_p, C.c_size_t, C.POINTER(_P)]),
    "rxg_multi_destroy": (None, [_P]),
    "rxg_multi_info": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "rxg_multi_tune": (C.c_int, [_P, _P, C.c_uint64, C.c_int32]),
    "rxg_multi_match_batch": (C.c_int, [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64), _P]),
    "rxg_match_many": (C.c_int, [C.c_int, C.c_char_p, C.c_int32, _P, C.c_uint64, C.c_int32, C.c_uint32, _P,
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
    "rxg_match_one_multi": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_char_p, C.c_size_t, _P, C.c_uint64,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "rxg_shard_bounds": (C.c_int, [_P, C.c_uint64, C.c_int32, C.c_uint32, C.c_int, C.POINTER(C.c_uint64)]),
    "rxg_count_strings": (C.c_int, [_P, C.c_uint64, C.c_int32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "rxg_last_launch_count": (C.c_int, []),
    "rxg_set_option": (C.c_int, [C.c_char_p, C.c_char_p]),
    "rxg_match_one_stats": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(rxg_match_stats)]),
    "rxg_par_task": (C.c_int, [_P, _P, C.c_int32, C.c_uint32]),
    "rxg_par_run_rounds": (C.c_int, [_P, _P, C.c_uint32, C.POINTER(C.c_uint64)]),
    "rxg_parse_ast": (C.c_int, [C.c_char_p, C.c_size_t, _P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_size_t)]),
    "rxg_print_ast": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rxg_compile_ast": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, C.c_int32, C.POINTER(C.c_int32)]),
    "rxg_evolve": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, _P, C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]),
    "rxg_eps_reaches_null": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.POINTER(C.c_int32)]),
    "rxg_step_char": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, C.c_uint32, _P, C.POINTER(C.c_int32)]),
    "rxg_synth_pattern": (C.c_int, [C.c_char, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rxg_synth_input_size": (C.c_uint64, [C.c_char]),
    "rxg_synth_input": (C.c_int, [C.c_char, C.c_uint64, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
}

OPTION_NAMES = ("RXG_NO_TMA", "RXG_NO_LT", "RXG_NO_FIXED_TMA", "RXG_LINE_CHUNK", "RXG_LT_SHAPE", "RXG_CHUNK_SHAPE",
                "RXG_TMA_PROMO", "RXG_SKIP_SHARE", "RXG_COL_BYTES", "RXG_NO_ROW_PAIRS", "RXG_FORCE_CLASS",
                "RXG_NO_RANGE_LAYOUT", "RXG_NO_PACKED", "RXG_CHUNK_FN", "RXG_COPY_THREADS", "RXG_NO_BITS_TMA")

_lib = None


def lib() -> C.CDLL:
    """The loaded product library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIG.items():
            if os.environ.get("RXG_LIB") and not hasattr(l, name):
                continue   # an older build under A/B: symbols added since are absent
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
        # dev/A-B convenience of the Python host only (the library reads no
        # environment): RXG_* tuning switches set in the environment of a tool
        for k in OPTION_NAMES:
            if os.environ.get(k) and hasattr(l, "rxg_set_option"):
                l.rxg_set_option(k.encode(), os.environ[k].encode())
    return _lib


def declared_symbols() -> list[str]:
    return list(_SIG)
