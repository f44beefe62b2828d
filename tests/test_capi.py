"""The C-ABI library (CPU-side checks): loads without a GPU, exports every
symbol include/rxg.h declares, reports errors like the reference, and has no
CPU fallback for matching."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1108_3126_b200 import _lib, rx

HEADER = Path(__file__).resolve().parent.parent / "include" / "rxg.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(rxg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # and the binding declares exactly the header's functions
    assert sorted(_lib.declared_symbols()) == names


def test_version_and_strerror():
    lib = _lib.lib()
    assert b"sm_100a" in lib.rxg_version()
    for code in range(11):
        assert lib.rxg_strerror(code)


def test_parse_error_status_and_position():
    lib = _lib.lib()
    n = C.c_int32(0)
    pos = C.c_size_t(0)
    rc = lib.rxg_parse_compile(b"ab\\", 3, None, None, 0, C.byref(n), C.byref(pos))
    assert rc == _lib.RXG_EPARSE and pos.value == 3
    assert b"illegal escape at position 3" in lib.rxg_last_error()


def test_host_only_handle_refuses_matching():
    """No CPU fallback: a handle without device tables cannot match."""
    m = rx.Matcher("(a|b)*abb", device=-1)
    with pytest.raises(rx.RxgError) as ei:
        m.lockstep_accepts(b"abb")
    assert ei.value.status == _lib.RXG_ENODEV
    with pytest.raises(rx.RxgError):
        m.match_batch(b"abb\n")


def test_malformed_heap_rejected():
    h = rx.compile(rx.parse("ab"))
    bad = rx.Heap(h.nodes, [5, 7, -1])
    with pytest.raises(rx.RxgError) as ei:
        rx.Matcher(bad, device=-1)
    assert ei.value.status == _lib.RXG_EHEAP


def test_heap_from_table_equals_pattern_handle():
    h = rx.compile(rx.parse(rx.synth_pattern("c")))
    a = rx.Matcher(h, device=-1).info()
    b = rx.Matcher(rx.synth_pattern("c"), device=-1).info()
    assert a == b


def test_info_of_config_c():
    i = rx.Matcher(rx.synth_pattern("c"), device=-1).info()
    assert i["nodes"] == 64 and i["positions"] == 31 and i["words"] == 1 and i["nullable"] == 1
    assert 0 < i["line_table_bytes"] < 64 * 1024
