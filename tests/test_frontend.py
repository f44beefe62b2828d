"""Front end parity (CPU): parse / compile / print / dump / check_knode of the
product library against the reference's own golden vectors
(proj/tests/test_regex.cpp, test_heap.cpp, acceptance_main.cpp:34-47) and, when
oracle/_ref is built, against the reference library on every small regex."""
import json
from pathlib import Path

import pytest

from oracle_bind import Ref
from paper_1108_3126_b200 import rx

GOLD = json.loads((Path(__file__).parent / "golden" / "frontend.json").read_text())


def test_worked_example_heap_layout():
    # test_heap.cpp:13-32 / acceptance criterion 1
    h = rx.compile(rx.parse("a**b"))
    assert h.size() == 5
    assert rx.dump(h) == ("p0\tseq p1 p2\tnull\n"
                          "p1\tstar p3\tp2\n"
                          "p2\tchar b\tnull\n"
                          "p3\tstar p4\tp1\n"
                          "p4\tchar a\tp3\n")
    assert [n.kind for n in h.nodes] == [rx.NODE_SEQ, rx.NODE_STAR, rx.NODE_CHR, rx.NODE_STAR, rx.NODE_CHR]
    assert h.knodes == [-1, 2, -1, 1, 3]


def test_leaf_cases():
    # test_heap.cpp:34-45
    h = rx.compile(rx.parse("()"))
    assert h.size() == 1 and h.node(0).kind == rx.NODE_EPS and h.knode(0) == -1
    g = rx.compile(rx.parse("a|b"))
    assert g.size() == 3 and g.node(0).kind == rx.NODE_ALT and g.knode(1) == -1 and g.knode(2) == -1


def test_precedence_and_associativity():
    # test_regex.cpp:14-35: abc is left-deep, a|b|c is left-deep, star binds tightest
    h = rx.compile(rx.parse("abc"))
    assert h.node(0).kind == rx.NODE_SEQ and h.node(h.node(0).left).kind == rx.NODE_SEQ
    h = rx.compile(rx.parse("a|b|c"))
    assert h.node(0).kind == rx.NODE_ALT and h.node(h.node(0).left).kind == rx.NODE_ALT
    h = rx.compile(rx.parse("a|bc*"))
    assert h.node(0).kind == rx.NODE_ALT and h.node(h.node(0).right).kind == rx.NODE_SEQ
    assert rx.dump(rx.compile(rx.parse("(a**)b"))) == rx.dump(rx.compile(rx.parse("a**b")))


def test_escapes_and_unicode():
    assert rx.compile(rx.parse("\\*")).node(0).sym == ord("*")
    assert rx.compile(rx.parse("\\\\")).node(0).sym == ord("\\")
    assert rx.compile(rx.parse("\\a")).node(0).sym == ord("a")
    h = rx.compile(rx.parse("α*"))
    assert h.node(0).kind == rx.NODE_STAR and h.node(1).sym == 0x3B1


@pytest.mark.parametrize("pattern", sorted(GOLD["dump"]))
def test_dump_goldens(pattern):
    assert rx.dump(rx.compile(rx.parse(pattern))) == GOLD["dump"][pattern]
    assert rx.print_regex(rx.parse(pattern)) == GOLD["print"][pattern]


@pytest.mark.parametrize("pattern", sorted(GOLD["errors"]))
def test_parse_errors_carry_positions(pattern):
    # test_regex.cpp:37-62
    want = GOLD["errors"][pattern]
    if want is None:
        rx.parse(pattern)
        return
    with pytest.raises(rx.ParseError) as ei:
        rx.parse(pattern)
    assert ei.value.pos == want[0]
    assert str(ei.value) == want[1]


def test_print_canonical_forms():
    # test_regex.cpp:64-73
    assert rx.print_regex(rx.parse("()")) == "()"
    assert rx.print_regex(rx.parse("a|b")) == "a|b"
    assert rx.print_regex(rx.parse("a**b")) == "a**b"
    assert rx.print_regex(rx.parse("a(bc)")) == "a(bc)"
    assert rx.print_regex(rx.parse("a|(b|c)")) == "a|(b|c)"
    assert rx.print_regex(rx.parse("(a|b)*")) == "(a|b)*"
    assert rx.print_regex(rx.parse("()*")) == "()*"
    assert rx.print_regex(rx.parse("\\*")) == "\\*"


def test_check_knode_rewires():
    # test_heap.cpp:65-80
    h = rx.compile(rx.parse("a**b"))
    assert rx.check_knode(h)
    for idx, val in [(4, 1), (0, 2), (1, -1)]:
        k = list(h.knodes)
        k[idx] = val
        assert not rx.check_knode(rx.Heap(h.nodes, k))


def test_dump_roundtrip_and_errors():
    # test_heap.cpp:110-122
    for p in GOLD["dump"]:
        if " " in p:   # the dump format cannot carry a space literal (heap.cpp:216-222, same in the reference)
            continue
        h = rx.compile(rx.parse(p))
        assert rx.dump(rx.parse_dump(rx.dump(h))) == rx.dump(h)
    for bad in ["p0\tbogus\tnull\n", "p0\tstar p9\tnull\n", "", "p1\teps\tnull\n"]:
        with pytest.raises(RuntimeError):
            rx.parse_dump(bad)


def test_utf8_errors():
    with pytest.raises(rx.Utf8Error):
        rx.parse(b"a\xff")
    with pytest.raises(rx.Utf8Error):
        rx.parse(b"\xc0\x80")   # overlong


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_compile_parity_exhaustive_against_reference():
    """Every regex <= 6 AST nodes over {a,b}: identical heap tables, dumps, prints."""
    pats = Ref.enumerate_regexes(6, "ab")
    assert len(pats) > 1000
    for p in pats:
        b = p.encode()
        nodes, kn = Ref.parse_compile(b)
        h = rx.compile(rx.parse(b))
        assert [(n.kind, n.sym, n.left, n.right) for n in h.nodes] == nodes, p
        assert h.knodes == kn, p
        assert rx.check_knode(h)


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_print_roundtrip_random_against_reference():
    for p in Ref.random_regexes(200, 14, seed=7):
        assert rx.print_regex(rx.parse(p)) == Ref.print_regex(p.encode())
        assert rx.dump(rx.compile(rx.parse(rx.print_regex(rx.parse(p))))) == rx.dump(rx.compile(rx.parse(p)))
