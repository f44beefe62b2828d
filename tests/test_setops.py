"""Host side of the reference's tree and set-level API in the C ABI
(csrc/setops.cpp): rxg_parse_ast / rxg_print_ast / rxg_compile_ast against
rxg_parse_compile and the reference printer, and rxg_evolve / rxg_step_char /
rxg_eps_reaches_null against the C oracle's restatement of lockstep.cpp
(itself pinned to the reference). No GPU needed."""
import ctypes as C

import numpy as np
import pytest

from oracle_bind import Oracle, Ref
from paper_1108_3126_b200 import _lib as L
from paper_1108_3126_b200 import rx


class Ast(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("pad", C.c_uint8 * 3), ("sym", C.c_uint32), ("left", C.c_int32),
                ("right", C.c_int32)]


def parse_ast(text: bytes):
    n, root, pos = C.c_int32(0), C.c_int32(0), C.c_size_t(0)
    assert L.lib().rxg_parse_ast(text, len(text), None, 0, C.byref(n), C.byref(root), C.byref(pos)) == 0
    arr = (Ast * n.value)()
    assert L.lib().rxg_parse_ast(text, len(text), arr, n.value, C.byref(n), C.byref(root), C.byref(pos)) == 0
    return arr, n.value, root.value


def compile_ast(arr, n, root):
    nodes = (L.rxg_node * n)()
    kn = (C.c_int32 * n)()
    got = C.c_int32(0)
    rc = L.lib().rxg_compile_ast(arr, n, root, nodes, kn, n, C.byref(got))
    return rc, nodes, kn, got.value


def _patterns():
    pats = ["a**b", "()", "a|b", "(a|b)*abb", "(a|())*b", "((ab)*|c)*d", "é(λ|😀)*"]
    if Ref.available():
        pats += Ref.random_regexes(150, 12, 3, "abc")
    return pats


def test_tree_parse_print_compile_equal_the_text_path():
    for p in _patterns():
        arr, n, root = parse_ast(p.encode())
        assert root == n - 1   # children precede parents
        ln = C.c_size_t(0)
        assert L.lib().rxg_print_ast(arr, n, root, None, 0, C.byref(ln)) == 0
        buf = C.create_string_buffer(ln.value + 1)
        L.lib().rxg_print_ast(arr, n, root, buf, ln.value + 1, C.byref(ln))
        assert buf.value.decode() == rx.print_regex(rx.parse(p)), p
        rc, nodes, kn, got = compile_ast(arr, n, root)
        h = rx.compile(rx.parse(p))
        assert rc == 0 and got == h.size()
        assert [(x.kind, x.sym, x.left, x.right) for x in nodes] == [(x.kind, x.sym, x.left, x.right) for x in h.nodes]
        assert list(kn) == h.knodes


def test_compile_ast_rejects_non_trees():
    arr = (Ast * 3)()
    arr[0] = Ast(1, (0, 0, 0), ord("a"), -1, -1)
    arr[1] = Ast(3, (0, 0, 0), 0, 0, 0)         # seq(a, a): node 0 used twice (shared)
    assert compile_ast(arr, 2, 1)[0] == L.RXG_EINVAL
    arr[1] = Ast(2, (0, 0, 0), 0, 2, -1)        # star whose child comes after it
    assert compile_ast(arr, 3, 1)[0] == L.RXG_EINVAL
    arr[1] = Ast(9, (0, 0, 0), 0, -1, -1)       # unknown kind
    assert compile_ast(arr, 2, 1)[0] == L.RXG_EINVAL


def _c(h):
    n = h.size()
    nodes = (L.rxg_node * n)()
    for i, x in enumerate(h.nodes):
        nodes[i].kind, nodes[i].sym, nodes[i].left, nodes[i].right = x.kind, x.sym, x.left, x.right
    return nodes, (C.c_int32 * n)(*h.knodes), n


def test_set_functions_equal_the_oracle():
    rng = np.random.default_rng(5)
    lib = L.lib()
    for p in _patterns()[:80]:
        h = rx.compile(rx.parse(p))
        o = Oracle(h)
        nodes, kn, n = _c(h)
        for _ in range(6):
            s = sorted({int(x) for x in rng.integers(-1, n, int(rng.integers(0, 4)))})
            arr = (C.c_int32 * max(len(s), 1))(*s)
            out = (C.c_int32 * (n + 1))()
            k = C.c_int32(0)
            enq = C.c_uint64(0)
            assert lib.rxg_evolve(nodes, kn, n, arr, len(s), out, C.byref(k), C.byref(enq)) == 0
            ev = set(out[: k.value])
            assert ev == o.evolve(set(s)), (p, s)
            r = C.c_int32(0)
            assert lib.rxg_eps_reaches_null(nodes, kn, n, arr, len(s), C.byref(r)) == 0
            assert bool(r.value) == o.eps_reaches_null(set(s)), (p, s)
            evs = sorted(ev)
            earr = (C.c_int32 * max(len(evs), 1))(*evs)
            out2 = (C.c_int32 * (len(evs) + 1))()
            for a in (ord("a"), ord("b")):
                assert lib.rxg_step_char(nodes, kn, n, earr, len(evs), a, out2, C.byref(k)) == 0
                assert set(out2[: k.value]) == o.step_char(ev, a), (p, evs, a)
        # step_char on an unevolved member is the reference's invalid_argument
        non_chr = [i for i in range(n) if h.nodes[i].kind != rx.NODE_CHR]
        if non_chr:
            arr = (C.c_int32 * 1)(non_chr[0])
            out2 = (C.c_int32 * 2)()
            assert lib.rxg_step_char(nodes, kn, n, arr, 1, ord("a"), out2, C.byref(k)) == L.RXG_EINVAL
            assert b"unevolved member" in lib.rxg_last_error()


def test_evolve_worked_example_and_enqueued():
    """test_lockstep.cpp:15-23 on a**b: evolve({p0}) = {p2, p4} in discovery order p4, p2; 5 addresses enqueued."""
    h = rx.compile(rx.parse("a**b"))
    nodes, kn, n = _c(h)
    arr = (C.c_int32 * 1)(0)
    out = (C.c_int32 * (n + 1))()
    k, enq = C.c_int32(0), C.c_uint64(0)
    assert L.lib().rxg_evolve(nodes, kn, n, arr, 1, out, C.byref(k), C.byref(enq)) == 0
    assert set(out[: k.value]) == {2, 4} and enq.value == 5
