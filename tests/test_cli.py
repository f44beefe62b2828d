"""rxgmatch — the `rxvm match` front end (reference tools/rxvm.cpp:74-115,
test_cli.cpp:42-59) on the GPU batch path: exit status contract and stdin
line filtering."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle_bind import Oracle
from paper_1108_3126_b200 import rx

CLI = Path(__file__).resolve().parent.parent / "paper_1108_3126_b200" / "rxgmatch"


def run(args, stdin=b""):
    return subprocess.run([str(CLI)] + args, input=stdin, capture_output=True)


def test_usage_and_syntax_errors_exit_2():
    assert run([]).returncode == 2
    r = run(["a("])
    assert r.returncode == 2 and b"unexpected end of pattern at position 2" in r.stderr


def expected_lines(pattern: str, data: bytes) -> bytes:
    o = Oracle(rx.compile(rx.parse(pattern)))
    lines = data.split(b"\n")
    if data.endswith(b"\n"):
        lines = lines[:-1]
    return b"".join(l + b"\n" for l in lines if o.accepts(l))


@pytest.mark.gpu
def test_exit_status_with_inputs():
    # test_cli.cpp:42-52
    assert run(["a**b", "aab"]).returncode == 0
    assert run(["a**b", "aa"]).returncode == 1
    assert run(["a**b", "aa", "ab"]).returncode == 0
    assert run(["a**", ""]).returncode == 0


@pytest.mark.gpu
def test_stdin_filtering_matches_reference_semantics():
    data = b"aab\naa\nb\nab\r\n\nabbb\nab"   # '\r' kept, empty line, final unterminated line
    for pattern in ["a**b", "(a|b)*b", "()", "a*"]:
        r = run([pattern], data)
        want = expected_lines(pattern, data)
        assert r.stdout == want, pattern
        assert r.returncode == (0 if want else 1)


@pytest.mark.gpu
def test_stdin_config_c_sample():
    text = rx.synth_input("c", 1 << 20).tobytes()
    pat = rx.synth_pattern("c")
    r = run([pat], text)
    assert r.returncode == 0
    assert r.stdout == expected_lines(pat, text)
    c = run(["--count", pat], text)
    assert int(c.stdout) == r.stdout.count(b"\n")


@pytest.mark.gpu
def test_invalid_utf8_line_is_an_error_after_earlier_matches():
    data = b"ab\nb\n\xff\nab\n"
    r = run(["(a|b)*b"], data)
    assert r.returncode == 2
    assert r.stdout == b"ab\nb\n"
    assert r.stderr == b"rxvm: invalid UTF-8 at byte 0\n"   # decode_utf8's message for that line
    # the byte offset is within the line, as decode_utf8(line) reports it
    r = run(["(a|b)*b"], b"ab\na\xc3\xa9\xe4\xb8\nb\n")
    assert r.returncode == 2 and r.stdout == b"ab\n"
    assert r.stderr == b"rxvm: invalid UTF-8 at byte 3\n"


@pytest.mark.gpu
def test_unicode_pattern():
    data = "é中\naé中\nb\n😀é\n".encode()
    r = run(["(a|é)*中"], data)
    assert r.returncode == 0 and r.stdout == "é中\naé中\n".encode()


def run_file(args, data: bytes, tmp_path):
    """stdin redirected from a regular file: the mapped-input path."""
    f = tmp_path / "in.txt"
    f.write_bytes(data)
    with open(f, "rb") as fh:
        return subprocess.run([str(CLI)] + args, stdin=fh, capture_output=True)


@pytest.mark.gpu
def test_file_stdin_matches_pipe_small(tmp_path):
    data = b"aab\naa\nb\nab\r\n\nabbb\nab"
    for pattern in ["a**b", "(a|b)*b", "()"]:
        assert run_file([pattern], data, tmp_path).stdout == expected_lines(pattern, data)
    r = run_file(["a*"], b"", tmp_path)   # empty file: no lines
    assert r.returncode == 1 and r.stdout == b""


@pytest.mark.gpu
def test_large_input_split_across_host_threads(tmp_path):
    # > 8 MiB: the line table and the output are built in pieces on several
    # host threads; the output must be the in-order filter of every line
    text = rx.synth_input("c", 24 << 20).tobytes()
    pat = rx.synth_pattern("c")
    lines = text.split(b"\n")
    if text.endswith(b"\n"):
        lines = lines[:-1]
    _, res = rx.Matcher(pat).match_batch(text, results=True)   # per-line results (parity-tested elsewhere)
    res = res[:len(lines)]
    want = b"".join(l + b"\n" for l, a in zip(lines, res) if a)
    piped = run([pat], text)
    assert piped.returncode == 0 and piped.stdout == want
    mapped = run_file([pat], text, tmp_path)
    assert mapped.returncode == 0 and mapped.stdout == want
    c = run_file(["--count", pat], text, tmp_path)
    assert int(c.stdout) == want.count(b"\n")
    # an invalid line deep in the input: everything before it, then the error
    cut = text.index(b"\n", 20 << 20) + 1
    bad = text[:cut] + b"xy\xc0z\n" + text[cut:]
    r = run_file([pat], bad, tmp_path)
    n_before = text[:cut].count(b"\n")
    assert r.returncode == 2
    assert r.stdout == b"".join(l + b"\n" for l, a in zip(lines[:n_before], res[:n_before]) if a)
    _, _, first_bad = rx.Matcher(pat).match_batch_utf8(bad)
    assert r.stderr == b"rxvm: invalid UTF-8 at byte %d\n" % (first_bad - cut)   # decode_utf8's offset in that line
