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
