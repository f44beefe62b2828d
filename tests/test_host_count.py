"""Host-side delimiter count used to place per-string results of host-buffer
calls (csrc/heap_internal.hpp count_byte): exact against a byte loop."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_count_byte_exact(tmp_path):
    out = tmp_path / "count_byte_test"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", f"-I{ROOT / 'paper_1108_3126_b200' / 'csrc'}",
                    "-I/usr/local/cuda/include", str(ROOT / "tests" / "cpp" / "count_byte_test.cpp"), "-pthread",
                    "-o", str(out)], check=True)
    r = subprocess.run([str(out)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr


def test_count_strings_matches_getline_split():
    """rxg_count_strings (host, threaded above 8 MiB): delimiters plus an
    unterminated last string; fixed stride: len / stride."""
    import numpy as np

    from paper_1108_3126_b200 import rx

    rng = np.random.default_rng(5)
    for n in (0, 1, 17, 4096, (9 << 20) + 3):
        a = rng.integers(0, 12, size=n, dtype=np.uint8)
        for d in (0, 10, 11):
            want = int(np.count_nonzero(a == d)) + (1 if n and a[-1] != d else 0)
            assert rx.count_strings(a, d) == want, (n, d)
    assert rx.count_strings(np.zeros(96, np.uint8), -1, 32) == 3
    assert rx.count_strings(b"ab\ncd", 10) == 2 and rx.count_strings(b"ab\n", 10) == 1 and rx.count_strings(b"", 10) == 0
