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
