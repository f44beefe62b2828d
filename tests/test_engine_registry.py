"""The GPU engine for the reference's engine registry (include/rxg_engine.hpp,
SURVEY §8(f) item 2): the adapter compiles against any rx::Heap-shaped type,
and on the GPU agrees with all seven reference engines over the reference's
own crosscheck suite (oracle/_ref/crosscheck_gpu links the unmodified
reference library)."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
XCHK = ROOT / "oracle" / "_ref" / "crosscheck_gpu"


@pytest.fixture(scope="module")
def engine_bin(tmp_path_factory):
    out = tmp_path_factory.mktemp("engine") / "engine_test"
    lib = ROOT / "paper_1108_3126_b200"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "engine_test.cpp"),
                    f"-L{lib}", "-lrxg", f"-Wl,-rpath,{lib}", "-o", str(out)], check=True)
    return out


def test_adapter_compiles_and_raises_without_device(engine_bin):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    r = subprocess.run([str(engine_bin), "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_adapter_on_gpu(engine_bin):
    r = subprocess.run([str(engine_bin), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def _xchk(*args):
    if not XCHK.exists():
        pytest.skip("oracle/_ref/crosscheck_gpu not built (needs the reference sources at build time)")
    r = subprocess.run([str(XCHK), *args], capture_output=True, text=True, timeout=900)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    return r.returncode, out


@pytest.mark.gpu
def test_seven_engines_plus_gpu_agree_enumerated_suite():
    rc, out = _xchk("--max-nodes", "6", "--max-len", "5", "--random", "2000", "--seed", "7")
    assert out["regexes"] == 1674 and out["strings"] == 63
    assert rc == 0 and out["gpu_disagreements"] == 0 and out["reference_disagreements"] == 0, out
    assert 0 < out["gpu_matches"] < out["cases"]


@pytest.mark.gpu
def test_seven_engines_plus_gpu_agree_unicode_alphabet():
    rc, out = _xchk("--max-nodes", "4", "--max-len", "4", "--random", "1000", "--alphabet", "aé中😀")
    assert rc == 0 and out["gpu_disagreements"] == 0, out
