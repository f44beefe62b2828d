"""Builds the product library librxg.so (sm_100a) in-tree with nvcc.

The library holds the host front end (parse/compile/tables), the CUDA
kernels and the extern "C" boundary declared in include/rxg.h.
"""
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "librxg.so"
CLI = PKG / "rxgmatch"
BUILD = ROOT / "build" / "rxg"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", f"-I{ROOT / 'include'}", f"-I{CSRC}"]
SOURCES = ["frontend.cpp", "program.cpp", "tables.cpp", "lines_tma_table.cpp", "synth.cpp",
           "kernels_batch.cu", "kernels_lines_tma.cu", "kernels_single.cu", "kernels_pernode.cu", "kernels_chunked.cu", "kernels_chunk_tma.cu", "kernels_many.cu", "kernels_utf8.cu", "kernels_fixed_tma.cu", "kernels_bits_tma.cu",
           "capi.cu", "multi.cu", "options.cpp", "setops.cpp"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or Path(c).exists()):
            return c
    raise RuntimeError("nvcc not found")


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rxg.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps if d.exists())


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for name in SOURCES:
        src = CSRC / name
        obj = BUILD / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            flags = list(COMMON)
            if name.endswith(".cu"):
                flags += ARCH + ["-Xptxas", "-v"] if verbose else ARCH
            cmd = [nvcc()] + flags + ["-c", str(src), "-o", str(obj)]
            jobs.append((name, cmd))
    procs = [(n, c, subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)) for n, c in jobs]
    for n, c, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {n}")
        if verbose and out:
            sys.stderr.write(out.decode())
    if force or not OUT.exists() or any(o.stat().st_mtime > OUT.stat().st_mtime for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", str(OUT)] + [str(o) for o in objs] + ["-ldl"]
        subprocess.run(cmd, check=True)
    # the `rxvm match` front end on the batch path (links librxg.so)
    cli_src = CSRC / "tools" / "rxgmatch.cpp"
    if force or not CLI.exists() or cli_src.stat().st_mtime > CLI.stat().st_mtime or OUT.stat().st_mtime > CLI.stat().st_mtime:
        subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(cli_src), f"-L{PKG}", "-lrxg",
                        "-Wl,-rpath,$ORIGIN", "-pthread", "-o", str(CLI)], check=True)
    # measurement tool (not product): the INT32 peak of SURVEY.md §8(d)'s roofline
    peak_src = ROOT / "tools" / "peaks" / "int32_peak.cu"
    peak_so = ROOT / "tools" / "peaks" / "libint32peak.so"
    if force or not peak_so.exists() or peak_src.stat().st_mtime > peak_so.stat().st_mtime:
        subprocess.run([nvcc(), "-O3", "-lineinfo"] + ARCH + ["-Xcompiler", "-fPIC", "-shared", "-o", str(peak_so),
                        str(peak_src)], check=True)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
