"""In-tree build of the CUDA library (sm_100a) and the parity checkers.

`build_native()` compiles paper_2207_11428_b200/csrc/*.cu into
paper_2207_11428_b200/_lib/libmiso_b200.so with nvcc (-gencode arch=compute_100a,code=sm_100a,
--fmad=false for bit-exact FP64). `build_oracle()` runs `make -C oracle` (test infrastructure).
"""
from __future__ import annotations

import os
import re
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libmiso_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-std=c++17", "-O3", "-lineinfo",
    "--fmad=false",            # no DFMA contraction: FP64 parity with the reference's SSE2 math
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    objdir = PKG / "_build"
    objdir.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "miso_b200.h"]
    srcs = _sources()
    objs = [objdir / (s.stem + ".o") for s in srcs]

    def compile_one(pair):
        src, obj = pair
        # a TU that #includes another .cu (sim_kernel_prune.cu) depends on it too
        inc = [CSRC / m for m in re.findall(r'#include "([^"]+\.cu)"', src.read_text())]
        if not force and not _stale(obj, [src, *headers, *inc]):
            return None
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        return (src.name, r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        for res in ex.map(compile_one, zip(srcs, objs)):
            if res and verbose and res[1].strip():
                print(res[0], res[1], file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB),
               *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    tool = LIBDIR / "c1_latency"  # bench.py --config c1: the C++ caller's latency loop
    src = ROOT / "tools" / "c1_latency.cpp"
    if force or _stale(tool, [src, LIB, ROOT / "include" / "miso_b200.h"]):
        cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(src), "-o", str(tool),
               f"-L{LIBDIR}", "-lmiso_b200", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"c1_latency build failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_oracle() -> None:
    r = subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
    build_oracle()
    print(LIB)
