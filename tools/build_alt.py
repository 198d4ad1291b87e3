#!/usr/bin/env python3
"""Link an alternate copy of the library for same-box A/B runs: the listed TUs recompiled with
extra nvcc flags, every other object taken from the in-tree build.
usage: tools/build_alt.py NAME "EXTRA FLAGS" tu1.cu [tu2.cu ...]  ->  _lib/alt_NAME.so"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2207_11428_b200 import build as B  # noqa: E402

name, extra, tus = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build_native()
objdir = B.PKG / "_build"
alt = objdir / f"alt_{name}"
alt.mkdir(exist_ok=True)
objs = []
for src in B._sources():
    if src.name in tus:
        o = alt / (src.stem + ".o")
        subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *extra, "-c", str(src), "-o", str(o)], check=True)
        objs.append(o)
    else:
        objs.append(objdir / (src.stem + ".o"))
out = B.LIBDIR / f"alt_{name}.so"
subprocess.run([B._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out),
                *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"], check=True)
print(out)
