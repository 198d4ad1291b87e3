#!/usr/bin/env python3
"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: tools/ncu_lines.py REPORT.ncu-rep CUBIN_SUBSTR KERNEL_SUBSTR [top] [column]
(column: the source page's sample column, default "Warp Stall Sampling (All Samples)"; e.g.
stall_no_inst, stall_long_sb, stall_wait)
Uses `ncu --page source --print-source sass` (samples per SASS instruction) and
`nvdisasm -g` of the matching cubin extracted from the built library (line table).
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2207_11428_b200" / "_lib" / "libmiso_b200.so"


def main():
    rep, cub_sub, kern_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    col = sys.argv[5] if len(sys.argv) > 5 else "Warp Stall Sampling (All Samples)"
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1]
    data = rows[2:]
    iall = h.index(col)
    iex = h.index("Instructions Executed")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=d, capture_output=True)
        cub = [p for p in Path(d).glob("*.cubin") if cub_sub in p.name][0]
        dis = subprocess.run(["nvdisasm", "-c", "-g", str(cub)], capture_output=True, text=True).stdout.split("\n")
    secs = [i for i, l in enumerate(dis) if l.startswith("//----") and ".text." in l and kern_sub in l]
    start = secs[0]
    end = next((i for i, l in enumerate(dis) if i > start and l.startswith("//----") and ".text." in l), len(dis))
    line_of, cur = {}, None
    for l in dis[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            line_of[int(m.group(1), 16) // 16] = cur
    agg, aex = collections.Counter(), collections.Counter()
    for i, r in enumerate(data):
        k = line_of.get(i, ("?", 0))
        agg[k] += int(r[iall] or 0)
        aex[k] += int(r[iex] or 0)
    tot = sum(agg.values()) or 1
    src = {}
    for f in (ROOT / "paper_2207_11428_b200" / "csrc").glob("*"):
        src[f.name] = f.read_text().split("\n")
    print(f"samples {tot}, instructions {sum(aex.values())}")
    for k, v in agg.most_common(top):
        txt = src[k[0]][k[1] - 1].strip()[:72] if k[0] in src else ""
        print(f"{v:8d} {100 * v / tot:5.1f}% ex={aex[k]:>11d} {k[0]}:{k[1]}  {txt}")


if __name__ == "__main__":
    main()
