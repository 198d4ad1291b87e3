#!/usr/bin/env python3
"""Aggregate an ncu source capture of a simulator kernel by engine function (sim_engine.cuh's
`static __device__` steps), for several source-page columns at once.

usage: tools/ncu_funcs.py REPORT.ncu-rep CUBIN_SUBSTR KERNEL_SUBSTR [top]
Columns: all warp-stall samples, long-scoreboard samples, instructions executed and the L2
sectors the global accesses request (L1 misses would be a subset of these).
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
COLS = ["Warp Stall Sampling (All Samples)", "stall_long_sb", "Instructions Executed",
        "L2 Theoretical Sectors Global"]


def line_map(cub_sub, kern_sub):
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
    return line_of


def func_of():
    src = (ROOT / "paper_2207_11428_b200" / "csrc" / "sim_engine.cuh").read_text().split("\n")
    starts = []
    for i, l in enumerate(src):
        m = re.match(r"\s*static __device__.*?(\w+)\(", l)
        if m:
            starts.append((i + 1, m.group(1)))
        m = re.match(r"\s*// ---- (.*?) -", l)
        if m and any(n == "run" for _, n in starts):
            starts.append((i + 1, "run:" + m.group(1)[:24]))

    def f(line):
        name = "?"
        for s, n in starts:
            if s <= line:
                name = n
        return name
    return f


def main():
    rep, cub_sub, kern_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1] if "Address" not in rows[0] else rows[0]
    data = rows[2:] if h is rows[1] else rows[1:]
    idx = [h.index(c) for c in COLS]
    lm, fn = line_map(cub_sub, kern_sub), func_of()
    agg = collections.defaultdict(lambda: [0] * len(COLS))
    for i, r in enumerate(data):
        f, ln = lm.get(i, ("?", 0))
        key = fn(ln) if f == "sim_engine.cuh" else f
        for c, j in enumerate(idx):
            try:
                agg[key][c] += int(float(r[j] or 0))
            except ValueError:
                pass
    tot = [sum(v[c] for v in agg.values()) or 1 for c in range(len(COLS))]
    print(f"{'function':28s} {'samples%':>9s} {'long_sb%':>9s} {'instr%':>8s} {'L2sect%':>8s}   totals {tot}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k:28s} " + " ".join(f"{100 * v[c] / tot[c]:8.1f}%" for c in range(len(COLS))))


if __name__ == "__main__":
    main()
