#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into JSON.
usage: tools/launch_summary.py launches.csv out.json "command that produced it"
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
gi = h.index("Grid Size") if "Grid Size" in h else None
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > mi and r[mi] == "gpu__time_duration.sum":
        key = r[ki][:100] + (f" grid{r[gi]}" if gi is not None else "")
        agg[key].append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
out = {"command": sys.argv[3] if len(sys.argv) > 3 else "", "note":
       "ncu per-launch device times (cold-cache, serialised): compare shares, not absolutes",
       "kernels": [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v),
                    "min_us": min(v), "share": sum(v) / tot} for k, v in agg.items()]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
