#!/usr/bin/env python3
"""Search-kernel time vs batch size (GPU): fits t = a + b*n to expose the fixed per-launch
cost (ramp-up, tail, launch) against the streaming rate. Prints one JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2207_11428_b200 as m  # noqa: E402

ctx = m.Context(0)
dev = torch.device("cuda", 0)
rows = []
for n in [250_000, 500_000, 1_000_000, 2_000_000, 4_000_000, 8_000_000, 16_000_000]:
    sp, offs, mm = bench.gen_mixes_device(7, n, dev)
    c = torch.empty(n, dtype=torch.uint8, device=dev)
    o = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(5):
        ctx.optimize_batch(sp, offs, c, o)
    torch.cuda.synchronize()
    K = 30
    # back-to-back launches between ONE event pair (an event between launches would serialise
    # the stream and hide programmatic-dependent-launch overlap)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        ctx.optimize_batch(sp, offs, c, o)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / K * 1e3
    alg = 40 * int(offs[-1]) + 13 * n + 4
    rows.append({"n": n, "us": t, "tbs": alg / t / 1e6})
    del sp, offs, c, o
x = np.array([r["n"] for r in rows], float)
y = np.array([r["us"] for r in rows])
b, a = np.polyfit(x, y, 1)
print(json.dumps({"rows": rows, "fixed_us": a, "us_per_M": b * 1e6}))
