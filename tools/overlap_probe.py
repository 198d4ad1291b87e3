#!/usr/bin/env python3
"""Config-2 steps (1M mixes each) back to back: one stream (PDL between launches) vs steps
alternating over S streams with per-stream output buffers, so one step's tail overlaps the
next step's ramp. Prints one JSON line (us per step for each variant)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2207_11428_b200 as m  # noqa: E402

ctx = m.Context(0)
dev = torch.device("cuda", 0)
n = 1_000_000
sp, offs, mm = bench.gen_mixes_device(7, n, dev)
alg = 40 * int(offs[-1]) + 13 * n + 4
out = {}
K = 60
for S in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(S)]
    bufs = [(torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.float64, device=dev))
            for _ in range(S)]
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        a.record(main)
        for s in streams:
            s.wait_stream(main)
        for i in range(K):
            s = streams[i % S]
            c, o = bufs[i % S]
            ctx.optimize_batch(sp, offs, c, o, stream=s.cuda_stream)
        for s in streams:
            main.wait_stream(s)
        b.record(main)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / K * 1e3
    out[f"streams_{S}"] = {"us_per_step": t, "GBps": alg / t / 1e3}
print(json.dumps(out))
