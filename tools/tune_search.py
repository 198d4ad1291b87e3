#!/usr/bin/env python3
"""Time the partition-search kernel under each MISO_B200_PIPE_CFG (tuning helper, GPU only).

Prints one JSON line per configuration: kernel ms (CUDA events, mean of 50 launches after 10
warm-ups) on the bench's 1M-instance config-2 batch, and whether the decisions match cfg 0.
"""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, ".")
import bench, paper_2207_11428_b200 as m
s, f, mm = bench.gen_mixes(1000, 1_000_000)
ctx = m.Context(0)
ds = torch.from_numpy(s).cuda(); df = torch.from_numpy(f.view(np.int32)).cuda()
c = torch.empty(len(mm), dtype=torch.uint8, device="cuda"); o = torch.empty(len(mm), dtype=torch.float64, device="cuda")
for _ in range(10): ctx.optimize_batch(ds, df, c, o)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ctx.optimize_batch(ds, df, c, o); b.record(); ts.append((a, b))
torch.cuda.synchronize()
ms = sum(a.elapsed_time(b) for a, b in ts) / len(ts)
h = (int(c.cpu().numpy().astype(np.int64).sum()), float(o.sum().item()))
print(json.dumps({"cfg": os.environ.get("MISO_B200_PIPE_CFG", "0"), "ms": ms, "hash": h,
                  "gbs": bench.algorithmic_bytes(mm) / ms / 1e6}))
'''

for cfg in sys.argv[1:] or ["0", "1", "2", "3", "4"]:
    env = dict(os.environ, MISO_B200_PIPE_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
