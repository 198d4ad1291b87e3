#!/usr/bin/env python3
"""Pinned host<->device copy bandwidth on this box (ceiling for bench.py's e2e leg)."""
import json
import torch

n = 164_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
for name, fn in [("h2d_1x164MB", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h_1x164MB", lambda: h.copy_(d, non_blocking=True))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn()
    b.record()
    torch.cuda.synchronize()
    out[name] = n * 10 / (a.elapsed_time(b) / 1e3) / 1e9
# chunked H2D on two streams (bench e2e pattern)
s = [torch.cuda.Stream(), torch.cuda.Stream()]
ch = 21_000_000
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for r in range(10):
    for k, o in enumerate(range(0, n, ch)):
        with torch.cuda.stream(s[k & 1]):
            d[o:o + ch].copy_(h[o:o + ch], non_blocking=True)
torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
out["h2d_chunked_2streams"] = n * 10 / (a.elapsed_time(b) / 1e3) / 1e9
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
