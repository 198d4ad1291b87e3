#!/usr/bin/env python3
"""Config-2 steps replayed from a CUDA graph (K launches alternating over 2 captured streams)
vs. the same launches issued directly. Prints us per step for each."""
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
sp2, offs2 = sp.clone(), offs.clone()
bufs = [(sp, offs, torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.float64, device=dev)),
        (sp2, offs2, torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.float64, device=dev))]
K = 50
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
out = {}


def issue(streams):
    main = torch.cuda.current_stream()
    for st in streams:
        st.wait_stream(main)
    for i in range(K):
        k = i % 2
        ctx.optimize_batch(*bufs[k], stream=streams[k].cuda_stream)
    for st in streams:
        main.wait_stream(st)


for _ in range(3):
    issue([s0, s1])
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); issue([s0, s1]); b.record(); torch.cuda.synchronize()
out["direct_us"] = a.elapsed_time(b) / K * 1e3
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.stream(cap):
    g.capture_begin()
    issue([s0, s1])
    g.capture_end()
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
out["graph_us"] = a.elapsed_time(b) / K * 1e3
ok = torch.equal(bufs[0][2], bufs[1][2])
out["outputs_equal"] = bool(ok)
print(json.dumps(out))
