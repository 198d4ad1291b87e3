#!/usr/bin/env python3
"""Where does the miso simulation's slowdown beside other kernels come from? (GPU only)
miso on 1024 config-4 seeds alone, then beside (a) the predictor kernel (integer/FMA-pipe
bound, little memory traffic), (b) the search kernel (HBM streaming), (c) the pruned
best-static search (the config-4 co-runner), each co-runner re-launched on its own stream until
miso finishes. Prints miso's duration (CUDA events on its stream) per case."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402

S = 1024
ctx_m, ctx_o = miso.Context(0), miso.Context(0)
tr = miso.generate_traces_device(ctx_m, np.arange(S, dtype=np.uint64), 1000, lambda_s=10.0)
opts = miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")
s_m, s_o = torch.cuda.Stream(), torch.cuda.Stream()

n = 4 * 1024 * 1024
rng = np.random.default_rng(5)
f4 = rng.uniform(0.3, 1.0, n)
truth = torch.from_numpy(np.stack([np.ones(n), f4, f4 * 0.8], 1).reshape(-1)).cuda()
pout = torch.empty(n * 5, dtype=torch.float64, device="cuda")
m = rng.integers(1, 8, 1_000_000)
offs = np.zeros(len(m) + 1, np.uint32)
offs[1:] = np.cumsum(m)
sp = torch.from_numpy(rng.uniform(0.1, 1.0, int(offs[-1]) * 5)).cuda()
d_offs = torch.from_numpy(offs.view(np.int32)).cuda()
cand = torch.empty(len(m), dtype=torch.uint8, device="cuda")
obj = torch.empty(len(m), dtype=torch.float64, device="cuda")


def co_pred():
    with torch.cuda.stream(s_o):
        ctx_o.predict_batch(truth, 7, 1, 42, 1, 0.017, out=pout)


def co_search():
    ctx_o.optimize_batch(sp, d_offs, cand, obj, stream=s_o.cuda_stream)


def co_static():
    with torch.cuda.stream(s_o):
        miso.best_static_partition(ctx_o, tr, cluster_size=100, stream=s_o, chosen_only=True)


def run(co, reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_m)
    r = miso.simulate_batch(ctx_m, tr, opts, stream=s_m, defer=True)
    b.record(s_m)
    for _ in range(reps):
        if co:
            co()
    r()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b), 1)


out = {}
run(None, 0)
for name, co, reps in (("alone", None, 0), ("predictor", co_pred, 200), ("search", co_search, 3000),
                       ("static", co_static, 2)):
    run(co, reps)
    out[name] = [run(co, reps) for _ in range(2)]
print(json.dumps(out))
