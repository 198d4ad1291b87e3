#!/usr/bin/env python3
"""Small invocations of every kernel, for compute-sanitizer (memcheck / racecheck / synccheck).
GPU only. Exercises: the search pipe kernel (aligned) and tile kernel (misaligned base), the
predictor, the fused decide kernel, the single-roster latency kernel, the simulator (every
policy, clones, optsta), and the device trace generator. Round 2: queued search batches, the
server's search-only requests, a caller-fitted small-slice model with a small event budget,
and the pruned best-static kernel."""
import sys

import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2207_11428_b200 as m  # noqa: E402
from oracle_lib import Oracle  # noqa: E402

ctx = m.Context(0)
orc = Oracle()
s, f = orc.gen_mixes(5, 5000)
cand, obj = ctx.optimize_batch(torch.from_numpy(s).cuda(), torch.from_numpy(f.astype(np.int32)).cuda())
buf = torch.zeros(len(s) + 1, dtype=torch.float64, device="cuda")
buf[1:] = torch.from_numpy(s).cuda()
ctx.optimize_batch(buf[1:], torch.from_numpy(f.astype(np.int32)).cuda())      # misaligned -> tile kernel
ctx.optimize_batch(s, f)                                                        # host pipeline
d_s, d_f = torch.from_numpy(s).cuda(), torch.from_numpy(f.astype(np.int32)).cuda()
q = [(d_s, d_f, torch.empty(5000, dtype=torch.uint8, device="cuda"),
      torch.empty(5000, dtype=torch.float64, device="cuda")) for _ in range(35)]
ctx.optimize_batches(q)                                                         # queued: 2 launches
ctx.optimize_partition([("a", [0.2, 0.4, 0.6, 0.8, 1.0]), ("b", [0.3, 0.5, 0.7, 0.9, 1.0])])  # search-only request
t, _ = orc.gen_profiles(3, 700)
ctx.predict_batch(t, 7, 1, 42, 1, 0.017)
mem = np.full(700, 5, np.uint8); qos = np.full(700, -1, np.int8)
offs = np.arange(0, 701, 7).astype(np.uint32)
ctx.decide_batch(t, mem, qos, offs, np.arange(1, 101, dtype=np.uint64), 7, 1, 0.017)
tr = m.generate_trace(7, 3)
jobs3 = [(f"j{i}", (tr.speeds5[i, 4], tr.speeds5[i, 3], tr.speeds5[i, 2]), int(tr.mem_gb[i]), None) for i in range(3)]
for nonce in range(1, 9):  # resident server: consecutive nonces exercise the draw-ahead ring
    ctx.decide(jobs3, nonce, 7)
    time.sleep(0.002 if nonce % 3 == 0 else 0.0)
ctx.decide(jobs3, 1000, 7)
ctx.decide_server(0)       # one launch per call
ctx.decide(jobs3, 1, 7)
ctx.optimize_partition([("a", [0.2, 0.4, 0.6, 0.8, 1.0])])  # search-only, one launch
ctx.decide_server(2000)
traces = m.generate_traces(range(6), 60, lambda_s=20.0)
traces[2].instances = np.array([1] * 10 + [3] + [1] * 49, np.uint8)
for pol in ("nopart", "oracle", "miso"):
    m.simulate_batch(ctx, list(traces), m.SimOptions(policy=pol, cluster_size=4, predictor="noisy"),
                     log_cap=4000, stp_cap=2000, want_jct=True)
w2, w1 = m.default_model()
m.simulate_batch(ctx, list(traces), m.SimOptions(policy="miso", cluster_size=4, predictor="noisy",
                                                 small_slice_model=(w2 * 0.9, w1), max_events=300))
m.best_static_partition(ctx, list(traces), cluster_size=4)
single = [t for i, t in enumerate(traces) if i != 2]
m.best_static_partition(ctx, single, cluster_size=4, chosen_only=True)  # pruned kernel
db = m.generate_traces_device(ctx, np.arange(8, dtype=np.uint64), 50, lambda_s=10.0)
m.simulate_batch(ctx, db, m.SimOptions(policy="miso", cluster_size=4, predictor="noisy"))
# the asynchronous-STP kernels (no log; STP series): engine and helper warps
m.simulate_batch(ctx, list(traces), m.SimOptions(policy="oracle", cluster_size=4), stp_cap=2000)
torch.cuda.synchronize()
print("sanitize run ok")
