#!/usr/bin/env python3
"""Time the chosen-only static search's two launches (probes, then the pruned rest) alone
and with miso / nopart running beside them, for 1024 config-4 traces."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200 import sim as S  # noqa: E402

ctx = miso.Context(0)
traces = miso.generate_traces_device(ctx, np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
orig = S.simulate_batch
rec = []


def timed_sim(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig(*a, **k)
    torch.cuda.synchronize()
    rec.append((len(k.get("task_trace") if k.get("task_trace") is not None else []),
                time.perf_counter() - t0, int((r.metrics["status"] == 5).sum()),
                float(r.metrics["events"].mean())))
    return r


S.simulate_batch = timed_sim
out = {}
for rep in range(2):
    rec.clear()
    t0 = time.perf_counter()
    miso.best_static_partition(ctx, traces, cluster_size=100, chosen_only=True)
    out["chosen_only_s"] = time.perf_counter() - t0
    out["launches"] = [{"tasks": n, "s": s, "stopped": p, "mean_events": e} for n, s, p, e in rec]
    rec.clear()
    t0 = time.perf_counter()
    miso.best_static_partition(ctx, traces, cluster_size=100)
    out["full_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
S.static_candidates(traces)
out["static_candidates_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
S._csr(traces)
out["csr_s"] = time.perf_counter() - t0
print(json.dumps(out, indent=1))
