#!/usr/bin/env python3
"""best_static_partition over config-4 traces (profiling/A-B helper, GPU only): one warm-up
call, then the median of 3 timed calls (host task building + one device launch each)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = miso.Context(0)
traces = miso.generate_traces(range(S), 1000, lambda_s=10.0)
miso.best_static_partition(ctx, traces, cluster_size=100)  # warm-up (the profiled launch)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    miso.best_static_partition(ctx, traces, cluster_size=100)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("static search", S, "traces median", round(statistics.median(ts), 4), "s", [round(t, 4) for t in ts])
