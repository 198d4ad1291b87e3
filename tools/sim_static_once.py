#!/usr/bin/env python3
"""One best_static_partition launch over config-4 traces (profiling helper, GPU only)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = miso.Context(0)
traces = [miso.generate_trace(s, 1000, lambda_s=10.0) for s in range(S)]
torch.cuda.synchronize()
t0 = time.perf_counter()
st = miso.best_static_partition(ctx, traces, cluster_size=100)
torch.cuda.synchronize()
print("static search", S, "traces", time.perf_counter() - t0, "s")
