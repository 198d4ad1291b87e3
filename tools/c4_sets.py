#!/usr/bin/env python3
"""Config-4 simulation sets, each alone on the GPU (GPU only): 1024 device-generated traces;
nopart, the chosen-only best-static search, optsta on one partition, and miso (noisy), each
timed as the median of 3 calls (wall clock around call + synchronize; traces stay on the
device, so the calls are dominated by their kernels)."""
import json
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = miso.Context(0)
tr = miso.generate_traces_device(ctx, np.arange(N, dtype=np.uint64), 1000, lambda_s=10.0)


def med(f, reps=3):
    f()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e3, 2), r


out = {"traces": N}
out["nopart_ms"], r = med(lambda: miso.simulate_batch(ctx, tr, miso.SimOptions(policy="nopart", cluster_size=100)))
out["ev_nopart"] = float(r.metrics["events"].mean())
out["static_pruned_ms"], _ = med(lambda: miso.best_static_partition(ctx, tr, cluster_size=100, chosen_only=True))
out["optsta_ms"], r = med(lambda: miso.simulate_batch(ctx, tr, miso.SimOptions(policy="optsta", cluster_size=100),
                                                     static_partitions=[miso.DEFAULT_CATALOG[8]] * N))
out["ev_optsta"] = float(r.metrics["events"].mean())
out["miso_ms"], r = med(lambda: miso.simulate_batch(ctx, tr, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")))
out["ev_miso"] = float(r.metrics["events"].mean())
print(json.dumps(out))
