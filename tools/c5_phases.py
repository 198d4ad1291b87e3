"""Config-5 trial phases at 8192 device traces: each simulation set alone (CUDA-synchronised
wall time), full and pruned static search."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ctx = miso.Context(0)
traces = miso.generate_traces_device(ctx, np.arange(S, dtype=np.uint64), 1000, lambda_s=10.0)


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return round(time.perf_counter() - t0, 4), r


for rep in range(2):
    out = {}
    out["nopart"], _ = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="nopart", cluster_size=100)))
    out["miso"], _ = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")))
    out["static_full"], st = t(lambda: miso.best_static_partition(ctx, traces, cluster_size=100))
    out["static_pruned"], sp = t(lambda: miso.best_static_partition(ctx, traces, cluster_size=100, chosen_only=True))
    out["same_entries"] = all(a[0] == b[0] for a, b in zip(st, sp))
    out["optsta"], _ = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="optsta", cluster_size=100),
                                                     static_partitions=[miso.DEFAULT_CATALOG[e] for e, _ in st]))
    print(json.dumps(out), flush=True)
