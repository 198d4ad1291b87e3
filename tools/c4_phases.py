import sys, time, json
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2207_11428_b200 as miso
ctx = miso.Context(0)
traces = [miso.generate_trace(s, 1000, lambda_s=10.0) for s in range(1024)]
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); return time.perf_counter() - t0, r
import time as _t
t0 = _t.perf_counter(); tasks = miso.best_static_partition  # warm import
for rep in range(2):
    a, nop = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="nopart", cluster_size=100)))
    b, st = t(lambda: miso.best_static_partition(ctx, traces, cluster_size=100))
    c, mis = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")))
    d, one = t(lambda: miso.simulate_batch(ctx, traces, miso.SimOptions(policy="optsta", cluster_size=100), static_partitions=[miso.DEFAULT_CATALOG[8]]*1024))
    print(json.dumps({"nopart_s": a, "static_search_s": b, "miso_s": c, "optsta_1024_s": d,
                      "ev_nopart": float(nop.metrics["events"].mean()), "ev_miso": float(mis.metrics["events"].mean()), "ev_optsta": float(one.metrics["events"].mean())}))
