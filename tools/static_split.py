import sys, time, numpy as np
sys.path.insert(0, ".")
import torch, paper_2207_11428_b200 as miso
from paper_2207_11428_b200 import sim as S
ctx = miso.Context(0)
traces = miso.generate_traces(range(1024), 1000, lambda_s=10.0)
miso.best_static_partition(ctx, traces, cluster_size=100)
torch.cuda.synchronize()
# phase 1: task building (copy of best_static_partition's loop)
t0 = time.perf_counter()
from paper_2207_11428_b200.catalog import DEFAULT_CATALOG, GPC, MEM_GB
cat = list(DEFAULT_CATALOG)
mem_gb = np.array(MEM_GB); gpc = np.array(GPC)
largest = np.array([max(k for k in range(5) if c[k] > 0) for c in cat])
tasks, parts = [], []
for ti, t in enumerate(traces):
    qos = np.full(t.n, -1) if t.qos_kind is None else np.asarray(t.qos_kind)
    qg = np.where(qos >= 0, gpc[np.maximum(qos, 0)], 0)
    ok = (mem_gb[None, :] >= np.asarray(t.mem_gb)[:, None]) & (gpc[None, :] >= qg[:, None])
    need = int(ok.argmax(axis=1).max())
    for e in np.nonzero(largest >= need)[0]:
        tasks.append((ti, int(e))); parts.append(cat[e])
t1 = time.perf_counter()
opts = miso.SimOptions(policy="optsta", cluster_size=100)
ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
ev0.record()
res = miso.simulate_batch(ctx, traces, opts, task_trace=[t for t, _ in tasks], static_partitions=parts, jct_only=True)
ev1.record(); torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"tasks {len(tasks)} build {t1-t0:.4f}s simulate_batch {t2-t1:.4f}s (events {ev0.elapsed_time(ev1)/1e3:.4f}s)")
