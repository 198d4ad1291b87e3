#!/usr/bin/env python3
"""How far apart are the best-static candidates? For 1024 config-4 traces: every feasible
(trace, entry) optsta simulation's avg JCT relative to the trace's best, and its event count."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200.catalog import DEFAULT_CATALOG  # noqa: E402

ctx = miso.Context(0)
traces = miso.generate_traces(range(1024), 1000, lambda_s=10.0)
res = miso.best_static_partition(ctx, traces, cluster_size=100)
tab = np.array([r[1] for r in res])
best = tab.min(axis=1, keepdims=True)
rel = tab / best
fin = np.isfinite(rel)
r = rel[fin]
# per entry: how often it wins, median relative JCT
win = np.bincount([c for c, _ in res], minlength=len(DEFAULT_CATALOG))
per_entry = {}
for e in range(len(DEFAULT_CATALOG)):
    col = rel[:, e][np.isfinite(rel[:, e])]
    if len(col):
        per_entry[str(DEFAULT_CATALOG[e])] = {"n": int(len(col)), "wins": int(win[e]),
                                               "median_rel": float(np.median(col)),
                                               "p10_rel": float(np.percentile(col, 10))}
# event counts of the candidates
opts = miso.SimOptions(policy="optsta", cluster_size=100)
ti, ee = np.nonzero(fin)
sub = ti < 256
out = miso.simulate_batch(ctx, traces, opts, task_trace=ti[sub].astype(np.int32),
                          static_partitions=np.asarray(DEFAULT_CATALOG, np.uint8)[ee[sub]], jct_only=True)
ev = out.metrics["events"]
relsub = rel[ti[sub], ee[sub]]
print(json.dumps({"candidates": int(fin.sum()), "rel_quantiles": {q: float(np.percentile(r, q)) for q in (10, 25, 50, 75, 90)},
                  "frac_rel_gt_1_5": float((r > 1.5).mean()), "frac_rel_gt_2": float((r > 2).mean()),
                  "events_mean": float(ev.mean()), "events_by_rel": {
                      "rel<1.2": float(ev[relsub < 1.2].mean()), "rel>2": float(ev[relsub > 2].mean()) if (relsub > 2).any() else None},
                  "per_entry": per_entry}, indent=1))
