#!/usr/bin/env python3
"""How much of the best-static search's work does pruning remove, and how much could it?
(GPU only.) For S config-4 traces: events and time of the full search, of the shipped
chosen-only search (probes first in one launch), of a two-launch variant (probes, then the
rest against their bound) and of the ideal (every candidate against the winner's exact JCT
sum from the start)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200 import sim as S  # noqa: E402
from paper_2207_11428_b200.catalog import DEFAULT_CATALOG  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = miso.Context(0)
traces = miso.generate_traces_device(ctx, np.arange(N, dtype=np.uint64), 1000, lambda_s=10.0)
cat = list(DEFAULT_CATALOG)
catc = np.asarray(cat, np.uint8).reshape(-1, 5)
opts = S.SimOptions(policy="optsta", cluster_size=100)
ti, e = S.static_candidates(traces, cat)
probe = S.static_probes(ti, e, catc)
dev = torch.device("cuda", 0)
out = {"traces": N, "candidates": int(len(ti)), "probes": int(probe.sum())}


def run(sel, bound, tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kw = {} if bound is None else {"prune_bound": bound}
    r = S.simulate_batch(ctx, traces, opts, task_trace=ti[sel].astype(np.int32),
                         static_partitions=catc[e[sel]], jct_only=True, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ev = r.metrics["events"].astype(np.int64)
    st = r.metrics["status"]
    out[tag] = {"s": round(dt, 4), "runs": int(len(sel)), "events": int(ev.sum()),
                "pruned": int((st == 5).sum()), "events_pruned_runs": int(ev[st == 5].sum())}
    return r


allsel = np.arange(len(ti))
for _ in range(2):
    full = run(allsel, None, "full")
table = np.full((N, len(cat)), np.inf)
table[ti, e] = full.metrics["avg_jct_s"]
win = table.argmin(axis=1)
out["full"]["events_winners"] = int(sum(full.metrics["events"][(ti == t) & (e == win[t])].sum() for t in range(N)))

sel = np.r_[np.nonzero(probe)[0], np.nonzero(~probe)[0]]
for _ in range(2):
    b = torch.full((N,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
    run(sel, b, "shipped")
ideal_bound = b.clone()  # after a complete pruned search: the winner's exact JCT sum
out["probe_is_winner"] = float(np.mean([win[t] in set(e[(ti == t) & probe]) for t in range(N)]))

for _ in range(2):
    b = torch.full((N,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
    run(np.nonzero(probe)[0], b, "two_launch_probes")
    run(np.nonzero(~probe)[0], b, "two_launch_rest")
for _ in range(2):
    b = ideal_bound.clone()
    run(allsel, b, "ideal_bound")
print(json.dumps(out))
