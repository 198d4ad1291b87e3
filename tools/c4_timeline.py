#!/usr/bin/env python3
"""Config-4 trial batch (as bench.py --config c4) with CUDA events around each stream's work:
prints start/end offsets (ms) of nopart, miso, the static search and the optsta re-run,
for the full and the chosen-only (pruned) static search."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402

S = 1024
ctx_a, ctx_b, ctx_c = miso.Context(0), miso.Context(0), miso.Context(0)
traces = miso.generate_traces_device(ctx_a, np.arange(S, dtype=np.uint64), 1000, lambda_s=10.0)
s_a, s_b, s_c, s_d = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ctx_d = miso.Context(0)
from paper_2207_11428_b200 import sim as SIM  # noqa: E402
cat = np.asarray(miso.DEFAULT_CATALOG, np.uint8)
ti, ee = SIM.static_candidates(traces)
probe = SIM.static_probes(ti, ee, cat)


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def batch(chosen_only, chunks=1, delay_ms=0.0):
    t0 = ev(torch.cuda.current_stream())
    for s in (s_a, s_b, s_c):
        s.wait_stream(torch.cuda.current_stream())
    if delay_ms > 0:  # the static search (and its re-run) start delay_ms after miso
        with torch.cuda.stream(s_b):
            torch.cuda._sleep(int(delay_ms * 1.965e6))
    a0 = ev(s_a)
    p_nop = miso.simulate_batch(ctx_a, traces, miso.SimOptions(policy="nopart", cluster_size=100), stream=s_a, defer=True)
    a1 = ev(s_a)
    c0 = ev(s_c)
    p_mis = miso.simulate_batch(ctx_c, traces, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy"), stream=s_c, defer=True)
    c1 = ev(s_c)
    b0 = ev(s_b)
    st = []
    step = S // chunks
    for c in range(chunks):  # fewer concurrent static warps: smaller L2 footprint beside miso
        st += miso.best_static_partition(ctx_b, traces[c * step:(c + 1) * step], cluster_size=100,
                                         stream=s_b, chosen_only=chosen_only)
    b1 = ev(s_b)
    miso.simulate_batch(ctx_b, traces, miso.SimOptions(policy="optsta", cluster_size=100),
                        static_partitions=[miso.DEFAULT_CATALOG[e] for e, _ in st], stream=s_b)
    b2 = ev(s_b)
    p_nop(); p_mis()
    torch.cuda.synchronize()
    f = lambda e: round(t0.elapsed_time(e), 1)  # noqa: E731
    return {"nopart": [f(a0), f(a1)], "miso": [f(c0), f(c1)], "static": [f(b0), f(b1)], "rerun": [f(b1), f(b2)]}


def batch_probes_full(rest_waits=False):
    """Probes in full mode (their metrics are the optsta result when one of them is chosen)
    beside the other candidates (JCT-only, pruned against the probes' bound) on a 4th stream."""
    t0 = ev(torch.cuda.current_stream())
    for s in (s_a, s_b, s_c, s_d):
        s.wait_stream(torch.cuda.current_stream())
    a0 = ev(s_a)
    p_nop = miso.simulate_batch(ctx_a, traces, miso.SimOptions(policy="nopart", cluster_size=100), stream=s_a, defer=True)
    a1 = ev(s_a)
    c0 = ev(s_c)
    p_mis = miso.simulate_batch(ctx_c, traces, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy"), stream=s_c, defer=True)
    c1 = ev(s_c)
    with torch.cuda.stream(s_b):
        bound = torch.full((S,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    s_d.wait_stream(s_b)
    opts = miso.SimOptions(policy="optsta", cluster_size=100)
    b0 = ev(s_b)
    p_pr = miso.simulate_batch(ctx_b, traces, opts, task_trace=ti[probe].astype(np.int32),
                               static_partitions=cat[ee[probe]], stream=s_b, defer=True, prune_bound=bound)
    b1 = ev(s_b)
    if rest_waits:  # the pruned rest starts once every trace's bound is set by its probes
        s_d.wait_stream(s_b)
    d0 = ev(s_d)
    p_rest = miso.simulate_batch(ctx_d, traces, opts, task_trace=ti[~probe].astype(np.int32),
                                 static_partitions=cat[ee[~probe]], jct_only=True, stream=s_d, defer=True,
                                 prune_bound=bound)
    d1 = ev(s_d)
    pr, rest = p_pr(), p_rest()
    table = np.full((S, len(cat)), np.inf)
    table[ti[probe], ee[probe]] = pr.metrics["avg_jct_s"]
    table[ti[~probe], ee[~probe]] = rest.metrics["avg_jct_s"]
    chosen = table.argmin(axis=1)
    n_rerun = int((~np.isin(np.arange(S) * 64 + chosen, ti[probe] * 64 + ee[probe])).sum())
    p_nop(); p_mis()
    torch.cuda.synchronize()
    f = lambda e: round(t0.elapsed_time(e), 1)  # noqa: E731
    return {"nopart": [f(a0), f(a1)], "miso": [f(c0), f(c1)], "probes_full": [f(b0), f(b1)],
            "rest_pruned": [f(d0), f(d1)], "reruns_needed": n_rerun}


out = {}
if len(sys.argv) > 1 and sys.argv[1] == "delay":  # static search started after a delay
    for rep in range(2):
        for d in (0, 80, 300):
            batch(True, 1, d)
            out[f"pruned_delay{d}_{rep}"] = batch(True, 1, d)
    print(json.dumps(out))
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "probes":  # probes (full metrics) first, then the rest
    for rep in range(2):
        for w in (False, True):
            batch_probes_full(w)
            out[f"probes_full{'_then_rest' if w else ''}_{rep}"] = batch_probes_full(w)
    print(json.dumps(out))
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "chunks":  # the static search split into sequential launches
    for rep in range(2):
        for ch in (1, 2, 4, 8):
            batch(True, ch)
            out[f"pruned_chunks{ch}_{rep}"] = batch(True, ch)
    print(json.dumps(out))
    sys.exit(0)
for rep in range(2):
    for mode in (False, True):
        batch(mode)
        out[f"{'pruned' if mode else 'full'}_{rep}"] = batch(mode)
    batch_probes_full()
    out[f"probes_full_{rep}"] = batch_probes_full()
print(json.dumps(out))
