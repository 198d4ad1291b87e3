#!/usr/bin/env python3
"""Config-4 step on the SM partition with the optsta re-run folded into the static search
(GPU only): the probes (each trace's two likeliest winners) run with full metrics, the other
candidates JCT-only and pruned against the probes' bound; when a trace's chosen entry is a
probe its metrics are the optsta result (else that trace is re-run). Compared with the
shipped runner (bench.TrialRunner): step time and the optsta metrics' bytes."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200 import sim as S  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
os.environ["MISO_C4_GREEN_SMS"] = str(K)
runner = bench.TrialRunner(0)
tr = miso.generate_traces_device(runner.ctx[0], np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
cat = np.asarray(miso.DEFAULT_CATALOG, np.uint8)
cd = miso.Context(0)
(s_r,) = runner.part.streams(1, 1)


def folded():
    (ca, cb, cc) = runner.ctx
    sa, sb, sc = runner.part_st
    p_nop = miso.simulate_batch(ca, tr, miso.SimOptions(policy="nopart", cluster_size=100), stream=sa, defer=True)
    sb.wait_stream(sa)
    s_r.wait_stream(sa)
    p_mis = miso.simulate_batch(cc, tr, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy"),
                                stream=sc, defer=True)
    ti, e = S.static_candidates(tr)
    probe = S.static_probes(ti, e, cat)
    with torch.cuda.stream(sb):
        bound = torch.full((len(tr),), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    s_r.wait_stream(sb)
    opts = miso.SimOptions(policy="optsta", cluster_size=100)
    pi, ri = np.nonzero(probe)[0], np.nonzero(~probe)[0]
    p_pr = miso.simulate_batch(cb, tr, opts, task_trace=ti[pi].astype(np.int32), static_partitions=cat[e[pi]],
                               stream=sb, defer=True, prune_bound=bound)
    p_rest = miso.simulate_batch(cd, tr, opts, task_trace=ti[ri].astype(np.int32), static_partitions=cat[e[ri]],
                                 jct_only=True, stream=s_r, defer=True, prune_bound=bound)
    pr, rest = p_pr(), p_rest()
    table = np.full((len(tr), len(cat)), np.inf)
    table[ti[pi], e[pi]] = pr.metrics["avg_jct_s"]
    table[ti[ri], e[ri]] = rest.metrics["avg_jct_s"]
    chosen = table.argmin(axis=1)
    where = {(int(a), int(b)): k for k, (a, b) in enumerate(zip(ti[pi], e[pi]))}
    rows = [where.get((t, int(chosen[t]))) for t in range(len(tr))]
    missing = [t for t, r in enumerate(rows) if r is None]
    met = pr.metrics[[r if r is not None else 0 for r in rows]].copy()
    return p_nop(), chosen, met, p_mis(), len(missing)


def timed(f):
    f()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(sorted(ts)[1] * 1e3, 1), r


out = {"k": K}
out["shipped_ms"], ref = timed(lambda: runner(tr))
out["folded_ms"], got = timed(folded)
out["reruns_needed"] = got[4]
out["chosen_same"] = [c for c, _ in ref[1]] == got[1].tolist()
out["optsta_metrics_same"] = ref[2].metrics.tobytes() == got[2].tobytes()
out["shipped_ms_again"], _ = timed(lambda: runner(tr))
print(json.dumps(out))
