#!/usr/bin/env python3
"""Config-4 trial step on the SM partition (as bench.py's TrialRunner): CUDA-event offsets of
each set and the host time spent preparing the static search and the re-run (GPU only)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200 import sim as S  # noqa: E402
from paper_2207_11428_b200.partition import SmPartition  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ca, cb, cc = miso.Context(0), miso.Context(0), miso.Context(0)
tr = miso.generate_traces_device(ca, np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
part = SmPartition(0, k)
(s_m,), (s_n, s_s) = part.streams(0), part.streams(1, 2)


def ev(s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    return e


def step():
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    t0 = ev(torch.cuda.current_stream())
    p_nop = miso.simulate_batch(ca, tr, miso.SimOptions(policy="nopart", cluster_size=100), stream=s_n, defer=True)
    n1 = ev(s_n)
    p_mis = miso.simulate_batch(cc, tr, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy"),
                                stream=s_m, defer=True)
    m1 = ev(s_m)
    h1 = time.perf_counter()
    st = miso.best_static_partition(cb, tr, cluster_size=100, stream=s_s, chosen_only=True)
    h2 = time.perf_counter()
    b1 = ev(s_s)
    sta = miso.simulate_batch(cb, tr, miso.SimOptions(policy="optsta", cluster_size=100),
                              static_partitions=[miso.DEFAULT_CATALOG[e] for e, _ in st], stream=s_s)
    h3 = time.perf_counter()
    b2 = ev(s_s)
    p_nop(), p_mis()
    torch.cuda.synchronize()
    h4 = time.perf_counter()
    f = lambda e: round(t0.elapsed_time(e), 1)  # noqa: E731
    return {"nopart_end": f(n1), "miso_end": f(m1), "static_end": f(b1), "rerun_end": f(b2),
            "host_launch_ms": round((h1 - h0) * 1e3, 1), "host_static_call_ms": round((h2 - h1) * 1e3, 1),
            "host_rerun_call_ms": round((h3 - h2) * 1e3, 1), "host_total_ms": round((h4 - h0) * 1e3, 1)}


step()
out = [step() for _ in range(2)]
# host-only parts of best_static_partition
cat = np.asarray(miso.DEFAULT_CATALOG, np.uint8)
t = time.perf_counter(); ti, e = S.static_candidates(tr); c1 = time.perf_counter() - t
t = time.perf_counter(); S.static_probes(ti, e, cat); c2 = time.perf_counter() - t
print(json.dumps({"k": k, "steps": out, "static_candidates_ms": round(c1 * 1e3, 1),
                  "static_probes_ms": round(c2 * 1e3, 1)}))
part.close()
