#!/usr/bin/env python3
"""What slows the config-4 miso launch when the best-static search is queued behind it?
(GPU only) miso (1024 config-4 seeds) timed with CUDA events on its stream: alone; with a
200 ms spin kernel on another stream; with nopart on another context; with the static
search's host-side preparation only (candidate list, probes); with the whole pruned static
search queued behind a 300 ms spin (so its kernel starts after miso ends)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402
from paper_2207_11428_b200 import sim as S  # noqa: E402

ctx, ctx2, ctx3 = miso.Context(0), miso.Context(0), miso.Context(0)
tr = miso.generate_traces_device(ctx, np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
opts = miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")


def run(extra):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s1)
    r = miso.simulate_batch(ctx, tr, opts, stream=s1, defer=True)
    b.record(s1)
    extra()
    r()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b), 1)


def sleep():
    with torch.cuda.stream(s2):
        torch.cuda._sleep(int(200 * 1.965e6))


def nopart():
    miso.simulate_batch(ctx2, tr, miso.SimOptions(policy="nopart", cluster_size=100), stream=s2)


def host_prep():
    cat = np.asarray(miso.DEFAULT_CATALOG, np.uint8)
    ti, e = S.static_candidates(tr)
    S.static_probes(ti, e, cat)


def static_queued():
    with torch.cuda.stream(s3):
        torch.cuda._sleep(int(300 * 1.965e6))
    miso.best_static_partition(ctx3, tr, cluster_size=100, stream=s3, chosen_only=True)


out = {}
for k, f in (("alone", lambda: None), ("sleep", sleep), ("nopart", nopart), ("host_prep", host_prep),
             ("static_queued", static_queued)):
    run(f)
    out[k] = [run(f) for _ in range(2)]
print(json.dumps(out))
