#!/usr/bin/env python3
"""Config-4 step (bench.py TrialRunner on the SM partition) with the static search staggered
behind nopart (MISO_C4_STAGGER=1, default) or launched beside it (0), alternating (GPU only)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402

runner = bench.TrialRunner(0)
tr = miso.generate_traces_device(runner.ctx[0], np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)


def t():
    runner(tr)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        runner(tr)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(sorted(ts)[1] * 1e3, 1)


out = {"stagger": [], "beside": []}
for i in range(3):
    os.environ["MISO_C4_STAGGER"] = "1"
    out["stagger"].append(t())
    os.environ["MISO_C4_STAGGER"] = "0"
    out["beside"].append(t())
print(json.dumps(out))
