#!/usr/bin/env python3
"""One chosen-only (pruned) best-static search over S config-4 traces (for ncu captures)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = miso.Context(0)
traces = miso.generate_traces_device(ctx, np.arange(S, dtype=np.uint64), 1000, lambda_s=10.0)
st = miso.best_static_partition(ctx, traces, cluster_size=100, chosen_only=True)
print("chosen entries", np.bincount([e for e, _ in st]).tolist())
