"""Run one simulator launch (policy, n seeds) -- for ncu captures."""
import sys
sys.path.insert(0, ".")
import paper_2207_11428_b200 as miso
pol, n = sys.argv[1], int(sys.argv[2])
ctx = miso.Context(0)
traces = [miso.generate_trace(s, 1000, lambda_s=10.0) for s in range(n)]
kw = {}
if pol == "optsta":
    kw["static_partitions"] = [miso.DEFAULT_CATALOG[8]] * n
opts = miso.SimOptions(policy=pol, cluster_size=100, predictor="noisy" if pol == "miso" else "oracle")
r = miso.simulate_batch(ctx, traces, opts, **kw)
print(r.metrics["events"].mean(), r.metrics["status"].max())
