#!/usr/bin/env python3
"""The asynchronous-STP kernels against the synchronous ones (GPU only): miso and oracle over
config-4 traces, with and without STP series -- every metric byte and every series point
identical -- then timings of both. Run as MISO_B200_SIM_ASYNC_STP=0 / =1 subprocesses."""
import json
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    sys.path.insert(0, ".")
    import paper_2207_11428_b200 as miso
    ctx = miso.Context(0)
    n = int(sys.argv[2])
    tr = miso.generate_traces_device(ctx, np.arange(n, dtype=np.uint64), 1000, lambda_s=10.0)
    out = {}
    for pol in ("miso", "oracle"):
        o = miso.SimOptions(policy=pol, cluster_size=100, predictor="noisy")
        r = miso.simulate_batch(ctx, tr, o)
        out[pol] = r.metrics.tobytes().hex()
        r2 = miso.simulate_batch(ctx, tr[:64], o, stp_cap=20000)
        out[pol + "_series"] = "".join(s.tobytes().hex() for s in r2.stp) + r2.metrics.tobytes().hex()
    # multi-instance jobs (clones spawned mid-run) and a QoS class, smaller cluster
    ht = miso.generate_traces(range(12), 120, lambda_s=20.0)
    for i, t in enumerate(ht):
        if i % 3 == 0:
            t.instances = np.array([1] * 10 + [3] + [1] * 109, np.uint8)
        if i % 4 == 1:
            t.qos_kind = np.array([-1] * 50 + [2] + [-1] * 69, np.int8)
    for pol in ("miso", "oracle"):
        o = miso.SimOptions(policy=pol, cluster_size=8, predictor="noisy")
        r = miso.simulate_batch(ctx, list(ht), o, stp_cap=5000)
        out[pol + "_clones"] = r.metrics.tobytes().hex() + "".join(s.tobytes().hex() for s in r.stp)
    o = miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        miso.simulate_batch(ctx, tr, o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["miso_ms"] = sorted(ts)[1]
    print(json.dumps(out))
    sys.exit(0)

res = {}
for mode in ("0", "1"):
    env = dict(os.environ, MISO_B200_SIM_ASYNC_STP=mode)
    p = subprocess.run([sys.executable, __file__, "child", sys.argv[1] if len(sys.argv) > 1 else "1024"],
                       env=env, capture_output=True, text=True, timeout=600)
    if p.returncode:
        print(p.stderr[-2000:])
        sys.exit(1)
    res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
same = {k: res["0"][k] == res["1"][k] for k in res["0"] if k != "miso_ms"}
print(json.dumps({"identical": same, "miso_ms_sync": res["0"]["miso_ms"], "miso_ms_async": res["1"]["miso_ms"]}))
