#!/usr/bin/env python3
"""Can the config-4 sets run on disjoint SM sets? (GPU only) Splits the device's SMs into two
green contexts (CUDA 12.4+ driver API via cuda-python), creates a stream in each, and checks
that torch tensors of the primary context are usable there and that the simulator launches on
them give the same results; then times miso alone on a K-SM partition."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import cuda.bindings.driver as drv  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402


def ok(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return rest[0] if len(rest) == 1 else rest


torch.cuda.init()
x = torch.zeros(1 << 20, device="cuda")
dev = ok(drv.cuDeviceGet(0))
res = ok(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
total = res.sm.smCount


def green_stream(k):
    """A stream on a green context holding k SMs (rounded by the split granularity)."""
    groups, n, rem = ok(drv.cuDevSmResourceSplitByCount(1, res, 0, k))
    desc = ok(drv.cuDevResourceGenerateDesc([groups[0]], 1))
    g = ok(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = ok(drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    r = ok(drv.cuGreenCtxGetDevResource(g, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    return g, st, r.sm.smCount


out = {"total_sms": total}
g1, s1, n1 = green_stream(64)
out["green_sms"] = n1
es = torch.cuda.ExternalStream(int(s1))
with torch.cuda.stream(es):
    x.add_(1.0)
torch.cuda.synchronize()
out["torch_on_green_stream"] = float(x.sum())
ctx = miso.Context(0)
tr = miso.generate_traces_device(ctx, np.arange(1024, dtype=np.uint64), 1000, lambda_s=10.0)
opts = miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")
want = miso.simulate_batch(ctx, tr, opts).metrics
got = miso.simulate_batch(ctx, tr, opts, stream=es)
out["sim_same_on_green"] = got.metrics.tobytes() == want.tobytes()
for k in (148, 96, 74, 48):
    try:
        g, s, n = green_stream(k)
    except Exception as e:  # noqa: BLE001
        out[f"miso_{k}"] = str(e)
        continue
    e2 = torch.cuda.ExternalStream(int(s))
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        miso.simulate_batch(ctx, tr, opts, stream=e2)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[f"miso_on_{n}_sms_ms"] = round(sorted(ts)[1] * 1e3, 1)
print(json.dumps(out))
