#!/usr/bin/env python3
"""Config-4 trial step with the miso simulations on a green context of K SMs and the other
sets (nopart, the chosen-only static search and its optsta re-run) on the remaining SMs
(GPU only): step time per K, against the shared-GPU runner (K = 0)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import cuda.bindings.driver as drv  # noqa: E402
import paper_2207_11428_b200 as miso  # noqa: E402


def ok(r):
    err, *rest = r if isinstance(r, tuple) else (r,)
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return rest[0] if len(rest) == 1 else rest


torch.cuda.init()
torch.zeros(1, device="cuda")
dev = ok(drv.cuDeviceGet(0))
res = ok(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))


def split(k):
    """Two green contexts: k SMs and the rest; two streams on the second."""
    groups, n, rem = ok(drv.cuDevSmResourceSplitByCount(1, res, 0, k))
    out = []
    for r, nst in ((groups[0], 1), (rem, 2)):
        desc = ok(drv.cuDevResourceGenerateDesc([r], 1))
        g = ok(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        sms = ok(drv.cuGreenCtxGetDevResource(g, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM)).sm.smCount
        sts = [torch.cuda.ExternalStream(int(ok(drv.cuGreenCtxStreamCreate(
            g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0)))) for _ in range(nst)]
        out.append((g, sms, sts))
    return out


ca, cb, cc = miso.Context(0), miso.Context(0), miso.Context(0)
import os
S = int(os.environ.get("GREEN_SEEDS", "1024"))
tr = miso.generate_traces_device(ca, np.arange(S, dtype=np.uint64), 1000, lambda_s=10.0)
sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def step(s_mis, s_nop, s_st):
    p_nop = miso.simulate_batch(ca, tr, miso.SimOptions(policy="nopart", cluster_size=100), stream=s_nop, defer=True)
    p_mis = miso.simulate_batch(cc, tr, miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy"),
                                stream=s_mis, defer=True)
    st = miso.best_static_partition(cb, tr, cluster_size=100, stream=s_st, chosen_only=True)
    sta = miso.simulate_batch(cb, tr, miso.SimOptions(policy="optsta", cluster_size=100),
                              static_partitions=[miso.DEFAULT_CATALOG[e] for e, _ in st], stream=s_st)
    return p_nop(), st, sta, p_mis()


def timed(*streams):
    step(*streams)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = step(*streams)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(sorted(ts)[1] * 1e3, 1), r


out = {}
out["shared_ms"], ref = timed(sc, sa, sb)
for k in [int(a) for a in sys.argv[1:]] or [40, 48, 56, 64, 72]:
    (gm, nm, (sm,)), (go, no, (so1, so2)) = split(k)
    ms, r = timed(sm, so1, so2)
    same = all(a.metrics.tobytes() == b.metrics.tobytes() for a, b in ((r[0], ref[0]), (r[2], ref[2]), (r[3], ref[3])))
    out[f"miso{nm}_rest{no}_ms"] = ms
    out[f"miso{nm}_same"] = same
print(json.dumps(out))
