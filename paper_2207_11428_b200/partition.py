"""SM partitions for concurrent simulation sets (green contexts, CUDA 12.4+ driver API).

A config-4 trial batch runs the miso simulations (a latency-bound chain per seed) beside the
best-static search and the other policies. Beside any co-runner the miso warps run about twice
as slow, through instruction fetch: every resident kernel's hot code competes for the SM's
instruction cache. `SmPartition` splits the device's SMs into two green
contexts and hands out streams on each, so the two groups of kernels never share an SM. Work
on these streams uses the ordinary (primary-context) allocations; results are unchanged.
"""
from __future__ import annotations

from typing import List


class SmPartition:
    """Two disjoint SM groups of one device: `first` holds about `k` SMs (the driver rounds to
    its split granularity), `second` the rest. `streams(group, n)` returns n torch streams whose
    kernels run only on that group's SMs. Raises RuntimeError if green contexts are unavailable."""

    def __init__(self, device: int, k: int):
        import torch
        try:
            import cuda.bindings.driver as drv
        except ImportError as e:  # pragma: no cover - cuda-python is in the image
            raise RuntimeError(f"cuda-python unavailable: {e}") from e
        self._drv, self._torch = drv, torch
        torch.cuda.init()
        with torch.cuda.device(device):
            torch.zeros(1, device=f"cuda:{device}")  # the primary context exists and is current
        dev = self._ok(drv.cuDeviceGet(device))
        res = self._ok(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
        groups, _, rest = self._ok(drv.cuDevSmResourceSplitByCount(1, res, 0, int(k)))
        self._ctx, self.sms = [], []
        for r in (groups[0], rest):
            desc = self._ok(drv.cuDevResourceGenerateDesc([r], 1))
            g = self._ok(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
            self._ctx.append(g)
            self.sms.append(self._ok(drv.cuGreenCtxGetDevResource(
                g, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM)).sm.smCount)
        self._streams = []

    def _ok(self, r):
        err, *rest = r if isinstance(r, tuple) else (r,)
        if err != self._drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"green context setup failed: {err}")
        return rest[0] if len(rest) == 1 else rest

    def streams(self, group: int, n: int = 1) -> List:
        drv = self._drv
        out = []
        for _ in range(n):
            s = self._ok(drv.cuGreenCtxStreamCreate(self._ctx[group], drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
            self._streams.append(s)
            out.append(self._torch.cuda.ExternalStream(int(s)))
        return out

    def close(self):
        drv = self._drv
        self._torch.cuda.synchronize()
        for s in self._streams:
            drv.cuStreamDestroy(s)
        for g in self._ctx:
            drv.cuGreenCtxDestroy(g)
        self._streams, self._ctx = [], []
