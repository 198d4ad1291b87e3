"""Multi-GPU sharding for the decision core (one process per GPU, torch.distributed).

Every instance (job mix) and every trace seed is independent, so the data
path has no collective: rank r owns the contiguous range [r*N/P, (r+1)*N/P) of instances or
seeds and computes it on its own GPU. The only communication is the final result gather to
rank 0 -- an all_gather of equal-size padded shards (NCCL has no gather; on NVLink/NVSwitch this
is one small collective per batch) -- and statistics are reduced on the host in global order,
so results are identical to a single-GPU run regardless of P (an FP64 NCCL reduction would
change the summation order).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block of [0, n) owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_csr(offsets: np.ndarray, rank: int, world: int):
    """Instances [lo, hi) of a CSR batch: (lo, hi, local offsets rebased to 0, row range)."""
    n = len(offsets) - 1
    lo, hi = shard_range(n, rank, world)
    off = np.asarray(offsets, np.int64)
    r0, r1 = int(off[lo]), int(off[hi])
    return lo, hi, (off[lo:hi + 1] - r0).astype(np.uint32), (r0, r1)


def gather_to_rank0(local: np.ndarray, n_total: int, rank: int, world: int, group=None,
                    device=None) -> Optional[np.ndarray]:
    """All-gather equal-size padded shards of a 1-D array (any fixed-width dtype) and return
    the concatenation in global order on rank 0 (None elsewhere). Byte-exact."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local.copy()
    per = -(-n_total // world)  # ceil
    raw = np.ascontiguousarray(local).view(np.uint8)
    isz = local.dtype.itemsize
    buf = np.zeros(per * isz, np.uint8)
    buf[: raw.size] = raw
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        parts.append(outs[r].cpu().numpy()[: (hi - lo) * isz])
    return np.concatenate(parts).view(local.dtype)
