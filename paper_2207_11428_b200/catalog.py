"""Slice vocabulary and the default MIG catalog (host-side constants).

Mirrors topology.hpp:27-45 (kSliceTable) and :149-156 (PartitionConfig::name). The
authoritative candidate table used by the kernels is csrc/candidates_gen.cuh; this module
only names things for callers.
"""
from __future__ import annotations

import itertools

KIND_NAMES = ("1g", "2g", "3g", "4g", "7g")
GPC = (1, 2, 3, 4, 7)
MEM_GB = (5, 10, 20, 20, 40)
UNITS = (1, 2, 4, 4, 8)
MAX_COUNT = (7, 3, 2, 1, 1)


def feasible(c) -> bool:
    """PartitionConfig::violation(...) == nullopt (topology.hpp:84-101)."""
    if any(c[k] > MAX_COUNT[k] for k in range(5)) or sum(c) == 0:
        return False
    if sum(c[k] * GPC[k] for k in range(5)) > 7 or sum(c[k] * UNITS[k] for k in range(5)) > 8:
        return False
    return not (c[3] > 0 and c[2] > 0)


def gpc_vector(c):
    return [GPC[k] for k in range(4, -1, -1) for _ in range(c[k])]


def partition_name(c) -> str:
    """PartitionConfig::name (topology.hpp:149-156), e.g. '3g+2g+2g'."""
    return "+".join(KIND_NAMES[k] for k in range(4, -1, -1) for _ in range(c[k]))


def build_catalog():
    """build_catalog (topology.hpp:189-202): 36 entries, descending gpc-vector order."""
    ents = [c for c in itertools.product(*(range(m + 1) for m in MAX_COUNT)) if feasible(c)]
    ents.sort(key=gpc_vector, reverse=True)
    return [tuple(c) for c in ents]


DEFAULT_CATALOG = build_catalog()


def min_slice_for(mem_gb: int, qos_min_gpc: int = 0):
    """topology.hpp:68-72; None when no kind fits."""
    for k in range(5):
        if MEM_GB[k] >= mem_gb and GPC[k] >= qos_min_gpc:
            return k
    return None


def effective_speed(speed: float, kind: int, mem_gb: int, qos_kind=None) -> float:
    """profiles.hpp:60-65."""
    if MEM_GB[kind] < mem_gb:
        return 0.0
    if qos_kind is not None and GPC[kind] < GPC[qos_kind]:
        return 0.0
    return speed
