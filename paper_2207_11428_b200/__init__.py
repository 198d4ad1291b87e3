"""B200-native MISO decision core (arXiv 2207.11428): predictor -> partition search -> simulator.

Python binding of the C ABI in include/miso_b200.h (the drop-in boundary). The compute path is
the in-tree CUDA library paper_2207_11428_b200/_lib/libmiso_b200.so; there is no CPU fallback:
importing this package without the built library raises.
"""
from __future__ import annotations

from ._native import (  # noqa: F401
    CAND_BAD_M,
    CAND_INFEASIBLE,
    KIND_NAMES,
    NUM_CANDIDATES,
    Assignment,
    AssignmentVector,
    BatchList,
    Context,
    MisoError,
    default_model,
    lib,
    lib_path,
)
from .catalog import DEFAULT_CATALOG, partition_name  # noqa: F401
from .sim import (DeviceTraceBatch, SimOptions, Trace, TraceBatch, best_static_partition,  # noqa: F401
                  generate_trace, generate_traces, generate_traces_device, render_log,
                  simulate_batch)
from . import tracefile  # noqa: F401,E402

__all__ = [
    "Context", "BatchList", "Assignment", "AssignmentVector", "MisoError", "DEFAULT_CATALOG",
    "partition_name", "CAND_INFEASIBLE", "CAND_BAD_M", "NUM_CANDIDATES", "KIND_NAMES",
    "SimOptions", "Trace", "TraceBatch", "DeviceTraceBatch", "generate_trace", "generate_traces",
    "generate_traces_device", "simulate_batch", "best_static_partition", "render_log", "tracefile",
]
