"""ctypes binding of include/miso_b200.h plus the reference-shaped Python API.

`Context.optimize_partition(jobs)` mirrors optimize_partition (optimizer.hpp:62-115): same
argument meaning (per-job speed tables, kind order 1g..7g, already zeroed by
effective_speed), same result (partition, per-job assignment in input order, objective),
same error behaviour (ValueError == std::invalid_argument for m outside 1..7, None ==
std::nullopt). Batch calls take torch CUDA tensors (device path, stream-ordered) or numpy
arrays (host path: H2D -> search -> D2H inside the library).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from .catalog import DEFAULT_CATALOG, KIND_NAMES, partition_name

lib_path = Path(__file__).resolve().parent / "_lib" / "libmiso_b200.so"

CAND_INFEASIBLE = 0xFF
CAND_BAD_M = 0xFE
NUM_CANDIDATES = 111

E_CODES = {-1: "unexpected", -2: "invalid argument", -3: "malformed input", -4: "infeasible"}


class MisoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"miso_b200 error {code} ({E_CODES.get(code, '?')}): {msg}")
        self.code = code


def _load():
    if not lib_path.exists():
        raise ImportError(
            f"{lib_path} is missing: the CUDA library must be built (python __graft_entry__.py "
            "build / paper_2207_11428_b200/build.py). There is no CPU fallback.")
    L = C.CDLL(str(lib_path))
    vp, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
    L.miso_b200_version.restype = i32
    L.miso_b200_last_error.restype = C.c_char_p
    L.miso_b200_create.argtypes = [i32, C.POINTER(vp)]
    L.miso_b200_destroy.argtypes = [vp]
    L.miso_b200_destroy.restype = None
    L.miso_b200_set_catalog.argtypes = [vp, vp, i32]
    L.miso_b200_get_catalog.argtypes = [vp, vp]
    L.miso_b200_candidate.argtypes = [vp, i32, C.POINTER(i32), C.POINTER(i32), vp]
    L.miso_b200_optimize_batch.argtypes = [vp, vp, vp, u64, vp, vp, vp]
    L.miso_b200_optimize_batch_host.argtypes = [vp, vp, vp, u64, vp, vp]
    L.miso_b200_optimize.argtypes = [vp, vp, i32, C.POINTER(i32), vp, vp]
    L.miso_b200_host_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.miso_b200_host_free.argtypes = [vp]
    L.miso_b200_host_free.restype = None
    return L


lib = _load()


def _check(rc: int) -> int:
    if rc < 0:
        raise MisoError(rc, lib.miso_b200_last_error().decode())
    return rc


@dataclass
class Assignment:
    job_id: str
    slice: int          # kind index 0..4 (1g..7g)
    speed: float

    @property
    def slice_name(self) -> str:
        return KIND_NAMES[self.slice]


@dataclass
class AssignmentVector:
    partition: tuple    # per-kind counts [1g,2g,3g,4g,7g]
    entry: int          # index in the context's catalog
    assignments: list = field(default_factory=list)
    objective: float = 0.0

    @property
    def partition_name(self) -> str:
        return partition_name(self.partition)


def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


class Context:
    """One context per device (miso_b200_create)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.miso_b200_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._table = None

    def close(self):
        if getattr(self, "_h", None):
            lib.miso_b200_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    # --- catalog -----------------------------------------------------------
    def set_catalog(self, counts: Sequence[Sequence[int]]):
        a = np.ascontiguousarray(np.asarray(counts, np.uint8).reshape(-1, 5))
        _check(lib.miso_b200_set_catalog(self._h, a.ctypes.data, len(a)))
        self._table = None

    def catalog(self) -> np.ndarray:
        buf = np.zeros((36, 5), np.uint8)
        n = _check(lib.miso_b200_get_catalog(self._h, buf.ctypes.data))
        return buf[:n].copy()

    def candidate_table(self):
        """(entry[111] in the active catalog, m[111], place[111,7])."""
        if self._table is None:
            ent = np.zeros(NUM_CANDIDATES, np.int32)
            ms = np.zeros(NUM_CANDIDATES, np.int32)
            pl = np.zeros((NUM_CANDIDATES, 7), np.uint8)
            for c in range(NUM_CANDIDATES):
                e, m = C.c_int(), C.c_int()
                _check(lib.miso_b200_candidate(self._h, c, C.byref(e), C.byref(m),
                                               pl[c].ctypes.data))
                ent[c], ms[c] = e.value, m.value
            self._table = (ent, ms, pl)
        return self._table

    # --- optimize ----------------------------------------------------------
    def optimize_batch(self, speeds, offsets, cand=None, obj=None, stream=None):
        """Batched optimize_partition. Device path if `speeds` is a torch CUDA tensor."""
        n = len(offsets) - 1
        if _is_torch_cuda(speeds):
            import torch
            if cand is None:
                cand = torch.empty(n, dtype=torch.uint8, device=speeds.device)
            if obj is None:
                obj = torch.empty(n, dtype=torch.float64, device=speeds.device)
            assert speeds.dtype == torch.float64 and offsets.dtype in (torch.int32, torch.uint32)
            s = stream if stream is not None else torch.cuda.current_stream(speeds.device).cuda_stream
            _check(lib.miso_b200_optimize_batch(self._h, speeds.data_ptr(), offsets.data_ptr(), n,
                                                cand.data_ptr(), obj.data_ptr(), s))
            return cand, obj
        speeds = np.ascontiguousarray(speeds, np.float64)
        offsets = np.ascontiguousarray(offsets, np.uint32)
        if cand is None:
            cand = np.empty(n, np.uint8)
        if obj is None:
            obj = np.empty(n, np.float64)
        _check(lib.miso_b200_optimize_batch_host(self._h, speeds.ctypes.data, offsets.ctypes.data,
                                                 n, cand.ctypes.data, obj.ctypes.data))
        return cand, obj

    def decode(self, cand: np.ndarray, offsets: np.ndarray):
        """Per-instance active-catalog entry (-1 nullopt, -2 bad m) and packed placement[sum m]."""
        ent, ms, pl = self.candidate_table()
        cand = np.asarray(cand)
        offsets = np.asarray(offsets, np.int64)
        entry = np.where(cand == CAND_INFEASIBLE, -1, np.where(cand == CAND_BAD_M, -2, 0)).astype(np.int32)
        ok = cand < NUM_CANDIDATES
        entry[ok] = ent[cand[ok]]
        m = np.diff(offsets)
        place = np.zeros(int(offsets[-1]) if len(offsets) else 0, np.uint8)
        idx = np.nonzero(ok)[0]
        if len(idx):
            rows = np.repeat(idx, m[idx])
            j = np.arange(len(rows)) - np.repeat(np.cumsum(m[idx]) - m[idx], m[idx])
            place[np.repeat(offsets[idx], m[idx]) + j] = pl[cand[rows], j]
        return entry, place

    def optimize_partition(self, jobs) -> Optional[AssignmentVector]:
        """optimize_partition(jobs, catalog) (optimizer.hpp:62-63).

        jobs: sequence of (job_id, speeds[5]) with speeds in kind order 1g..7g.
        """
        m = len(jobs)
        if m < 1 or m > 7:
            raise ValueError(f"optimize_partition needs 1..7 jobs, got {m}")
        sp = np.ascontiguousarray([list(s) for _, s in jobs], np.float64).reshape(m, 5)
        e = C.c_int()
        place = np.zeros(7, np.uint8)
        objv = C.c_double()
        r = _check(lib.miso_b200_optimize(self._h, sp.ctypes.data, m, C.byref(e), place.ctypes.data,
                                          C.byref(objv)))
        if r == 0:
            return None
        counts = tuple(int(x) for x in self.catalog()[e.value])
        asg = [Assignment(jobs[i][0], int(place[i]), float(sp[i, place[i]])) for i in range(m)]
        return AssignmentVector(counts, e.value, asg, objv.value)


def host_alloc(nbytes: int):
    """Pinned host buffer (miso_b200_host_alloc) as a ctypes address; free with host_free."""
    p = C.c_void_p()
    _check(lib.miso_b200_host_alloc(nbytes, C.byref(p)))
    return p.value


def host_free(addr: int):
    lib.miso_b200_host_free(addr)


assert DEFAULT_CATALOG  # imported for callers
