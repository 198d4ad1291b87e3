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

import os

# MISO_B200_LIB selects an alternative in-tree build (tuning experiments only).
lib_path = Path(os.environ.get("MISO_B200_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libmiso_b200.so")

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
    L.miso_b200_optimize_batches.argtypes = [vp, vp, i32, vp]
    L.miso_b200_optimize.argtypes = [vp, vp, i32, C.POINTER(i32), vp, vp]
    L.miso_b200_default_model.argtypes = [vp, vp]
    L.miso_b200_predict_batch.argtypes = [vp, vp, u64, i32, u64, u64, i32, C.c_double, vp, vp,
                                          vp, vp]
    L.miso_b200_decide_batch.argtypes = [vp, vp, vp, vp, vp, vp, u64, u64, i32, C.c_double, vp,
                                         vp, vp, vp, vp, vp]
    L.miso_b200_decide.argtypes = [vp, vp, vp, vp, i32, u64, u64, i32, C.c_double,
                                   C.POINTER(i32), vp, C.POINTER(C.c_double), vp]
    L.miso_b200_decide_server.argtypes = [vp, i32]
    L.miso_b200_max_spare_slice.argtypes = [vp, vp, i32, C.POINTER(i32)]
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


class _BatchC(C.Structure):
    """miso_b200_batch (include/miso_b200.h)."""
    _fields_ = [("speeds", C.c_void_p), ("offsets", C.c_void_p), ("n", C.c_uint64),
                ("cand", C.c_void_p), ("obj", C.c_void_p)]


class BatchList:
    """The miso_b200_batch descriptors of a list of (speeds, offsets, cand, obj) CUDA tensor
    tuples, checked once (the tensors must outlive the list)."""

    def __init__(self, batches):
        self.arr = (_BatchC * max(1, len(batches)))()
        self.n = len(batches)
        self.device = None
        self._keep = list(batches)
        for i, (sp, off, cand, obj) in enumerate(batches):
            n = len(off) - 1
            _check_device_args(sp, off, cand, obj, n)
            if self.device is None:
                self.device = sp.device
            elif sp.device != self.device:
                raise ValueError("all batches must be on one device")
            self.arr[i] = _BatchC(sp.data_ptr(), off.data_ptr(), n, cand.data_ptr(), obj.data_ptr())


def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _check_device_args(speeds, offsets, cand, obj, n: int) -> None:
    """The device-pointer optimize call dereferences every tensor on speeds' device: reject
    host tensors, other devices, strided views, wrong dtypes and short buffers up front
    (the reference raises invalid_argument for malformed input, optimizer.hpp:65-66)."""
    import torch
    if speeds.dtype != torch.float64:
        raise ValueError("speeds must be float64")
    if offsets.dtype not in (torch.int32, torch.uint32):
        raise ValueError("offsets must be int32/uint32")
    if cand.dtype != torch.uint8 or obj.dtype != torch.float64:
        raise ValueError("cand must be uint8 and obj float64")
    for name, t in (("speeds", speeds), ("offsets", offsets), ("cand", cand), ("obj", obj)):
        if not _is_torch_cuda(t) or t.device != speeds.device:
            raise ValueError(f"{name} must be a CUDA tensor on {speeds.device}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if cand.numel() < n or obj.numel() < n:
        raise ValueError(f"cand/obj hold fewer than {n} instances")
    if speeds.numel() % 5:
        raise ValueError("speeds must hold 5 kind speeds per job")


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
            _check_device_args(speeds, offsets, cand, obj, n)
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

    def optimize_batches(self, batches, stream=None):
        """miso_b200_optimize_batches: several independent device batches, each a tuple
        (speeds, offsets, cand, obj) of CUDA tensors as optimize_batch takes them, in one
        stream-ordered call (up to 32 batches per persistent launch). `batches` may also be a
        BatchList prepared once (checked descriptors, reusable across calls)."""
        import torch
        bl = batches if isinstance(batches, BatchList) else BatchList(batches)
        if not bl.n:
            return
        s = stream if stream is not None else torch.cuda.current_stream(bl.device).cuda_stream
        _check(lib.miso_b200_optimize_batches(self._h, C.cast(bl.arr, C.c_void_p), bl.n, s))

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


def _dev(x, dtype, device):
    """torch tensor on `device` (copies numpy/host tensors)."""
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x)).to(device=device, dtype=dtype).contiguous()


def _ptr(t):
    return None if t is None else t.data_ptr()


def default_model():
    """fit_small_slice_model(make_training_corpus(3000, 0x5eed)) weights (w2, w1)."""
    w2 = np.zeros(4)
    w1 = np.zeros(4)
    _check(lib.miso_b200_default_model(w2.ctypes.data, w1.ctypes.data))
    return w2, w1


def _predict_batch(self, truth3, cols_per_group, first_nonce, rng_seed, mode, target_mae,
                   w2=None, w1=None, out=None, stream=None):
    """Batched predict_mig_speeds + extrapolate_small_slices; returns a (ncols, 5) tensor
    (kind order 1g..7g) on the context's device."""
    import torch
    dev = torch.device("cuda", self.device)
    t = _dev(truth3, torch.float64, dev).reshape(-1)
    ncols = t.numel() // 3
    if out is None:
        out = torch.empty(ncols * 5, dtype=torch.float64, device=dev)
    w2a = None if w2 is None else np.ascontiguousarray(w2, np.float64)
    w1a = None if w1 is None else np.ascontiguousarray(w1, np.float64)
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _check(lib.miso_b200_predict_batch(self._h, t.data_ptr(), ncols, cols_per_group, first_nonce,
                                       rng_seed, mode, target_mae,
                                       None if w2a is None else w2a.ctypes.data,
                                       None if w1a is None else w1a.ctypes.data,
                                       out.data_ptr(), s))
    return out.reshape(ncols, 5)


def _decide_batch(self, truth3, mem_gb, qos_kind, offsets, nonce, rng_seed, mode, target_mae,
                  want_est=False, stream=None):
    """Fused predict -> effective_speed -> optimize for n rosters (device). Returns
    (cand, obj, est5 or None) as torch tensors."""
    import torch
    dev = torch.device("cuda", self.device)
    t = _dev(truth3, torch.float64, dev).reshape(-1)
    mem = _dev(mem_gb, torch.uint8, dev)
    qos = _dev(qos_kind, torch.int8, dev)
    off = _dev(np.asarray(offsets).astype(np.int64), torch.int64, dev).to(torch.int32)
    non = _dev(np.asarray(nonce, np.uint64).view(np.int64), torch.int64, dev)
    n = off.numel() - 1
    cand = torch.empty(n, dtype=torch.uint8, device=dev)
    obj = torch.empty(n, dtype=torch.float64, device=dev)
    est = torch.empty(t.numel() // 3 * 5, dtype=torch.float64, device=dev) if want_est else None
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    _check(lib.miso_b200_decide_batch(self._h, t.data_ptr(), mem.data_ptr(), qos.data_ptr(),
                                      off.data_ptr(), non.data_ptr(), n, rng_seed, mode,
                                      target_mae, None, None, cand.data_ptr(), obj.data_ptr(),
                                      _ptr(est), s))
    return cand, obj, est


def _decide(self, jobs, nonce, rng_seed, mode=1, target_mae=0.017):
    """Config-1 chain for one roster (host pointers): jobs = [(job_id, (f7,f4,f3), mem_gb,
    qos_kind or None)]. Returns (AssignmentVector or None, est5 (m,5))."""
    m = len(jobs)
    if m < 1 or m > 7:
        raise ValueError(f"optimize_partition needs 1..7 jobs, got {m}")
    t = np.ascontiguousarray([list(j[1]) for j in jobs], np.float64)
    mem = np.ascontiguousarray([j[2] for j in jobs], np.uint8)
    qos = np.ascontiguousarray([-1 if j[3] is None else j[3] for j in jobs], np.int8)
    e = C.c_int()
    place = np.zeros(7, np.uint8)
    objv = C.c_double()
    est = np.zeros((m, 5))
    r = _check(lib.miso_b200_decide(self._h, t.ctypes.data, mem.ctypes.data, qos.ctypes.data, m,
                                    nonce, rng_seed, mode, target_mae, C.byref(e),
                                    place.ctypes.data, C.byref(objv), est.ctypes.data))
    if r == 0:
        return None, est
    counts = tuple(int(x) for x in self.catalog()[e.value])
    asg = [Assignment(jobs[i][0], int(place[i]), float(est[i, place[i]])) for i in range(m)]
    return AssignmentVector(counts, e.value, asg, objv.value), est


Context.predict_batch = _predict_batch
Context.decide_batch = _decide_batch
Context.decide = _decide


def _decide_server(self, idle_us):
    """miso_b200_decide_server: idle_us > 0 keeps a one-warp server kernel resident between
    decide() calls (exits after idle_us without a request); 0 = one launch per call."""
    _check(lib.miso_b200_decide_server(self._h, int(idle_us)))


Context.decide_server = _decide_server


def _max_spare_slice(self, min_kinds):
    """max_spare_slice_for (topology.hpp:227-252) over the context's catalog, from the table
    the device simulator reads: kind 0..4 or None."""
    k = np.ascontiguousarray(min_kinds, np.uint8)
    out = C.c_int()
    _check(lib.miso_b200_max_spare_slice(self._h, k.ctypes.data, len(k), C.byref(out)))
    return None if out.value < 0 else out.value


Context.max_spare_slice = _max_spare_slice


def host_alloc(nbytes: int):
    """Pinned host buffer (miso_b200_host_alloc) as a ctypes address; free with host_free."""
    p = C.c_void_p()
    _check(lib.miso_b200_host_alloc(nbytes, C.byref(p)))
    return p.value


def host_free(addr: int):
    lib.miso_b200_host_free(addr)


assert DEFAULT_CATALOG  # imported for callers
