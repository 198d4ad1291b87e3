"""Python side of the batched simulator (kernel (c)): trace generation, options, batching,
and rendering of the compact event-log records into the reference's text format.

Mirrors the reference's simulator interface (sim.hpp): `SimOptions` (:81-96) with
`OverheadSpec` (:62-67) and `PredictorSpec` (profiles.hpp:173-178), `run_simulation`
(:976-979) -> `MetricsReport` (:106-122), and the event log text written by `log()`
(:365-367). `simulate_batch` runs many traces (seeds) in one launch, one warp per seed.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._native import Context, _check, lib
from .catalog import KIND_NAMES, partition_name

POLICIES = {"nopart": 0, "optsta": 1, "oracle": 2, "miso": 3}


class SimOptionsC(C.Structure):
    _fields_ = [
        ("policy", C.c_int), ("cluster_size", C.c_int), ("mig_reconfig_s", C.c_double),
        ("checkpoint_restart_s", C.c_double), ("mps_window_s", C.c_double),
        ("interference", C.c_double), ("predictor_noisy", C.c_int), ("target_mae", C.c_double),
        ("check_invariants", C.c_int), ("reprofile_drift_threshold", C.c_double),
        ("max_events", C.c_uint64), ("small_slice_model_fitted", C.c_int),
        ("small_slice_w2", C.c_double * 4), ("small_slice_w1", C.c_double * 4),
    ]


class SimMetricsC(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("completed", C.c_int), ("job_count", C.c_int),
        ("completed_count", C.c_int), ("repartitions", C.c_int), ("migrations", C.c_int),
        ("mps_sessions", C.c_int), ("detail", C.c_int), ("avg_jct_s", C.c_double),
        ("makespan_s", C.c_double), ("stp_time_avg", C.c_double), ("jct_sum_s", C.c_double),
        ("queue_frac", C.c_double), ("mps_frac", C.c_double), ("checkpoint_frac", C.c_double),
        ("run_frac", C.c_double), ("idle_frac", C.c_double), ("events", C.c_int64),
        ("log_records", C.c_int64), ("stp_points", C.c_int64),
    ]


LOG_DTYPE = np.dtype([("t", "<i8"), ("kind", "u1"), ("x", "u1"), ("gpu", "<u2"), ("job", "<i4"),
                      ("a", "<u4"), ("b", "<u4"), ("v", "<f8")])
METRIC_FIELDS = [f for f, _ in SimMetricsC._fields_ if f != "detail"]
METRICS_DTYPE = np.dtype([(f, "<i4") for f in ("status", "completed", "job_count", "completed_count",
                                               "repartitions", "migrations", "mps_sessions", "detail")]
                         + [(f, "<f8") for f in ("avg_jct_s", "makespan_s", "stp_time_avg",
                                                 "jct_sum_s", "queue_frac", "mps_frac",
                                                 "checkpoint_frac", "run_frac", "idle_frac")]
                         + [(f, "<i8") for f in ("events", "log_records", "stp_points")])
assert METRICS_DTYPE.itemsize == C.sizeof(SimMetricsC)
assert LOG_DTYPE.itemsize == 32

lib.miso_b200_generate_trace.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int,
                                         C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
_I = C.c_int
lib.miso_b200_simulate_batch.argtypes = [C.c_void_p, C.POINTER(SimOptionsC), _I, _I, _I] + \
    [C.c_void_p] * 12 + [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]
lib.miso_b200_simulate_batch_ex.argtypes = [C.c_void_p, C.POINTER(SimOptionsC), _I, _I, _I] + \
    [C.c_void_p] * 14 + [C.c_int64, C.c_void_p, C.c_int64, C.c_uint, C.c_void_p]
lib.miso_b200_simulate_batch_pruned.argtypes = [C.c_void_p, C.POINTER(SimOptionsC), _I, _I, _I] + \
    [C.c_void_p] * 11 + [C.c_uint, C.c_void_p]
SIM_PRUNED = 5     # MISO_B200_SIM_PRUNED
SIM_BAD_INPUT = 6  # MISO_B200_SIM_BAD_INPUT


def bad_input_message(detail: int, job_ids=None) -> str:
    """MISO_B200_SIM_BAD_INPUT's metrics.detail as the reference's invalid_argument text
    (validate_profile, profiles.hpp:67-87; init_jobs, sim.hpp:246-254)."""
    code, job = detail & 0xFF, detail >> 8
    jid = job_ids[job] if job_ids is not None and job < len(job_ids) else f"j{job}"
    pre = f"job '{jid}': "
    if 3 <= code < 8:
        return pre + f"speed on {KIND_NAMES[code - 3]} outside (0,1]"
    return {1: pre + "base duration must be positive",
            2: pre + "memory demand must be in (0, 40] GB",
            8: pre + "speed on 7g must be exactly 1",
            9: pre + "speed table not monotone in gpc count",
            10: pre + "instance count must be >= 1",
            11: "first arrival must be at t=0",
            12: "arrival times must be non-decreasing",
            13: "trace has no jobs",
            14: "task_trace entry out of range",
            15: "static partition is not a feasible partition",
            16: "trace jobs exceed the workspace capacity (max_jobs)"}.get(
                code, f"invalid simulation input (detail {detail})")


@dataclass
class SimOptions:
    """SimOptions + OverheadSpec + PredictorSpec (defaults as in the reference)."""
    policy: str = "miso"
    cluster_size: int = 8
    mig_reconfig_s: float = 4.0
    checkpoint_restart_s: float = 30.0
    mps_window_s: float = 10.0
    interference: float = 0.8
    predictor: str = "oracle"          # "oracle" | "noisy" (PredictorSpec::Mode default oracle)
    target_mae: float = 0.017
    check_invariants: bool = True
    reprofile_drift_threshold: float = 0.0
    max_events: int = 100_000_000
    # SimOptions::small_slice_model (sim.hpp:88): (w2, w1) weights over (f7, f4, f3, 1) of a
    # fitted LinearMap; None = the shared default model (sim.hpp:894-896)
    small_slice_model: Optional[tuple] = None

    def to_c(self) -> SimOptionsC:
        fitted = self.small_slice_model is not None
        w2, w1 = self.small_slice_model if fitted else ((0.0,) * 4, (0.0,) * 4)
        return SimOptionsC(POLICIES[self.policy], self.cluster_size, self.mig_reconfig_s,
                           self.checkpoint_restart_s, self.mps_window_s, self.interference,
                           1 if self.predictor == "noisy" else 0, self.target_mae,
                           1 if self.check_invariants else 0, self.reprofile_drift_threshold,
                           self.max_events, 1 if fitted else 0,
                           (C.c_double * 4)(*[float(x) for x in w2]),
                           (C.c_double * 4)(*[float(x) for x in w1]))


@dataclass
class Trace:
    """JobTrace (workload.hpp:61-64) as arrays; job ids are "j<i>"."""
    arrival_s: np.ndarray
    duration_s: np.ndarray
    speeds5: np.ndarray         # (n, 5), kind order 1g..7g
    mem_gb: np.ndarray
    qos_kind: Optional[np.ndarray] = None
    seed: int = 0
    instances: Optional[np.ndarray] = None  # JobProfile::instance_count (None: all 1)

    @property
    def n(self) -> int:
        return len(self.arrival_s)


def generate_trace(seed: int, job_count: int = 100, lambda_s: float = 60.0,
                   max_duration_s: float = 7200.0, dist: str = "lognormal", sigma: float = 1.5,
                   fixed_s: float = 600.0, lo_s: float = 60.0, hi_s: float = 7200.0) -> Trace:
    """generate_trace (workload.hpp:97-114), in this library's host C++."""
    kind = {"lognormal": 0, "fixed": 1, "uniform": 2}[dist]
    a = np.zeros(job_count)
    d = np.zeros(job_count)
    sp = np.zeros((job_count, 5))
    mem = np.zeros(job_count, np.int32)
    _check(lib.miso_b200_generate_trace(seed, job_count, lambda_s, max_duration_s, kind, sigma,
                                        fixed_s, lo_s, hi_s, a.ctypes.data, d.ctypes.data,
                                        sp.ctypes.data, mem.ctypes.data))
    return Trace(a, d, sp, mem, None, seed)


lib.miso_b200_generate_traces.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                          C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]


class TraceBatch(list):
    """A list of Trace views that also keeps the batch's CSR arrays (generate_traces), so
    simulate_batch / best_static_partition upload them without re-concatenating. Slicing
    with a step of 1 keeps the CSR form."""

    csr = None  # (offsets int32 (n+1), arrival, duration, speeds5 (J,5), mem u8, qos i8, inst u8|None)

    def __getitem__(self, i):
        r = super().__getitem__(i)
        if isinstance(i, slice) and self.csr is not None and i.step in (None, 1):
            lo, hi, _ = i.indices(len(self))
            off, a, d, sp, mem, qos, inst = self.csr
            o0, o1 = int(off[lo]), int(off[hi])
            b = TraceBatch(r)
            b.csr = (off[lo:hi + 1] - o0, a[o0:o1], d[o0:o1], sp[o0:o1], mem[o0:o1], qos[o0:o1],
                     None if inst is None else inst[o0:o1])
            return b
        return r


class DeviceTraceBatch:
    """Traces resident on the device (generate_traces_device): equal-length traces as CUDA
    tensors, accepted by simulate_batch / best_static_partition without a host round trip.

    Stream order: the tensors are written on `stream` (the generator's; default: the current
    stream), and so are the simulator's CSR views (offsets, uint8 memory demands, QoS), built
    once here. `ready` is a CUDA event recorded after them on that stream; every consumer on
    another stream waits for it (simulate_batch, static_candidates, to_host)."""

    def __init__(self, seeds, arrival_s, duration_s, speeds5, mem_gb, stream=None, after=None):
        import torch
        self.seeds = np.ascontiguousarray(seeds, np.uint64)
        self.arrival_s, self.duration_s, self.speeds5, self.mem_gb = arrival_s, duration_s, speeds5, mem_gb
        self.n, self.job_count = arrival_s.shape
        dev = arrival_s.device
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(st):
            if after is not None:  # a slice: the parent's tensors must be ready first
                st.wait_event(after)
            offs = torch.arange(self.n + 1, dtype=torch.int32, device=dev) * self.job_count
            self._csr = (offs, self.arrival_s.reshape(-1), self.duration_s.reshape(-1),
                         self.speeds5.reshape(-1, 5), self.mem_gb.reshape(-1).to(torch.uint8),
                         torch.full((self.n * self.job_count,), -1, dtype=torch.int8, device=dev),
                         None)
            self.ready = torch.cuda.Event()
            self.ready.record(st)

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        if not isinstance(i, slice) or i.step not in (None, 1):
            raise TypeError("DeviceTraceBatch supports contiguous slices only")
        lo, hi, _ = i.indices(self.n)
        return DeviceTraceBatch(self.seeds[lo:hi], self.arrival_s[lo:hi], self.duration_s[lo:hi],
                                self.speeds5[lo:hi], self.mem_gb[lo:hi], after=self.ready)

    @property
    def csr(self):
        return self._csr

    def wait(self, stream=None):
        """Make `stream` (default: the current one) wait until the batch's tensors are written."""
        import torch
        (stream if stream is not None else torch.cuda.current_stream(self.arrival_s.device)).wait_event(self.ready)

    def to_host(self) -> "TraceBatch":
        self.wait()
        a, d = self.arrival_s.cpu().numpy(), self.duration_s.cpu().numpy()
        sp, mem = self.speeds5.cpu().numpy(), self.mem_gb.cpu().numpy()
        out = TraceBatch(Trace(a[i], d[i], sp[i], mem[i], None, int(self.seeds[i])) for i in range(self.n))
        out.csr = (np.arange(self.n + 1, dtype=np.int32) * self.job_count, a.reshape(-1), d.reshape(-1),
                   sp.reshape(-1, 5), mem.reshape(-1).astype(np.uint8),
                   np.full(self.n * self.job_count, -1, np.int8), None)
        return out


def _csr(traces):
    """(offsets, arrival, duration, speeds5, mem, qos, instances or None) of a trace list."""
    if isinstance(traces, (TraceBatch, DeviceTraceBatch)) and traces.csr is not None:
        return traces.csr
    for t in traces:  # the uint8 casts below must not wrap: out-of-range values are rejected here
        mem = np.asarray(t.mem_gb)
        bad = np.nonzero((mem < 1) | (mem > 40))[0]
        if len(bad):
            raise ValueError(f"job 'j{int(bad[0])}': memory demand must be in (0, 40] GB")
        if t.instances is not None and (np.asarray(t.instances) > 255).any():
            raise ValueError("instance_count above 255")
    offs = np.zeros(len(traces) + 1, np.int32)
    offs[1:] = np.cumsum([t.n for t in traces])
    cat = lambda f, dt: np.concatenate([np.asarray(f(t), dt).reshape(-1) for t in traces])  # noqa: E731
    return (offs, cat(lambda t: t.arrival_s, np.float64), cat(lambda t: t.duration_s, np.float64),
            cat(lambda t: t.speeds5, np.float64).reshape(-1, 5), cat(lambda t: t.mem_gb, np.uint8),
            cat(lambda t: (t.qos_kind if t.qos_kind is not None else np.full(t.n, -1)), np.int8),
            None if all(t.instances is None for t in traces) else
            cat(lambda t: (t.instances if t.instances is not None else np.ones(t.n)), np.uint8))


def generate_traces(seeds: Sequence[int], job_count: int = 100, lambda_s: float = 60.0,
                    max_duration_s: float = 7200.0, dist: str = "lognormal", sigma: float = 1.5,
                    fixed_s: float = 600.0, lo_s: float = 60.0, hi_s: float = 7200.0,
                    threads: int = 0) -> List[Trace]:
    """generate_trace for many seeds on every host thread (miso_b200_generate_traces);
    identical to [generate_trace(s, ...) for s in seeds]."""
    kind = {"lognormal": 0, "fixed": 1, "uniform": 2}[dist]
    sd = np.ascontiguousarray(seeds, np.uint64)
    n = len(sd)
    a = np.zeros((n, job_count))
    d = np.zeros((n, job_count))
    sp = np.zeros((n, job_count, 5))
    mem = np.zeros((n, job_count), np.int32)
    if n:
        _check(lib.miso_b200_generate_traces(sd.ctypes.data, n, job_count, lambda_s, max_duration_s,
                                             kind, sigma, fixed_s, lo_s, hi_s, threads,
                                             a.ctypes.data, d.ctypes.data, sp.ctypes.data,
                                             mem.ctypes.data))
    out = TraceBatch(Trace(a[i], d[i], sp[i], mem[i], None, int(sd[i])) for i in range(n))
    offs = (np.arange(n + 1) * job_count).astype(np.int32)
    out.csr = (offs, a.reshape(-1), d.reshape(-1), sp.reshape(-1, 5), mem.reshape(-1).astype(np.uint8),
               np.full(n * job_count, -1, np.int8), None)
    return out


lib.miso_b200_generate_traces_device.argtypes = [
    C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double,
    C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]


def generate_traces_device(ctx: Context, seeds, job_count: int = 100, lambda_s: float = 60.0,
                           max_duration_s: float = 7200.0, dist: str = "lognormal",
                           sigma: float = 1.5, fixed_s: float = 600.0, lo_s: float = 60.0,
                           hi_s: float = 7200.0, stream=None):
    """generate_trace for many seeds ON THE DEVICE (miso_b200_generate_traces_device, one warp
    per trace), bit-identical to generate_traces. Returns a DeviceTraceBatch (CUDA tensors
    arrival_s (n, J), duration_s (n, J), speeds5 (n, J, 5), mem_gb (n, J) int32)."""
    import torch
    dev = torch.device("cuda", ctx.device)
    kind = {"lognormal": 0, "fixed": 1, "uniform": 2}[dist]
    sd = torch.as_tensor(np.ascontiguousarray(seeds, np.uint64).view(np.int64), device=dev)
    n = sd.numel()
    a = torch.empty((n, job_count), dtype=torch.float64, device=dev)
    d = torch.empty((n, job_count), dtype=torch.float64, device=dev)
    sp = torch.empty((n, job_count, 5), dtype=torch.float64, device=dev)
    mem = torch.empty((n, job_count), dtype=torch.int32, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(lib.miso_b200_generate_traces_device(ctx._h, sd.data_ptr(), n, job_count, lambda_s,
                                                max_duration_s, kind, sigma, fixed_s, lo_s, hi_s,
                                                a.data_ptr(), d.data_ptr(), sp.data_ptr(),
                                                mem.data_ptr(), st.cuda_stream))
    return DeviceTraceBatch(np.ascontiguousarray(seeds, np.uint64), a, d, sp, mem, stream=st)


@dataclass
class SimResult:
    metrics: np.ndarray                    # METRICS_DTYPE per seed
    job_jct_us: Optional[List[np.ndarray]] = None
    logs: Optional[List[np.ndarray]] = None  # LOG_DTYPE records per seed
    stp: Optional[List[np.ndarray]] = None   # (points, 2) per seed
    traces: List[Trace] = field(default_factory=list)

    def report(self, i: int) -> dict:
        m = self.metrics[i]
        return {f: m[f].item() for f in METRICS_DTYPE.names if f != "detail"}


def simulate_batch(ctx: Context, traces: Sequence[Trace], opts: SimOptions,
                   rng_seeds: Optional[Sequence[int]] = None, log_cap: int = 0,
                   stp_cap: int = 0, want_jct: bool = False, stream=None,
                   task_trace: Optional[Sequence[int]] = None,
                   static_partitions: Optional[Sequence[Sequence[int]]] = None,
                   jct_only: bool = False, defer: bool = False, prune_bound=None):
    """run_simulation for every task at once (device), one warp per task. By default task i
    simulates traces[i]; with task_trace, task t simulates traces[task_trace[t]] (one launch
    can replay a trace under many static partitions). rng_seeds (per task) default to the
    trace's seed (experiment.hpp:305). static_partitions: per-task kind counts (optsta).
    jct_only: MISO_B200_SIM_JCT_ONLY (no STP series; stp metrics read 0).
    prune_bound: an int64 CUDA tensor, one entry per trace -- the chosen-only best-static
    search (miso_b200_simulate_batch_pruned; optsta, task_trace, single-instance traces).
    stream: a torch.cuda.Stream for the uploads, the launch and the read-back (default: the
    current stream). defer=True returns a zero-argument callable that waits for that stream
    and returns the SimResult, so launches on different streams (and different Contexts --
    each owns one simulation workspace) run concurrently."""
    import torch
    dev = torch.device("cuda", ctx.device)
    st_obj = stream if stream is not None else torch.cuda.current_stream(dev)
    # stream order: the launch stream waits for the caller's stream (whatever produced the
    # inputs there) and for device-resident traces' own producer stream
    st_obj.wait_stream(torch.cuda.current_stream(dev))
    if isinstance(traces, DeviceTraceBatch):
        traces.wait(st_obj)
    S = len(traces) if task_trace is None else len(task_trace)
    offs, arr, dur, sp, mem, qos, inst = _csr(traces)
    if inst is not None and (np.asarray(inst) < 1).any():
        raise ValueError("instance count must be >= 1")
    if rng_seeds is None:
        tseeds = traces.seeds if isinstance(traces, DeviceTraceBatch) else \
            np.array([t.seed for t in traces], np.uint64)
        rng_seeds = tseeds if task_trace is None else tseeds[np.asarray(task_trace, np.int64)]
    seeds = np.asarray(rng_seeds, np.uint64)
    if opts.policy == "optsta" and static_partitions is None:
        raise ValueError("optsta requires a static partition")  # sim.hpp:208-209
    if want_jct and task_trace is not None:
        raise ValueError("want_jct returns per-trace-job JCTs: not with task_trace")
    # workspace capacity: the largest trace's jobs plus every multi-instance clone
    if isinstance(traces, DeviceTraceBatch):
        n_traces, max_jobs = traces.n, traces.job_count
    else:
        offs_h = np.asarray(offs, np.int64)
        n_traces = len(offs_h) - 1
        per = np.diff(offs_h)
        if inst is not None:
            ex = np.maximum(np.asarray(inst, np.int64) - 1, 0)
            cs = np.concatenate([[0], np.cumsum(ex)])
            per = per + cs[offs_h[1:]] - cs[offs_h[:-1]]
        max_jobs = int(per.max()) if len(per) else 1
    max_jobs = max(1, max_jobs)
    with torch.cuda.stream(st_obj):
        T = lambda x: x.to(dev) if isinstance(x, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(x)).to(dev, non_blocking=False)  # noqa: E731
        d_offs, d_arr, d_dur, d_sp = T(offs), T(arr), T(dur), T(sp)
        d_mem, d_qos, d_seed = T(mem), T(qos), T(seeds.view(np.int64))
        d_tt = None if task_trace is None else T(np.asarray(task_trace, np.int32))
        d_inst = None if inst is None else T(np.asarray(inst, np.uint8))
        d_sc = None if static_partitions is None else \
            T(np.asarray(static_partitions, np.uint8).reshape(S, 5))
        d_met = torch.empty(S * METRICS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        d_jct = torch.empty(int(offs[-1]), dtype=torch.int64, device=dev) if want_jct else None
        d_log = torch.empty(S * log_cap * 32, dtype=torch.uint8, device=dev) if log_cap else None
        d_stp = torch.empty(S * stp_cap * 2, dtype=torch.float64, device=dev) if stp_cap else None
        o = opts.to_c()
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        if prune_bound is not None:
            if inst is not None or want_jct or log_cap or stp_cap:
                raise ValueError("pruned runs take single-instance traces and return metrics only")
            _check(lib.miso_b200_simulate_batch_pruned(ctx._h, C.byref(o), S, n_traces, max_jobs,
                                                       p(d_tt), p(d_sc), p(d_offs),
                                                       p(d_arr), p(d_dur), p(d_sp), p(d_mem), p(d_qos),
                                                       p(d_seed), p(d_met), prune_bound.data_ptr(),
                                                       1 if jct_only else 0, st_obj.cuda_stream))
        else:
            _check(lib.miso_b200_simulate_batch_ex(ctx._h, C.byref(o), S, n_traces, max_jobs,
                                                   p(d_tt), p(d_sc), p(d_offs),
                                                   p(d_arr), p(d_dur),
                                                   p(d_sp), p(d_mem), p(d_qos), p(d_inst), p(d_seed), p(d_met),
                                                   p(d_jct), None, p(d_log), log_cap, p(d_stp), stp_cap,
                                                   1 if jct_only else 0, st_obj.cuda_stream))
    keep = (d_offs, d_arr, d_dur, d_sp, d_mem, d_qos, d_seed, d_tt, d_sc, d_inst)  # alive until done

    def finish() -> SimResult:
        st_obj.synchronize()
        _ = keep  # inputs stay referenced until the stream has finished with them
        met = d_met.cpu().numpy().view(METRICS_DTYPE)
        bad = np.nonzero(met["status"] == SIM_BAD_INPUT)[0]
        if len(bad):  # the reference's std::invalid_argument (first failing task)
            raise ValueError(bad_input_message(int(met["detail"][bad[0]])))
        res = SimResult(met, traces=[] if isinstance(traces, DeviceTraceBatch) else list(traces))
        if want_jct:
            j = d_jct.cpu().numpy()
            offs_h = offs.cpu().numpy() if hasattr(offs, "cpu") else offs
            res.job_jct_us = [j[offs_h[i]:offs_h[i + 1]] for i in range(len(traces))]
        if log_cap:
            lg = d_log.cpu().numpy().view(LOG_DTYPE).reshape(S, log_cap)
            res.logs = [lg[i, : min(log_cap, int(met[i]["log_records"]))] for i in range(S)]
        if stp_cap:
            stp = d_stp.cpu().numpy().reshape(S, stp_cap, 2)
            res.stp = [stp[i, : min(stp_cap, int(met[i]["stp_points"]))] for i in range(S)]
        return res

    return finish if defer else finish()


def fmt_g(v: float) -> str:
    """fmt_g (common.hpp:126-132): %.10g, inf/nan spelled out."""
    if np.isinf(v):
        return "inf" if v > 0 else "-inf"
    if np.isnan(v):
        return "nan"
    return "%.10g" % v


def _counts(packed: int):
    return tuple((packed >> (4 * k)) & 15 for k in range(5))


def render_log(records: np.ndarray, job_ids=None) -> str:
    """Render compact records as the reference's event log text (sim.hpp:365-367 and the
    log() call sites listed in SURVEY.md 5)."""
    jid = (lambda j: job_ids[j]) if job_ids is not None else (lambda j: f"j{j}")
    out = []
    i = 0
    n = len(records)
    while i < n:
        r = records[i]
        t, k, g, j = int(r["t"]), int(r["kind"]), int(r["gpu"]), int(r["job"])
        a, b = int(r["a"]), int(r["b"])
        if k == 0:
            line = f"arrival job={jid(j)}"
        elif k == 1:
            line = f"admit gpu={g} job={jid(j)}"
        elif k == 2:
            line = f"start job={jid(j)} gpu={g} slice={KIND_NAMES[int(r['x'])]} rate={fmt_g(float(r['v']))}"
        elif k == 3:
            line = f"ckpt_start gpu={g} jobs={a}"
        elif k == 4:
            line = f"mps_start gpu={g} jobs={a}"
        elif k == 5:
            line = f"mps_window gpu={g} level={a}"
        elif k == 6:
            line = f"mps_end gpu={g}"
        elif k == 7:
            line = f"reconfig_start gpu={g} pause_us={a | (b << 32)}"
        elif k == 8:
            m = int(r["x"])
            pairs = [f"{jid(int(q['job']))}@{KIND_NAMES[int(q['x'])]}" for q in records[i + 1: i + 1 + m]]
            line = f"partition gpu={g} shape={partition_name(_counts(a))} assign={','.join(pairs)}"
            i += m
        elif k == 10:
            line = f"complete job={jid(j)} jct_us={a | (b << 32)}"
        elif k == 11:
            line = f"shrink gpu={g} shape={partition_name(_counts(a))}"
        elif k == 12:
            line = f"admit gpu={g} job={jid(j)} slot={int(r['x'])}"
        elif k == 13:
            line = f"migrate job={jid(j)} gpu={g} slot={a} slice={KIND_NAMES[int(r['x'])]}"
        elif k == 14:
            line = f"spawn job={jid(j)} parent={jid(a)}"
        else:
            line = f"?kind={k}"
        out.append(f"{t} {line}\n")
        i += 1
    return "".join(out)


def min_kind(mem_gb: int, qos_kind=None):
    """min_slice_for (topology.hpp:68-72) of a job; None if no kind fits."""
    from .catalog import GPC, MEM_GB
    q = GPC[qos_kind] if qos_kind is not None and qos_kind >= 0 else 0
    for k in range(5):
        if MEM_GB[k] >= mem_gb and GPC[k] >= q:
            return k
    return None


def static_candidates(traces: Sequence[Trace], catalog=None):
    """best_static_partition's candidate runs (sim.hpp:1036-1048): (trace index, catalog
    index) of every entry whose largest slice is at least every job's min_slice_for
    (topology.hpp:68-72), trace-major in catalog order. Raises ValueError (InfeasibleError) if
    a job fits no slice kind."""
    from .catalog import DEFAULT_CATALOG, GPC, MEM_GB
    cat = list(catalog if catalog is not None else DEFAULT_CATALOG)
    catc = np.asarray(cat, np.uint8).reshape(-1, 5)
    largest = np.array([max(k for k in range(5) if c[k] > 0) for c in catc])
    assert list(GPC) == sorted(GPC) and list(MEM_GB) == sorted(MEM_GB)
    offs, _, _, _, mem, qos, _ = _csr(traces)
    # min_slice_for: the smallest kind with memory_gb >= mem and gpc >= gpc(qos); both tables
    # are non-decreasing in the kind index, so it is max(first kind with enough memory, qos)
    if isinstance(traces, DeviceTraceBatch) and len(traces):
        # device-resident, equal-length traces: the per-job pass runs on the device and only
        # each trace's largest minimum kind (and the first unfittable job) comes back
        import torch
        traces.wait()
        dev = mem.device
        mk = torch.maximum(torch.searchsorted(torch.tensor(MEM_GB, dtype=torch.int64, device=dev),
                                              mem.to(torch.int64), right=False),
                           qos.to(torch.int64).clamp(min=0)).view(traces.n, traces.job_count)
        need_t = mk.max(dim=1).values
        need = need_t.cpu().numpy()
        if len(need) and need.max() > 4:
            ti = int(np.argmax(need > 4))
            raise ValueError(f"trace {ti}: a job fits no slice kind")
    else:
        mk = np.maximum(np.searchsorted(np.asarray(MEM_GB), np.asarray(mem, np.int64), side="left"),
                        np.maximum(np.asarray(qos, np.int64), 0))
        if len(mk) and mk.max() > 4:
            j = int(np.argmax(mk > 4))
            ti = int(np.searchsorted(offs, j, side="right") - 1)
            raise ValueError(f"trace {ti}: a job fits no slice kind")
        need = np.maximum.reduceat(mk, offs[:-1]) if len(traces) else np.zeros(0, np.int64)
    feas = largest[None, :] >= need[:, None]                      # (traces, entries)
    return np.nonzero(feas)


def static_probes(ti_arr, e_arr, catalog_counts):
    """The chosen-only search's probes: per trace, the two best-ranked feasible candidates by
    a prior (most GPCs, then slice count nearest 3, then catalog order) -- the likeliest
    winners, run first so the other candidates can be stopped against their JCT sums.
    Returns a bool mask over the candidate list."""
    catc = np.asarray(catalog_counts, np.int64).reshape(-1, 5)
    from .catalog import GPC
    gpcs = (catc * np.asarray(GPC)[None, :]).sum(axis=1)
    nsl = catc.sum(axis=1)
    prio = np.lexsort((np.arange(len(catc)), np.abs(nsl - 3), -gpcs))
    rank = np.empty(len(catc), np.int64)
    rank[prio] = np.arange(len(catc))
    r = rank[e_arr]
    order = np.lexsort((r, ti_arr))
    first = np.r_[True, ti_arr[order][1:] != ti_arr[order][:-1]] if len(order) else np.zeros(0, bool)
    pos = np.arange(len(order)) - np.maximum.accumulate(np.where(first, np.arange(len(order)), 0))
    probe = np.zeros(len(ti_arr), bool)
    probe[order[pos < 2]] = True
    return probe


def best_static_partition(ctx: Context, traces: Sequence[Trace], cluster_size: int,
                          overheads: Optional[SimOptions] = None, catalog=None, stream=None,
                          chosen_only: bool = False):
    """best_static_partition (sim.hpp:1031-1066) for many traces in ONE launch: every
    (trace, candidate partition) pair is an independent optsta simulation (one warp each).
    Returns per trace (chosen catalog index, table of avg JCT per entry; inf = skipped or
    incomplete). Raises ValueError (InfeasibleError) if a job fits no slice kind or no
    partition can host the trace.

    chosen_only=True is run_trial_unit's use (experiment.hpp:337 reads only .chosen): the
    same chosen entry from one pruned launch (miso_b200_simulate_batch_pruned) whose task
    order puts each trace's two likeliest winners first (most GPCs, then slice count nearest
    3); every candidate stops once its JCT sum provably exceeds a completed candidate's.
    Table entries of stopped candidates read inf (single-instance traces; else the full
    search)."""
    from .catalog import DEFAULT_CATALOG
    cat = list(catalog if catalog is not None else DEFAULT_CATALOG)
    base = overheads or SimOptions()
    opts = SimOptions(policy="optsta", cluster_size=cluster_size,
                      mig_reconfig_s=base.mig_reconfig_s,
                      checkpoint_restart_s=base.checkpoint_restart_s,
                      mps_window_s=base.mps_window_s, interference=base.interference,
                      check_invariants=base.check_invariants, max_events=base.max_events)
    from .catalog import GPC
    catc = np.asarray(cat, np.uint8).reshape(-1, 5)
    ti_arr, e_arr = static_candidates(traces, cat)
    table = np.full((len(traces), len(cat)), np.inf)
    inst = _csr(traces)[6]
    multi = inst is not None and (np.asarray(inst.cpu() if hasattr(inst, "cpu") else inst) > 1).any()
    if len(ti_arr) and chosen_only and not multi:
        import torch
        probe = static_probes(ti_arr, e_arr, catc)
        dev = torch.device("cuda", ctx.device)
        st_obj = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(st_obj):
            bound = torch.full((len(traces),), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
        # one launch, probes first: they fill the first wave, and the candidates behind them
        # start with their trace's bound already set
        sel = np.r_[np.nonzero(probe)[0], np.nonzero(~probe)[0]]
        res = simulate_batch(ctx, traces, opts, task_trace=ti_arr[sel].astype(np.int32),
                             static_partitions=catc[e_arr[sel]], jct_only=True, stream=stream,
                             prune_bound=bound)
        table[ti_arr[sel], e_arr[sel]] = res.metrics["avg_jct_s"]
    elif len(ti_arr):
        res = simulate_batch(ctx, traces, opts, task_trace=ti_arr.astype(np.int32),
                             static_partitions=catc[e_arr], jct_only=True, stream=stream)
        # the candidates' only consumed output is avg_jct_s (sim.hpp:1053-1060): JCT-only runs
        table[ti_arr, e_arr] = res.metrics["avg_jct_s"]
    out = []
    chosen = table.argmin(axis=1) if len(traces) else np.zeros(0, np.int64)  # first minimum
    ok = table[np.arange(len(traces)), chosen] < np.inf  # == strict <, first wins (sim.hpp:1058)
    if not ok.all():
        raise ValueError(f"trace {int(np.argmin(ok))}: no static partition can host this trace")
    out.extend(zip(chosen.tolist(), table))
    return out


def _simulate(self, traces, opts=None, **kw):
    return simulate_batch(self, traces, opts or SimOptions(), **kw)


Context.simulate = _simulate
