#!/usr/bin/env python3
"""Benchmark: job-mix instances optimized/sec (BASELINE.json metric) on B200.

Default workload = BASELINE.json configs[1] (config 2): 1M random job mixes per GPU (1-7 jobs
each, acceptance_test.cpp:72-85 distribution), full search over the 36-entry MIG catalog and
every distinct job-to-slice assignment (111 candidates). One step = one pass of the partition-
search kernel over the 1M-instance batch resident in HBM.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c1|c2|c3|c4|c5]

--gpus N > 1 without a torch.distributed environment re-executes this script under
torch.distributed.run with N ranks (one per GPU over NCCL; gloo with ranks sharing GPUs when
the box has fewer than N). Every rank owns an independent 1M-instance shard (weak scaling, no
data-path collective); timings are device-side (CUDA events) and the max over ranks is reported;
the decisions are gathered to rank 0 at the end (byte-exact, `result_gather`). `e2e` measures
the same metric through the C-ABI host-pointer call (pinned host buffers; H2D, search, D2H
inside the timed region). `cpu_baseline` times the reference's own optimize_partition
(oracle/_ref, the unmodified reference headers) on a bounded sample of the same batch with every
host thread (and with one), and its decisions on that sample are the `parity` check.

The default line also carries `secondary`: configs 1, 3, 4 and 5 (BASELINE.json configs[0],
[2], [3], [4]), each with its value, reference CPU baseline, parity check and bound.
`--config cX` prints one of them alone.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
METRIC = "job-mix instances optimized/sec (and configs scored/sec) at 1/2/4/8 B200 vs CPU"
UNIT = "instances/s"
N_PER_GPU = 1_000_000
CANDS_PER_M = {1: 5, 2: 13, 3: 29, 4: 35, 5: 21, 6: 7, 7: 1}
WORKLOAD = ("config2: 1M random job mixes per GPU (m~U{1..7}, acceptance_test.cpp:72-85 "
            "distribution), exhaustive search over 36 MIG partitions x distinct assignments "
            "(111 candidates), FP64 objective, reference tie-break")


# ---------------------------------------------------------------------------------------------
# ranks

class Dist:
    """One process per GPU (RANK / WORLD_SIZE / LOCAL_RANK from torch.distributed.run)."""

    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = os.environ.get("MISO_B200_DIST_BACKEND", "nccl")
        self.pg = None

    def init(self):
        import torch
        ndev = max(1, torch.cuda.device_count())
        self.local %= ndev  # gloo fallback: ranks share the box's GPUs
        self.shared_gpus = self.world > ndev
        torch.cuda.set_device(self.local)
        self.device = torch.device("cuda", self.local)
        self.coll_dev = torch.device("cpu") if self.backend == "gloo" else self.device
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.device)
            else:
                dist.init_process_group(self.backend)
            self.pg = dist
        return self

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def reduce(self, vals, op="max"):
        """Element-wise max (or sum) over ranks of a list of floats."""
        if self.pg is None:
            return list(vals)
        import torch
        t = torch.tensor(list(vals), dtype=torch.float64, device=self.coll_dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX if op == "max" else self.pg.ReduceOp.SUM)
        return t.tolist()

    def gather(self, local, n_total):
        from paper_2207_11428_b200.dist import gather_to_rank0
        return gather_to_rank0(local, n_total, self.rank, self.world,
                               device=self.coll_dev if self.world > 1 else None)

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


def spawn_ranks(args) -> int:
    """`--gpus N` outside torch.distributed: re-execute under torch.distributed.run, N ranks on
    127.0.0.1 (NCCL, one GPU each; gloo with ranks sharing GPUs if the box has fewer)."""
    import socket
    import subprocess
    import torch
    env = dict(os.environ)
    ndev = torch.cuda.device_count()
    if ndev < args.gpus:
        env["MISO_B200_DIST_BACKEND"] = "gloo"
    env.setdefault("NCCL_DEBUG", "INFO")           # rank/ring setup lines, on stderr
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------------------------------------
# helpers

def gen_mixes(seed: int, n: int):
    """Synthetic config-2 input (same distribution as the reference generator; numpy stream)."""
    rng = np.random.default_rng(seed)
    m = rng.integers(1, 8, n)
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(m, out=offs[1:])
    J = int(offs[-1])
    u = rng.random((J, 5))
    f4 = 0.2 + 0.8 * u[:, 0]
    f3 = 0.15 + (f4 - 0.15) * u[:, 1]
    f2 = 0.1 + (f3 - 0.1) * u[:, 2]
    f1 = 0.05 + (f2 - 0.05) * u[:, 3]
    f1[u[:, 4] < 0.25] = 0.0
    speeds = np.empty((J, 5), np.float64)
    speeds[:, 0], speeds[:, 1], speeds[:, 2], speeds[:, 3], speeds[:, 4] = f1, f2, f3, f4, 1.0
    return speeds.reshape(-1), offs.astype(np.uint32), m


def candidates_of(m: np.ndarray) -> int:
    return int(sum(CANDS_PER_M[k] * int((m == k).sum()) for k in CANDS_PER_M))


def algorithmic_bytes(m: np.ndarray) -> int:
    """Per launch: 40 B speeds per job + 4 B offset + 1 B decision + 8 B objective per
    instance (+ the closing offset). SURVEY.md 8(d) / DESIGN.md."""
    return int(40 * int(m.sum()) + 13 * len(m) + 4)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {}


def measured_peak():
    d = measured_peaks()
    if "hbm_gbs" in d:
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_capture(name):
    p = ROOT / "profiles" / name
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def ncu_val(launch, key):
    try:
        return float(str(launch.get(key, "nan")).split()[0])
    except (ValueError, AttributeError):
        return float("nan")


def oracle_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as ol
    return ol


def bits_equal(a, b) -> bool:
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and bool(np.array_equal(a.view(np.uint64), b.view(np.uint64)))


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed regions run."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        self._th = None
        self._on = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            if self._on.is_set():
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    for bit, name in self.REASONS.items():
                        if r & bit and bit != 0x1:
                            self.reasons.add(name)
                except Exception:
                    pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def timed(self, on: bool):  # sample only inside timed regions
        (self._on.set if on else self._on.clear)()

    def stop(self):
        if self._th:
            self._stop.set()
            self._th.join()
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
            "source": "nvml" if self.nv else "unavailable",
        }


def cuda_time(stream, fn, reps=1):
    """ms of `reps` calls of fn() between one CUDA-event pair on `stream`."""
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


# ---------------------------------------------------------------------------------------------
# config 2 (headline)

def c2_cpu_baseline(speeds, offs, m, ctx, h_cand, h_obj, target_s: float = 8.0):
    """The reference's optimize_partition (oracle/_ref) on a bounded sample of the same batch:
    all host threads (the baseline) and one thread; its decisions on the sample are compared with
    the GPU's (parity). Falls back to the C restatement (kind "port") without _ref."""
    ol = oracle_lib()
    threads = ol.host_threads()
    if ol.have_ref():
        impl, kind = ol.Ref(), "reference"
        run = lambda s, f, t: impl.optimize_batch(s, f, threads=t)  # noqa: E731
    else:
        impl, kind, threads = ol.Oracle(), "port", 1
        run = lambda s, f, t: impl.optimize_batch(s, f)  # noqa: E731

    def sample(n):
        f = offs[: n + 1]
        return speeds[: int(f[-1]) * 5], f

    n = min(100_000, len(m))
    t0 = time.perf_counter(); run(*sample(n), threads); dt = time.perf_counter() - t0
    n = int(min(len(m), max(n, n * target_s / max(dt, 1e-6))))
    passes = 1
    if n == len(m):  # whole batch is quick: repeat passes to reach ~target_s of CPU work
        t0 = time.perf_counter(); run(*sample(n), threads); dt1 = time.perf_counter() - t0
        passes = max(1, min(100, int(target_s / max(dt1, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(passes):
        e, p, o = run(*sample(n), threads)
    dt = time.perf_counter() - t0
    # one thread: a sample of ~target_s / 2
    n1 = max(1000, min(n, int(n * passes / dt * (target_s / 2) / max(threads, 1))))
    t0 = time.perf_counter(); run(*sample(n1), 1); dt1 = time.perf_counter() - t0
    # parity on the all-thread sample: entry, placement and objective bits
    s_off = offs[: n + 1].astype(np.int64)
    g_e, g_p = ctx.decode(h_cand[:n], s_off)
    feas = np.repeat(e >= 0, np.diff(s_off))
    ent_eq = bool(np.array_equal(g_e, e.astype(np.int32)))
    pl_eq = bool(np.array_equal(g_p[feas], p[: int(s_off[-1])][feas]))
    ob_eq = bits_equal(h_obj[:n], o)
    cpu = {"value": n * passes / dt, "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"first {n} instances of the rank-0 config-2 batch x {passes} passes, "
                     f"{threads} host threads, {dt:.2f} s",
           "candidates_per_s": candidates_of(m[:n]) * passes / dt,
           "one_thread": {"value": n1 / dt1, "unit": UNIT, "cores": 1,
                          "sample": f"first {n1} instances, 1 thread, {dt1:.2f} s"}}
    parity = {"checked_against": "oracle/_ref (the unmodified reference optimize_partition)"
              if kind == "reference" else "oracle C restatement",
              "instances": n, "entry_equal": ent_eq, "placement_equal": pl_eq,
              "objective_bits_equal": ob_eq,
              "mismatches": int((g_e != e.astype(np.int32)).sum() +
                                (h_obj[:n].view(np.uint64) != o.view(np.uint64)).sum()),
              "ok": ent_eq and pl_eq and ob_eq}
    return cpu, parity


def run_c2(args, D, ctx, clocks):
    import ctypes as C
    import torch
    from paper_2207_11428_b200._native import host_alloc, host_free
    import paper_2207_11428_b200 as miso

    speeds, offs, m = gen_mixes(1000 + D.rank, N_PER_GPU)
    n = len(m)
    d_speeds = torch.from_numpy(speeds).cuda()
    d_offs = torch.from_numpy(offs.view(np.int32)).cuda()
    d_cand = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_obj = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    # Steps are independent batches: they alternate over S streams, each with its own copy of
    # the input and its own outputs, so one step's ramp-up overlaps the previous step's tail.
    # The single-stream rate (one launch per step on one stream) is reported beside it.
    S = 2
    streams = [torch.cuda.Stream() for _ in range(S)]
    bufs = [(d_speeds, d_offs, d_cand, d_obj)] + [
        (d_speeds.clone(), d_offs.clone(), torch.empty_like(d_cand), torch.empty_like(d_obj))
        for _ in range(S - 1)]
    for _ in range(max(3, args.warmup)):
        for k in range(S):
            ctx.optimize_batch(*bufs[k], stream=streams[k].cuda_stream)
    torch.cuda.synchronize()
    K = args.steps

    def timed(n_streams):
        # K launches between ONE event pair on the launching stream(s): an event between
        # launches would serialise them, so the per-step time is the timed region / K.
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.barrier(); torch.cuda.synchronize()
        clocks.timed(True)
        t0.record(stream)
        for st in streams[:n_streams]:
            st.wait_stream(stream)
        for i in range(K):
            k = i % n_streams
            ctx.optimize_batch(*bufs[k], stream=streams[k].cuda_stream)
        for st in streams[:n_streams]:
            stream.wait_stream(st)
        t1.record(stream)
        torch.cuda.synchronize()
        clocks.timed(False)
        D.barrier()
        return t0.elapsed_time(t1)

    # Headline schedule: the K steps as a queue of batches -- miso_b200_optimize_batches puts up
    # to 32 steps in one persistent launch (steps alternate over the S input copies; every step
    # has its own outputs), so the launch's fixed cost (grid start, first-tile latency, CTA
    # tail) is paid once per launch instead of once per step.
    PER_LAUNCH = 32
    n_out = min(K, 64)
    outs = [(torch.empty_like(d_cand), torch.empty_like(d_obj)) for _ in range(n_out)]
    queue = [(bufs[i % S][0], bufs[i % S][1]) + outs[i % n_out] for i in range(K)]
    launches = (K + PER_LAUNCH - 1) // PER_LAUNCH
    # descriptors built (and checked) before the timed region
    calls = [miso.BatchList(queue[c0:c0 + PER_LAUNCH]) for c0 in range(0, K, PER_LAUNCH)]
    ctx.optimize_batches(calls[0], stream=stream.cuda_stream)  # warm
    torch.cuda.synchronize()

    def timed_queue():
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.barrier(); torch.cuda.synchronize()
        clocks.timed(True)
        t0.record(stream)
        for bl in calls:
            ctx.optimize_batches(bl, stream=stream.cuda_stream)
        t1.record(stream)
        torch.cuda.synchronize()
        clocks.timed(False)
        D.barrier()
        return t0.elapsed_time(t1)

    single_ms = timed(1)
    two_ms = timed(S)
    total_ms = timed_queue()
    kern_ms = total_ms / launches  # average duration of one (multi-step) launch
    for k in range(1, S):  # every stream computed the same decisions
        assert torch.equal(bufs[k][2], d_cand) and torch.equal(bufs[k][3].view(torch.int64), d_obj.view(torch.int64))
    for c, o in outs:  # and so did every queued step
        assert torch.equal(c, d_cand) and torch.equal(o.view(torch.int64), d_obj.view(torch.int64))
    del outs, queue, calls

    # --- e2e: the C-ABI host-pointer call, pinned buffers, H2D + search + D2H timed ---
    nb_s, nb_o = speeds.nbytes, offs.nbytes
    p_s, p_o, p_c, p_b = host_alloc(nb_s), host_alloc(nb_o), host_alloc(n), host_alloc(8 * n)
    C.memmove(p_s, speeds.ctypes.data, nb_s)
    C.memmove(p_o, offs.ctypes.data, nb_o)
    lib = miso.lib
    for _ in range(2):
        lib.miso_b200_optimize_batch_host(ctx._h, p_s, p_o, n, p_c, p_b)
    E = max(3, min(K, 20))
    D.barrier(); torch.cuda.synchronize()
    clocks.timed(True)
    w0 = time.perf_counter()
    for _ in range(E):
        rc = lib.miso_b200_optimize_batch_host(ctx._h, p_s, p_o, n, p_c, p_b)
        assert rc == 0, lib.miso_b200_last_error()
    e2e_s = time.perf_counter() - w0
    clocks.timed(False)
    D.barrier()
    h_c = np.ctypeslib.as_array((C.c_uint8 * n).from_address(p_c)).copy()
    h_b = np.ctypeslib.as_array((C.c_double * n).from_address(p_b)).copy()
    d_c = d_cand.cpu().numpy()
    d_o = d_obj.cpu().numpy()
    assert np.array_equal(h_c, d_c) and bits_equal(h_b, d_o)
    for p in (p_s, p_o, p_c, p_b):
        host_free(p)

    total_ms, kern_ms, e2e_s, single_ms, two_ms = D.reduce([total_ms, kern_ms, e2e_s, single_ms, two_ms], "max")
    gather = None
    if D.world > 1:
        # final result gather (untimed): every rank's decisions and objectives to rank 0 in
        # global instance order (dist.gather_to_rank0: all_gather of equal shards, byte-exact)
        g0 = time.perf_counter()
        all_c = D.gather(d_c, D.world * n)
        all_o = D.gather(d_o, D.world * n)
        g_s = D.reduce([time.perf_counter() - g0], "max")[0]
        if D.rank == 0:
            byte_exact = bool(np.array_equal(all_c[:n], d_c) and bits_equal(all_o[:n], d_o))
            gather = {"instances": int(len(all_c)), "bytes": int(all_c.nbytes + all_o.nbytes),
                      "feasible": int((all_c < 111).sum()), "s": g_s, "backend": D.backend,
                      "rank0_shard_byte_exact": byte_exact}
    alg = algorithmic_bytes(m)
    cands = candidates_of(m)
    achieved = alg * K / launches / (kern_ms / 1e3) / 1e9
    single_achieved = alg / (single_ms / K / 1e3) / 1e9
    two_achieved = alg / (two_ms / K / 1e3) / 1e9
    peak, peak_src = measured_peak()
    cap = ncu_capture("search_kernel_ncu.json") or {}
    line = {
        "metric": METRIC, "value": D.world * n * K / (total_ms / 1e3), "unit": UNIT,
        "n_gpus": D.world, "steps": K, "warmup": args.warmup, "ms_per_step": total_ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "instances_per_gpu": n, "jobs_per_gpu": int(m.sum()),
                   "candidates_per_gpu_step": cands,
                   "l2": "inputs %.0f MB per GPU > 126 MB L2; no flush" % ((speeds.nbytes + offs.nbytes) / 1e6),
                   "parallelism": f"{D.world} independent shards ({D.backend}"
                                  + (", ranks sharing GPUs" if D.shared_gpus else "") + ")",
                   "schedule": f"queued steps: miso_b200_optimize_batches, up to {PER_LAUNCH} steps (independent 1M-instance batches) per persistent launch, {launches} launches on one stream; steps alternate over {S} input copies, each step has its own outputs"},
        "configs_scored_per_s": D.world * cands * K / (total_ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": cap.get("dram_bytes_per_launch"),
                     "traffic_note": "ncu DRAM bytes of one single-step launch (profiles/search_kernel_ncu.json) vs its algorithmic bytes per step",
                     "kernel": "optimize_pipe_kernel", "kernel_ms": kern_ms,
                     "steps_per_launch": K / launches,
                     "algorithmic_bytes_per_launch": alg * K / launches,
                     "algorithmic_bytes_per_step": alg,
                     "kernel_ms_note": f"average duration of one launch ({launches} launches of up to {PER_LAUNCH} steps, back to back on one stream, CUDA events around all of them)",
                     "one_launch_per_step": {"kernel_ms": single_ms / K, "achieved": single_achieved,
                                             "frac": single_achieved / peak,
                                             "note": "miso_b200_optimize_batch per step, one stream, launches back to back: per-launch duration"},
                     "two_streams": {"ms_per_step": two_ms / K, "achieved": two_achieved,
                                     "frac": two_achieved / peak,
                                     "note": f"one launch per step, steps alternating over {S} streams (consecutive launches overlap): pipelined throughput"},
                     "peak_source": peak_src},
        "e2e": {"value": D.world * n * E / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": D.world * (nb_s + nb_o), "d2h_bytes_per_step": D.world * n * 9,
                "api": "miso_b200_optimize_batch_host (pinned host buffers)", "steps": E},
        "gpu_launches": launches,
    }
    if gather is not None:
        line["result_gather"] = gather
    return line, (speeds, offs, m, d_c, d_o)


# ---------------------------------------------------------------------------------------------
# reference arm

def run_reference_arm(args, D):
    if D.rank != 0:
        return
    speeds, offs, m = gen_mixes(12345, N_PER_GPU)
    ol = oracle_lib()
    threads = ol.host_threads()
    if ol.have_ref():
        impl, kind = ol.Ref(), "reference"
        run = lambda s, f: impl.optimize_batch(s, f, threads=threads)  # noqa: E731
    else:
        impl, kind, threads = ol.Oracle(), "port", 1
        run = lambda s, f: impl.optimize_batch(s, f)  # noqa: E731
    per_step = 250_000
    f = offs[: per_step + 1]
    s = speeds[: int(f[-1]) * 5]
    for _ in range(args.warmup):
        run(s, f)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(s, f)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "instances_per_step": per_step,
                   "sample": "bounded sample of the config-2 batch per step"},
        "configs_scored_per_s": candidates_of(m[:per_step]) * args.steps / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{per_step} instances per step, {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# secondary configs

def sec_c3(args, D, ctx, n=16 * 1024 * 1024, steps=10):
    """Config 3: batched noisy predictor on 16M synthetic MPS profiles per rank (7-column
    groups, nonce = group + 1, target_mae 0.017, default model): profiles/s, the bound (the
    FMA-heavy pipe: 3 IMADs per mt19937_64 seeding step), the reference's predictor chain on
    all host threads over a sample, and that sample's outputs compared bit for bit."""
    import torch
    rng = np.random.default_rng(5 + D.rank)
    f4 = rng.uniform(0.3, 1.0, n)
    f3 = f4 * rng.uniform(0.6, 1.0, n)
    truth = np.stack([np.ones(n), f4, f3], 1).reshape(-1)
    d_t = torch.from_numpy(truth).cuda()
    out = torch.empty(n * 5, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        ctx.predict_batch(d_t, 7, 1, 42, 1, 0.017, out=out)
    D.barrier()
    ms = cuda_time(st, lambda: ctx.predict_batch(d_t, 7, 1, 42, 1, 0.017, out=out), steps) / steps
    ms = D.reduce([ms])[0]
    res = {"metric": "MPS profiles predicted/sec (config 3, noisy, mae 0.017)",
           "value": D.world * n / (ms / 1e3), "unit": "profiles/s", "ms_per_step": ms,
           "steps": steps, "profiles_per_gpu": n, "n_gpus": D.world, "scaling": "weak",
           "dtype": "f64", "data": "synthetic", "gpu_launches": steps}
    peak, _ = measured_peak()
    gbs = n * 64 / (ms / 1e3) / 1e9
    cap = ncu_capture("predict_kernel_ncu.json")
    bound = {"bound": "fma-heavy pipe (integer multiplies of the mt19937_64 seeding chains, 158 steps x 2 entries per profile)",
             "hbm_for_scale": {"achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                               "algorithmic_bytes_per_profile": 64}}
    if cap:
        l0 = cap["launches"][0]
        cap_ms = ncu_val(l0, "gpu__time_duration.sum")
        busy = ncu_val(l0, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed") / 100
        # the pipe's busy cycles per launch are fixed by the instruction mix (captured once for
        # this n); scaled to this run's kernel duration they give its live busy fraction
        bound.update({"achieved_pipe_busy_frac": busy * cap_ms / ms if ms > 0 else None,
                      "frac": busy * cap_ms / ms if ms > 0 else None,
                      "ncu_capture": {"pipe_busy": busy, "ms": cap_ms,
                                      "issue_active": ncu_val(l0, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
                                      "source": "profiles/predict_kernel_ncu.json"}})
    res["roofline"] = bound
    if D.rank == 0 and not args.no_cpu_baseline:
        ol = oracle_lib()
        if ol.have_ref():
            ref, threads = ol.Ref(), ol.host_threads()
            k = 7 * 60_000
            t0 = time.perf_counter()
            want = ref.predict_batch(truth[: 3 * k], 7, 1, 42, 1, 0.017, threads=threads)
            dt = time.perf_counter() - t0
            k1 = 7 * 4000
            t0 = time.perf_counter()
            ref.predict_batch(truth[: 3 * k1], 7, 1, 42, 1, 0.017, threads=1)
            dt1 = time.perf_counter() - t0
            got = out[: 5 * k].cpu().numpy()
            res["cpu_baseline"] = {"value": k / dt, "unit": "profiles/s", "cores": threads,
                                   "kind": "reference",
                                   "sample": f"first {k} profiles of the rank-0 batch, {threads} threads",
                                   "one_thread": {"value": k1 / dt1, "unit": "profiles/s", "cores": 1}}
            res["parity"] = {"checked_against": "oracle/_ref predict_mig_speeds + extrapolate_small_slices",
                             "profiles": k, "bits_equal": bits_equal(got, want),
                             "mismatches": int((got.view(np.uint64) != want.view(np.uint64)).sum()),
                             "ok": bits_equal(got, want)}
    return res


def sec_c1(args, ctx):
    """Config 1 (BASELINE.json configs[0], the reference CPU example): one A100 with 3
    co-located jobs (generate_trace seed 7), noisy predictor (target MAE 0.017, rng_seed 7) ->
    default small-slice model -> effective_speed -> optimize_partition, through the C-ABI
    host-pointer call miso_b200_decide made from C++ (tools/c1_latency.cpp). Latency metric:
    microseconds per decision, call nonces 1..K; also: non-consecutive nonces, one launch per
    call, the scalar optimize_partition drop-in (miso_b200_optimize), ctypes / Python. Beside
    it the reference's own chain (oracle/_ref) on one host thread over the same nonces."""
    import ctypes as C
    import subprocess
    import paper_2207_11428_b200 as miso
    tr = miso.generate_trace(7, 3)
    jobs = [(f"j{i}", (tr.speeds5[i, 4], tr.speeds5[i, 3], tr.speeds5[i, 2]), int(tr.mem_gb[i]), None)
            for i in range(3)]
    K = max(args.steps, 1000)
    t3 = np.ascontiguousarray([list(j[1]) for j in jobs], np.float64)
    mem = np.ascontiguousarray([j[2] for j in jobs], np.uint8)
    qos = np.full(3, -1, np.int8)
    e, objv, place = C.c_int(), C.c_double(), np.zeros(7, np.uint8)
    fn = miso.lib.miso_b200_decide
    args_c = (ctx._h, t3.ctypes.data, mem.ctypes.data, qos.ctypes.data, 3)
    tail = (1, 0.017, C.byref(e), place.ctypes.data, C.byref(objv), None)
    for r in range(10):
        fn(*args_c, r + 1, 7, *tail)
    lat = []
    acc = 0.0
    for r in range(K):
        t0 = time.perf_counter()
        rc = fn(*args_c, r + 1, 7, *tail)
        lat.append(time.perf_counter() - t0)
        assert rc >= 0
        if rc == 1:
            acc += objv.value
    py_lat = []
    for r in range(200):
        t0 = time.perf_counter()
        ctx.decide(jobs, nonce=r + 1, rng_seed=7)
        py_lat.append(time.perf_counter() - t0)
    first, _ = ctx.decide(jobs, nonce=1, rng_seed=7)
    exe = ROOT / "paper_2207_11428_b200" / "_lib" / "c1_latency"
    # the scalar optimize_partition drop-in on 2000 acceptance-distribution mixes (DetRng
    # 0xacce91, acceptance_test.cpp:72-85), one instance per call from C++
    import tempfile
    ol = oracle_lib()
    have_ref = ol.have_ref()
    n_opt = 2000
    o_sp, o_off = (ol.Ref() if have_ref else ol.Oracle()).gen_mixes(0xACCE91, n_opt)
    tmpd = tempfile.mkdtemp(prefix="miso_c1_")
    mixf, outf = os.path.join(tmpd, "mixes.bin"), os.path.join(tmpd, "out.bin")
    with open(mixf, "wb") as f:
        f.write(np.uint64(n_opt).tobytes() + o_off.astype(np.uint32).tobytes() + o_sp.tobytes())
    cpp = json.loads(subprocess.run([str(exe), str(K), mixf, outf], check=True, capture_output=True,
                                    text=True).stdout)
    raw = open(outf, "rb").read()
    g_ent = np.frombuffer(raw[:4 * n_opt], np.int32)
    g_obj = np.frombuffer(raw[4 * n_opt:], np.float64)
    res = {"metric": "config-1 decision latency (MPS profile -> predictor -> best MIG partition, 3 jobs)",
           "value": cpp["consecutive_us"], "unit": "us/decision", "higher_is_better": False,
           "p99_us": cpp["consecutive_p99_us"],
           "nonconsecutive_nonce_us": cpp["nonconsecutive_us"],
           "launch_per_call_us": cpp["launch_per_call_us"],
           "python_ctypes_us": float(np.median(np.array(lat) * 1e6)),
           "python_api_us": float(np.median(py_lat) * 1e6), "steps": K,
           "dtype": "f64", "data": "synthetic (generate_trace seed 7, 3 jobs; nonce 1..K)",
           "config": {"workload": "config1: single A100 model, 3 co-located jobs",
                      "api": "miso_b200_decide called from C++ (tools/c1_latency.cpp; host pointers; resident server kernel polling a mapped pinned mailbox, draw-ahead for consecutive nonces, results through mapped pinned memory)"},
           "anchor": {"partition": first.partition_name if first else None,
                      "objective": first.objective if first else None},
           "roofline": {"bound": "latency (PCIe round trip of one request; see DESIGN.md 4(a))"},
           "e2e": {"value": cpp["consecutive_us"], "unit": "us/decision",
                   "h2d_bytes_per_step": 320, "d2h_bytes_per_step": 8 * (4 + 5 * 3)}}
    opt = {"value": cpp["optimize_us"], "p99_us": cpp["optimize_p99_us"], "unit": "us/call",
           "calls": cpp["optimize_calls"],
           "api": "miso_b200_optimize from C++ (one instance per call, host pointers; search-only request to the resident server)",
           "data": "acceptance_test.cpp:72-85 mixes, DetRng(0xacce91), m ~ U{1..7}"}
    if have_ref and not args.no_cpu_baseline:
        r = ol.Ref()
        r.optimize_batch(o_sp, o_off, threads=1)  # warm
        t0 = time.perf_counter()
        w_ent, _, w_obj = r.optimize_batch(o_sp, o_off, threads=1)
        opt["cpu_baseline"] = {"value": (time.perf_counter() - t0) / n_opt * 1e6, "unit": "us/call",
                               "cores": 1, "kind": "reference",
                               "sample": f"the same {n_opt} mixes, optimize_partition per instance, 1 thread"}
        ok = bool(np.array_equal(g_ent, w_ent.astype(np.int32)) and bits_equal(g_obj, w_obj))
        opt["parity"] = {"checked_against": "oracle/_ref optimize_partition", "instances": n_opt,
                         "entry_and_objective_bits_equal": ok, "ok": ok}
    res["optimize_partition"] = opt
    if ol.have_ref() and not args.no_cpu_baseline:
        sec, ref_acc = ol.Ref().c1_time(K)
        res["cpu_baseline"] = {"value": sec / K * 1e6, "unit": "us/decision", "cores": 1,
                               "kind": "reference", "sample": f"{K} decisions, nonce 1..{K}, 1 thread"}
        rbits = int(np.float64(ref_acc).view(np.uint64))
        ok = bool(int(np.float64(acc).view(np.uint64)) == rbits and int(cpp["obj_sum_hex"], 16) == rbits)
        res["parity"] = {"checked_against": "oracle/_ref config-1 chain", "decisions": K,
                         "objective_sum_bit_equal": ok, "ok": ok}
    return res


class TrialRunner:
    """run_trial_unit's work per seed (experiment.hpp:299-362) for a batch of device-resident
    traces: nopart, the best-static search (every feasible catalog entry, one launch; chosen-
    only pruning: a candidate stops once it provably loses), the optsta re-run with the chosen
    partition, and miso (noisy predictor, rng_seed = seed). Three
    contexts (one simulation workspace each) on three streams: nopart and miso overlap the
    static search and the optsta re-run that depends on it.

    For batches that fit the GPU in about one wave (<= 8 seeds per SM, config 4) the miso
    simulations run on their own SM partition (a green context of ~43% of the SMs, 64 of 148)
    and the other sets on the rest, so the two never share an SM's instruction cache
    (paper_2207_11428_b200/partition.py). On the partition the miso batch no longer fits one
    wave of two-warp blocks, so the library picks the one-warp (synchronous STP) kernel there
    (config 4: 5.37e3 -> 6.5e3 trials/s on one box). Larger batches (config 5: 8192 seeds) share the whole GPU, which
    measured faster there. MISO_C4_GREEN_SMS=<k> sets the miso partition's SM count (0: off)."""

    def __init__(self, device):
        import torch
        import paper_2207_11428_b200 as miso
        self.miso = miso
        self.device = device
        self.ctx = [miso.Context(device) for _ in range(3)]
        self.st = [torch.cuda.Stream() for _ in range(3)]
        self.part, self.part_st, self.part_note = None, None, "shared GPU"
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        self.sms = sms
        k = int(os.environ.get("MISO_C4_GREEN_SMS", str(int(round(sms * 0.43 / 8)) * 8)))
        if k > 0:
            try:
                from paper_2207_11428_b200.partition import SmPartition
                self.part = SmPartition(device, k)
                # miso on group 0; nopart and the static search (+ re-run) on group 1
                self.part_st = (self.part.streams(1, 1)[0], self.part.streams(1, 1)[0],
                                self.part.streams(0, 1)[0])
                self.part_note = f"miso on {self.part.sms[0]} SMs, other sets on {self.part.sms[1]} SMs (green contexts)"
            except Exception as e:  # noqa: BLE001 -- no green contexts here: share the GPU
                self.part, self.part_note = None, f"shared GPU (no SM partition: {e})"

    def __call__(self, traces, pruned=True):
        """pruned: the chosen-only best-static search (config 4's default; config 5's 8192
        seeds run the full search, which measured faster there). MISO_C4_PRUNED_STATIC=0/1
        overrides both."""
        miso = self.miso
        env = os.environ.get("MISO_C4_PRUNED_STATIC")
        if env is not None:
            pruned = env == "1"
        (ca, cb, cc), (sa, sb, sc) = self.ctx, self.st
        self.last_note = "shared GPU"
        if self.part is not None and len(traces) <= 8 * self.sms:
            sa, sb, sc = self.part_st
            self.last_note = self.part_note
        p_nop = miso.simulate_batch(ca, traces, miso.SimOptions(policy="nopart", cluster_size=100),
                                    stream=sa, defer=True)
        if self.last_note != "shared GPU" and os.environ.get("MISO_C4_STAGGER", "1") == "1":
            # on the partition, the static search follows nopart instead of starting beside it:
            # the miso seeds' first events then run with less beside them (measured faster)
            sb.wait_stream(sa)
        p_mis = miso.simulate_batch(cc, traces, miso.SimOptions(policy="miso", cluster_size=100,
                                                                predictor="noisy"),
                                    stream=sc, defer=True)
        # run_trial_unit reads only best_static_partition(...).chosen (experiment.hpp:337): the
        # chosen-only pruned search gives the same entries
        st = miso.best_static_partition(cb, traces, cluster_size=100, stream=sb,
                                        chosen_only=pruned)
        sta = miso.simulate_batch(cb, traces, miso.SimOptions(policy="optsta", cluster_size=100),
                                  static_partitions=[miso.DEFAULT_CATALOG[e] for e, _ in st],
                                  stream=sb)
        return p_nop(), st, sta, p_mis()

    def close(self):
        for c in self.ctx:
            c.close()
        if self.part is not None:
            self.part.close()


def ref_trials(seeds):
    """The reference's run_trial_unit-equivalent (oracle/_ref ref_trial) on every host thread:
    (trials/s, threads, per-seed (static entry, [nopart, optsta, miso] avg JCT))."""
    from concurrent.futures import ThreadPoolExecutor
    ol = oracle_lib()
    ref, threads = ol.Ref(), ol.host_threads()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda s: ref.trial(int(s)), seeds))
    return len(seeds) / (time.perf_counter() - t0), threads, outs


def trial_parity(outs, seeds_idx, nop, st, sta, mis):
    got = np.stack([nop.metrics["avg_jct_s"][seeds_idx], sta.metrics["avg_jct_s"][seeds_idx],
                    mis.metrics["avg_jct_s"][seeds_idx]], 1)
    want = np.stack([o for _, o in outs])
    jct_eq = bits_equal(got, want)
    ent_eq = bool(all(e == st[i][0] for i, (e, _) in zip(seeds_idx, outs)))
    return {"trials_compared": len(outs), "avg_jct_bit_equal": jct_eq,
            "static_entry_equal": ent_eq, "ok": jct_eq and ent_eq}


def sec_c4(args, D, runner, seeds_per_rank=1024, steps=3):
    """Config 4 (BASELINE.json configs[3]): 100 GPUs, 1000-job Poisson traces (lambda 10 s),
    default overheads, 1024 seeds per rank; per seed the reference's run_trial_unit policy set.
    Trials/s, the bound (one warp's dependent event chain: per-event time against the issue
    floor and against one CPU core), the reference's trials on every host thread, parity of
    16 trials."""
    import torch
    miso = runner.miso
    seeds = np.arange(D.rank * seeds_per_rank, (D.rank + 1) * seeds_per_rank, dtype=np.uint64)
    traces = miso.generate_traces_device(runner.ctx[0], seeds, 1000, lambda_s=10.0)
    runner(traces)
    times = []
    for _ in range(steps):
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nop, st, sta, mis = runner(traces)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    dt = D.reduce([statistics.median(times)])[0]
    # the miso simulations alone (the critical path): one launch, CUDA events on its stream
    ctx_m, s_m = runner.ctx[2], runner.st[2]
    opts = miso.SimOptions(policy="miso", cluster_size=100, predictor="noisy")
    ms_m = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s_m)
        r = miso.simulate_batch(ctx_m, traces, opts, stream=s_m, defer=True)
        b.record(s_m)
        r = r()
        ms_m.append(a.elapsed_time(b))
    ms_miso = D.reduce([min(ms_m)])[0]
    ms_miso_part = None
    if runner.part is not None and len(traces) <= 8 * runner.sms:  # the same on its SM partition
        s_p = runner.part_st[2]
        ms_p = []
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s_p)
            r = miso.simulate_batch(ctx_m, traces, opts, stream=s_p, defer=True)
            b.record(s_p)
            r = r()
            ms_p.append(a.elapsed_time(b))
        ms_miso_part = D.reduce([min(ms_p)])[0]
    ev = float(mis.metrics["events"].mean())
    S = len(seeds)
    us_ev = ms_miso * 1e3 / ev  # each warp walks its seed's events one after another
    res = {"metric": "cluster-simulation trials/sec (config 4: nopart + optsta(best static) + miso, 100 GPUs x 1000 jobs)",
           "value": D.world * S / dt, "unit": "trials/s", "s_per_step": dt, "seeds_per_gpu": S,
           "n_gpus": D.world, "scaling": "weak", "steps": steps,
           "simulations_per_step": int(S * 3 + len(miso.sim.static_candidates(traces)[0])),
           "miso_events_per_seed": ev, "dtype": "f64",
           "data": "synthetic (generate_trace seeds, generated on the device)",
           "median_jct_norm": {"optsta": float(np.median(sta.metrics["avg_jct_s"] / nop.metrics["avg_jct_s"])),
                               "miso": float(np.median(mis.metrics["avg_jct_s"] / nop.metrics["avg_jct_s"]))},
           "gpu_launches_per_step": "5 of the library's kernels (nopart, the predictor draws and "
                                    "miso, the pruned static search, the optsta re-run) + torch "
                                    "helper ops (candidate feasibility, bound init) and uploads/readbacks",
           "placement": runner.last_note}
    cap = ncu_capture("sim_kernel_ncu.json")
    bound = {"bound": "latency (one warp walks one seed's sequential event chain)",
             "miso_ms": ms_miso, "miso_us_per_event_per_warp": us_ev,
             "miso_events_per_s": S * ev / (ms_miso / 1e3)}
    if cap:
        l0 = cap["launches"][0]
        inst = ncu_val(l0, "smsp__inst_executed.sum")
        cap_ev = cap.get("events_total") or 1024 * 7510
        ipe = inst / cap_ev
        clk = (measured_peaks().get("sm_clock_max_mhz") or 1965.0) * 1e6
        floor = ipe / clk * 1e6  # a warp issues at most one instruction per cycle
        bound.update({"warp_instructions_per_event": ipe,
                      "issue_floor_us_per_event": floor,
                      "frac": floor / us_ev,
                      "frac_note": "issue floor / achieved: the fraction of cycles a simulation warp issues",
                      "ncu_capture": {"issue_active": ncu_val(l0, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
                                      "source": "profiles/sim_kernel_ncu.json"}})
    # the step's own floor: its longest dependent chain is one miso seed's event sequence, so the
    # step cannot end before the miso launch alone would (the other sets run beside it)
    bound["critical_path"] = {"miso_alone_ms": ms_miso, "step_ms": dt * 1e3,
                              "frac": ms_miso / (dt * 1e3),
                              "note": "miso simulations alone on the whole GPU (CUDA events) / the "
                                      "trial step: the step's distance from its critical-path "
                                      "floor"}
    if ms_miso_part is not None:
        bound["critical_path"].update({
            "miso_alone_on_partition_ms": ms_miso_part,
            "partition_frac": ms_miso_part / (dt * 1e3),
            "partition_note": "miso alone on its own SM partition (the step runs it there beside "
                              "the other sets on the remaining SMs): the step's floor under that "
                              "placement"})
    res["roofline"] = bound
    if D.rank == 0 and not args.no_cpu_baseline and oracle_lib().have_ref():
        k = min(S, max(16, oracle_lib().host_threads()))
        rate, threads, outs = ref_trials(seeds[:k])
        # the reference's miso simulation of seed 0 on one core: its time per (live) event
        t0h = traces[0:1].to_host()[0]
        ref = oracle_lib().Ref()
        t0 = time.perf_counter()
        ref.simulate_trace(t0h.arrival_s, t0h.duration_s, t0h.speeds5, t0h.mem_gb, None,
                           seed=int(seeds[0]), cluster_size=100, policy=3, noisy=True,
                           target_mae=0.017, rng_seed=int(seeds[0]))
        ref_s = time.perf_counter() - t0
        ev0 = float(mis.metrics["events"][0])
        res["cpu_baseline"] = {"value": rate, "unit": "trials/s", "cores": threads,
                               "kind": "reference",
                               "sample": f"{k} trials (nopart + best static search + optsta + miso), {threads} threads",
                               "one_core_miso_us_per_event": ref_s * 1e6 / ev0}
        bound["cpu_one_core_us_per_event"] = ref_s * 1e6 / ev0
        res["parity"] = trial_parity(outs, np.arange(k), nop, st, sta, mis)
    return res


def gen_mixes_device(chunk: int, n: int, device):
    """Config-2 distribution generated on the device for chunk `chunk` (Philox seeded by the
    chunk id, so the global dataset is the same for any sharding). Returns (speeds (J*5,),
    offsets (n+1,) int32, m (n,))."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(0xC5000 + chunk)
    m = torch.randint(1, 8, (n,), generator=g, device=device, dtype=torch.int32)
    offs = torch.zeros(n + 1, dtype=torch.int64, device=device)
    offs[1:] = torch.cumsum(m, 0)
    J = int(offs[-1])
    u = torch.rand((J, 5), generator=g, device=device, dtype=torch.float64)
    sp = torch.empty((J, 5), dtype=torch.float64, device=device)
    f4 = 0.2 + 0.8 * u[:, 0]
    f3 = 0.15 + (f4 - 0.15) * u[:, 1]
    f2 = 0.1 + (f3 - 0.1) * u[:, 2]
    f1 = 0.05 + (f2 - 0.05) * u[:, 3]
    f1 = torch.where(u[:, 4] < 0.25, torch.zeros_like(f1), f1)
    sp[:, 0], sp[:, 1], sp[:, 2], sp[:, 3], sp[:, 4] = f1, f2, f3, f4, 1.0
    return sp.reshape(-1), offs.to(torch.int32), m


def sec_c5(args, D, ctx, runner, steps=10):
    """Config 5 (BASELINE.json configs[4]): scaling sweep. A FIXED workload -- 64M config-2 job
    mixes (64 chunks of 1M, generated on the device per chunk) and 8192 trace seeds (config-4
    trials: nopart + best static + miso + optsta re-run) -- sharded over the ranks (strong
    scaling: rank r owns a contiguous block of chunks and of seeds; no data-path collective).
    Search: K launches over the rank's whole shard, CUDA events, max over ranks. Trials: the
    rank's seeds all in flight at once (one launch per policy), max over ranks. Per-seed JCTs
    are gathered to rank 0 (dist.py). Parity: a sample of the last chunk and the last 16 seeds
    against the reference."""
    import torch
    from paper_2207_11428_b200.dist import shard_range
    miso = runner.miso
    dev = D.device
    chunks, per_chunk, S = args.c5_chunks, 1_000_000, args.c5_seeds
    c_lo, c_hi = shard_range(chunks, D.rank, D.world)
    parts = [gen_mixes_device(c, per_chunk, dev) for c in range(c_lo, c_hi)]
    sp = torch.cat([p[0] for p in parts]) if parts else torch.zeros(0, dtype=torch.float64, device=dev)
    offs = torch.zeros(len(parts) * per_chunk + 1, dtype=torch.int32, device=dev)
    base = 0
    for i, p in enumerate(parts):
        offs[i * per_chunk + 1:(i + 1) * per_chunk + 1] = p[1][1:] + base
        base += int(p[1][-1])
    n = len(parts) * per_chunk
    # the last chunk's first instances (for parity on the last rank)
    last = None
    if parts and c_hi == chunks:
        k = 50_000
        lo_row = int(offs[n - per_chunk])
        o_loc = (offs[n - per_chunk: n - per_chunk + k + 1] - lo_row).cpu().numpy().astype(np.uint32)
        last = (sp[lo_row * 5: (lo_row + int(o_loc[-1])) * 5].cpu().numpy(), o_loc)
    del parts
    cand = torch.empty(n, dtype=torch.uint8, device=dev)
    obj = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    for _ in range(3):
        ctx.optimize_batch(sp, offs, cand, obj)
    D.barrier()
    search_ms = cuda_time(st, lambda: ctx.optimize_batch(sp, offs, cand, obj), steps) / steps
    feasible = int((cand < 111).sum().item())
    par_search = None
    cpu_search = 0.0
    if last is not None and not args.no_cpu_baseline and oracle_lib().have_ref():
        ol = oracle_lib()
        k = len(last[1]) - 1
        t0 = time.perf_counter()
        e, p, o = ol.Ref().optimize_batch(last[0], last[1], threads=ol.host_threads())
        cpu_search = k / (time.perf_counter() - t0)
        g_e, g_p = ctx.decode(cand[n - per_chunk: n - per_chunk + k].cpu().numpy(), last[1])
        ok = bool(np.array_equal(g_e, e.astype(np.int32)) and
                  bits_equal(obj[n - per_chunk: n - per_chunk + k].cpu().numpy(), o))
        par_search = {"instances": k, "chunk": chunks - 1, "ok": ok}
    # every chunk, sampled: 2 x 1000 instances (its start and its middle) of each of this rank's
    # chunks against the reference (one thread), decisions, placements and objective bits
    samp_n = samp_bad = 0
    if not args.no_cpu_baseline and oracle_lib().have_ref():
        ref = oracle_lib().Ref()
        for i in range(c_hi - c_lo):
            for j0 in (0, per_chunk // 2):
                a = i * per_chunk + j0
                b = min(a + 1000, n)
                o = offs[a:b + 1]
                r0 = int(o[0])
                o_loc = (o - r0).cpu().numpy().astype(np.uint32)
                spd = sp[r0 * 5:(r0 + int(o_loc[-1])) * 5].cpu().numpy()
                e, p, ob = ref.optimize_batch(spd, o_loc, threads=1)
                g_e, g_p = ctx.decode(cand[a:b].cpu().numpy(), o_loc)
                feas = np.repeat(e >= 0, np.diff(o_loc.astype(np.int64)))
                ok = (np.array_equal(g_e, e.astype(np.int32)) and bits_equal(obj[a:b].cpu().numpy(), ob)
                      and np.array_equal(g_p[feas], p[:len(feas)][feas]))
                samp_n += b - a
                samp_bad += 0 if ok else 1
    del sp, offs, cand, obj
    torch.cuda.empty_cache()
    # ---- trials: every seed of this rank's shard in one launch per policy ----
    s_lo, s_hi = shard_range(S, D.rank, D.world)
    seeds = np.arange(s_lo, s_hi, dtype=np.uint64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    traces = miso.generate_traces_device(runner.ctx[0], seeds, 1000, lambda_s=10.0)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    # the chosen-only pruned static search (with the per-partition speed ceiling in its bound)
    # beats the full search at 1k and at 8k seeds per GPU (profiles/r02_c5_prune_ab.txt)
    pruned = True
    env = os.environ.get("MISO_C4_PRUNED_STATIC")
    if env is not None:
        pruned = env == "1"
    # warm-up at full size: the contexts' workspaces grow to this shard's task counts here
    # (cudaMalloc of up to tens of GB for the static search's candidate runs), not in the
    # timed call
    runner(traces, pruned=pruned)
    D.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nop, stc, sta, mis = runner(traces, pruned=pruned)
    torch.cuda.synchronize()
    trial_s = time.perf_counter() - t0
    rows = np.stack([nop.metrics["avg_jct_s"], sta.metrics["avg_jct_s"], mis.metrics["avg_jct_s"]], 1)
    par_trials = None
    cpu_trials = 0.0
    if s_hi == S and not args.no_cpu_baseline and oracle_lib().have_ref():
        k = min(16, len(seeds))
        cpu_trials, _, outs = ref_trials(seeds[-k:])
        par_trials = trial_parity(outs, np.arange(len(seeds) - k, len(seeds)), nop, stc, sta, mis)
    search_ms, trial_s = D.reduce([search_ms, trial_s], "max")
    feasible = int(D.reduce([float(feasible)], "sum")[0])
    allrows = D.gather(rows.reshape(-1), S * 3)
    # parity results live on the last rank: bring them to rank 0
    flags = D.reduce([0.0 if par_search is None else (1.0 if par_search["ok"] else -1.0),
                      0.0 if par_trials is None else (1.0 if par_trials["ok"] else -1.0),
                      cpu_search, cpu_trials, float(samp_n), float(samp_bad)], "sum")
    if D.rank != 0:
        return None
    r = allrows.reshape(S, 3)
    peak, _ = measured_peak()
    gbs = 173.07e6 * chunks / (search_ms / 1e3) / 1e9 / D.world  # per GPU
    res = {
        "metric": "config-5 scaling sweep: 64M job mixes + 8192 trial seeds, fixed total, sharded",
        "value": chunks * per_chunk / (search_ms / 1e3), "unit": "instances/s",
        "n_gpus": D.world, "steps": steps, "higher_is_better": True, "scaling": "strong",
        "dtype": "f64",
        "data": "synthetic (device Philox per 1M chunk; generate_trace seeds 0..S-1 generated on the device)",
        "config": {"workload": "config5", "mixes": chunks * per_chunk, "seeds": S,
                   "parallelism": f"{D.world} shards, no data-path collective"},
        "search_ms_per_pass": search_ms, "feasible_instances": feasible,
        "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                     "frac": gbs / peak,
                     "note": "per GPU; algorithmic bytes ~173.07 MB per 1M mixes (41m+13 B per mix, E[m]=4)"},
        "trials": {"value": S / trial_s, "unit": "trials/s", "s": trial_s,
                   "seeds_in_flight_per_gpu": s_hi - s_lo,
                   "static_search": "chosen-only pruned" if pruned else "full",
                   "placement": runner.last_note,
                   "device_trace_gen_s_rank0": gen_s},
        "median_jct_norm": {"optsta": float(np.median(r[:, 1] / r[:, 0])),
                            "miso": float(np.median(r[:, 2] / r[:, 0]))},
        "gpu_launches": steps,
    }
    if flags[0] != 0 or flags[1] != 0:
        res["parity"] = {"search_sample_of_last_chunk_ok": None if flags[0] == 0 else bool(flags[0] > 0),
                         "every_chunk_sampled": {"instances": int(flags[4]), "chunks": chunks,
                                                 "failed_samples": int(flags[5]), "ok": flags[5] == 0},
                         "last_16_trials_ok": None if flags[1] == 0 else bool(flags[1] > 0),
                         "checked_against": "oracle/_ref (optimize_partition on 50k mixes of the last chunk and on 2 x 1000 mixes of every chunk; run_trial_unit-equivalent trials of the last 16 seeds)",
                         "ok": bool(flags[0] >= 0 and flags[1] >= 0 and flags[5] == 0)}
        threads = oracle_lib().host_threads()
        res["cpu_baseline"] = {"value": flags[2], "unit": "instances/s", "cores": threads,
                               "kind": "reference",
                               "sample": f"50k mixes of the last chunk, {threads} threads",
                               "trials": {"value": flags[3], "unit": "trials/s", "cores": threads,
                                          "sample": f"the last 16 seeds, {threads} threads"}}
    return res


# ---------------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="headline (config 2) only; skip configs 1/3/4/5")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4", "c5"], default="c2",
                    help="c2 = headline (config 2, + secondary); c1 / c3 / c4 / c5 alone")
    ap.add_argument("--c5-chunks", type=int, default=64, help="c5: 1M-mix chunks in total")
    ap.add_argument("--c5-seeds", type=int, default=8192, help="c5: trial seeds in total")
    ap.add_argument("--seeds", type=int, default=1024, help="c4: trace seeds per GPU")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(spawn_ranks(args))

    D = Dist()
    if args.impl == "reference":
        # the reference's own CPU implementation: rank 0 alone (n_gpus as launched)
        if "WORLD_SIZE" not in os.environ:
            D.world = args.gpus
        run_reference_arm(args, D)
        return

    D.init()
    import paper_2207_11428_b200 as miso
    ctx = miso.Context(D.local)
    out = None
    if args.config == "c1":
        out = sec_c1(args, ctx) if D.rank == 0 else None
    elif args.config == "c3":
        out = sec_c3(args, D, ctx, steps=args.steps)
    elif args.config in ("c4", "c5"):
        runner = TrialRunner(D.local)
        out = sec_c4(args, D, runner, args.seeds, steps=max(1, args.steps)) if args.config == "c4" \
            else sec_c5(args, D, ctx, runner, steps=args.steps)
        runner.close()
    else:
        clocks = ClockSampler(D.local).start()
        line, (speeds, offs, m, h_cand, h_obj) = run_c2(args, D, ctx, clocks)
        if D.rank == 0 and not args.no_cpu_baseline:
            line["cpu_baseline"], line["parity"] = c2_cpu_baseline(speeds, offs, m, ctx, h_cand, h_obj)
        if not args.no_secondary:
            sec = {}
            if D.rank == 0:
                sec["c1"] = sec_c1(args, ctx)
            clocks.timed(True)
            sec["c3"] = sec_c3(args, D, ctx)
            runner = TrialRunner(D.local)
            sec["c4"] = sec_c4(args, D, runner, args.seeds)
            clocks.timed(False)
            sec["c5"] = sec_c5(args, D, ctx, runner)
            runner.close()
            line["secondary"] = sec
        line["clocks"] = clocks.stop()
        out = line if D.rank == 0 else None
    if out is not None and D.rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    D.close()


if __name__ == "__main__":
    main()
