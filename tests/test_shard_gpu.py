"""Several contexts (the multi-device C ABI) and the simulator's input
contract: miso_b200_optimize_batch_sharded / miso_b200_simulate_batch_sharded over two
contexts give the bytes of one context's call (on a 1-GPU box both contexts sit on GPU 0; the
split, per-shard threads and scatter are the same code), and invalid traces are reported the
way the reference throws (validate_profile, init_jobs)."""
import ctypes as C

import numpy as np
import pytest

import paper_2207_11428_b200 as miso
from paper_2207_11428_b200 import sim as simmod

pytestmark = pytest.mark.gpu
L = miso.lib
vp = C.c_void_p
L.miso_b200_optimize_batch_sharded.argtypes = [vp, C.c_int, vp, vp, C.c_uint64, vp, vp]
L.miso_b200_simulate_batch_sharded.argtypes = [vp, C.c_int, C.POINTER(simmod.SimOptionsC), C.c_int,
                                               C.c_int] + [vp] * 13 + [C.c_int64, vp, C.c_int64, C.c_uint]
L.miso_b200_simulate_batch_host.argtypes = [vp, C.POINTER(simmod.SimOptionsC), C.c_int, C.c_int] + \
    [vp] * 13 + [C.c_int64, vp, C.c_int64, C.c_uint]
L.miso_b200_device_count.restype = C.c_int


def _ctx_array(ctxs):
    arr = (C.c_void_p * len(ctxs))(*[c._h.value for c in ctxs])
    return arr


def test_device_count():
    import torch
    assert L.miso_b200_device_count() == torch.cuda.device_count() >= 1


def test_optimize_sharded_equals_single(ctx, oracle):
    speeds, offs = oracle.gen_mixes(0xACCE91, 200_003)
    n = len(offs) - 1
    c1, o1 = ctx.optimize_batch(speeds, offs)
    extra = [miso.Context(0) for _ in range(2)]
    for k in (2, 3):
        ctxs = [ctx] + extra[: k - 1]
        cand, obj = np.empty(n, np.uint8), np.empty(n)
        rc = L.miso_b200_optimize_batch_sharded(_ctx_array(ctxs), k, speeds.ctypes.data,
                                                offs.ctypes.data, n, cand.ctypes.data, obj.ctypes.data)
        assert rc == 0, L.miso_b200_last_error()
        assert np.array_equal(cand, c1) and np.array_equal(obj.view(np.uint64), o1.view(np.uint64))
    e, _, o = oracle.optimize_batch(speeds, offs)
    assert np.array_equal(ctx.decode(c1, offs)[0], e.astype(np.int32))
    for c in extra:
        c.close()


def _host_sim(ctxs, opts, traces, task_trace=None, static=None, log_cap=0, stp_cap=0, flags=0):
    offs, arr, dur, sp, mem, qos, inst = simmod._csr(traces)
    n_traces = len(traces)
    S = n_traces if task_trace is None else len(task_trace)
    seeds = np.array([t.seed for t in traces], np.uint64)
    if task_trace is not None:
        seeds = seeds[np.asarray(task_trace)]
    tt = None if task_trace is None else np.ascontiguousarray(task_trace, np.int32)
    sc = None if static is None else np.ascontiguousarray(static, np.uint8).reshape(-1)
    inst_a = None if inst is None else np.ascontiguousarray(inst, np.uint8)
    per = np.diff(offs)
    mj = int(per.max())
    if inst_a is not None:
        cs = np.concatenate([[0], np.cumsum(np.maximum(inst_a.astype(np.int64) - 1, 0))])
        mj = int((per + cs[offs[1:]] - cs[offs[:-1]]).max())
    met = np.zeros(S, simmod.METRICS_DTYPE)
    jo = np.zeros(S * mj * 8, np.int64)
    lg = np.zeros(S * log_cap, simmod.LOG_DTYPE) if log_cap else None
    stp = np.zeros(S * stp_cap * 2) if stp_cap else None
    o = opts.to_c()
    args = (C.byref(o), S, n_traces, None if tt is None else tt.ctypes.data,
            None if sc is None else sc.ctypes.data, offs.ctypes.data, arr.ctypes.data,
            dur.ctypes.data, np.ascontiguousarray(sp).ctypes.data, mem.ctypes.data,
            qos.ctypes.data, None if inst_a is None else inst_a.ctypes.data, seeds.ctypes.data,
            met.ctypes.data, jo.ctypes.data, None if lg is None else lg.ctypes.data, log_cap,
            None if stp is None else stp.ctypes.data, stp_cap, flags)
    if len(ctxs) == 1:
        rc = L.miso_b200_simulate_batch_host(ctxs[0]._h, *args)
    else:
        rc = L.miso_b200_simulate_batch_sharded(_ctx_array(ctxs), len(ctxs), *args)
    assert rc == 0, L.miso_b200_last_error()
    return met, jo, lg, stp


def test_simulate_sharded_equals_single(ctx):
    traces = miso.generate_traces(range(40, 51), 70, lambda_s=25.0)
    for t in traces[::3]:
        t.instances = np.ones(t.n, np.uint8)
        t.instances[4] = 3
    traces = list(traces)
    other = miso.Context(0)
    for pol in ("miso", "oracle", "nopart"):
        opts = miso.SimOptions(policy=pol, cluster_size=4, predictor="noisy")
        one = _host_sim([ctx], opts, traces, log_cap=4096, stp_cap=2048)
        two = _host_sim([ctx, other], opts, traces, log_cap=4096, stp_cap=2048)
        met = one[0]
        assert np.array_equal(met.view(np.uint8), two[0].view(np.uint8)), pol
        assert np.array_equal(one[1], two[1]), pol  # job_out (unused rows are zeros)
        for i in range(len(traces)):  # event logs and STP series up to their lengths
            nl, ns = int(met["log_records"][i]), int(met["stp_points"][i])
            assert np.array_equal(one[2][i * 4096: i * 4096 + nl].view(np.uint8),
                                  two[2][i * 4096: i * 4096 + nl].view(np.uint8)), pol
            assert np.array_equal(one[3][i * 4096: i * 4096 + 2 * ns].view(np.uint64),
                                  two[3][i * 4096: i * 4096 + 2 * ns].view(np.uint64)), pol
    # a best-static-style batch (task_trace, static partitions, JCT-only) split by trace
    tt = np.repeat(np.arange(len(traces)), 4).astype(np.int32)
    static = np.array([miso.DEFAULT_CATALOG[e] for e in (0, 8, 13, 20)] * len(traces), np.uint8)
    opts = miso.SimOptions(policy="optsta", cluster_size=4)
    one = _host_sim([ctx], opts, traces, task_trace=tt, static=static, flags=1)
    two = _host_sim([ctx, other], opts, traces, task_trace=tt, static=static, flags=1)
    assert np.array_equal(one[0].view(np.uint8), two[0].view(np.uint8))
    assert np.array_equal(one[1], two[1])
    other.close()


def _bad(trace, **kw):
    return miso.Trace(trace.arrival_s.copy(), trace.duration_s.copy(), trace.speeds5.copy(),
                      trace.mem_gb.copy(), None, trace.seed, **kw)


@pytest.mark.parametrize("mutate, msg", [
    (lambda t: t.duration_s.__setitem__(5, 0.0), "job 'j5': base duration must be positive"),
    (lambda t: t.speeds5.__setitem__((7, 2), 1.5), "job 'j7': speed on 3g outside (0,1]"),
    (lambda t: t.speeds5.__setitem__((3, 4), 0.9), "job 'j3': speed on 7g must be exactly 1"),
    (lambda t: t.speeds5.__setitem__((9, 1), 0.99), "job 'j9': speed table not monotone in gpc count"),
    (lambda t: t.arrival_s.__setitem__(0, 1.0), "first arrival must be at t=0"),
    (lambda t: t.arrival_s.__setitem__(6, 0.0), "arrival times must be non-decreasing"),
])
def test_invalid_trace_rejected_like_reference(ctx, mutate, msg):
    t = _bad(miso.generate_trace(3, 20, lambda_s=30.0))
    mutate(t)
    with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        miso.simulate_batch(ctx, [t], miso.SimOptions(policy="miso", cluster_size=2))


def test_invalid_memory_not_wrapped(ctx):
    t = _bad(miso.generate_trace(3, 20, lambda_s=30.0))
    t.mem_gb[2] = 300  # would wrap to 44 in a uint8 cast
    with pytest.raises(ValueError, match="j2': memory demand must be in"):
        miso.simulate_batch(ctx, [t], miso.SimOptions(policy="nopart", cluster_size=2))


def test_device_tensor_inputs_report_per_task_status(ctx):
    """Device-resident traces are checked on the device (no host read-back): the task's status
    is MISO_B200_SIM_BAD_INPUT with the failing job and check in metrics.detail."""
    import torch
    tb = miso.generate_traces_device(ctx, np.arange(3, dtype=np.uint64), 40, lambda_s=30.0)
    tb.speeds5[1, 12, 0] = 2.0
    with pytest.raises(ValueError, match="job 'j12': speed on 1g outside"):
        miso.simulate_batch(ctx, tb, miso.SimOptions(policy="miso", cluster_size=2))
    torch.cuda.synchronize()


def test_want_jct_with_task_trace_rejected(ctx):
    tr = [miso.generate_trace(1, 20, lambda_s=30.0)]
    with pytest.raises(ValueError):
        miso.simulate_batch(ctx, tr, miso.SimOptions(policy="nopart", cluster_size=2),
                            task_trace=[0, 0], want_jct=True)


def test_custom_small_slice_model(ctx):
    """SimOptions.small_slice_model: the default weights reproduce the default run bit for bit;
    other weights change the miso estimates (parity with the reference's caller-fitted model is
    tools/dropin/sim_parity.cpp, a GPU test in test_dropin_gpu.py)."""
    traces = miso.generate_traces(range(5), 60, lambda_s=20.0)
    base = miso.SimOptions(policy="miso", cluster_size=3, predictor="noisy")
    r0 = miso.simulate_batch(ctx, traces, base)
    w2, w1 = miso.default_model()
    same = miso.SimOptions(policy="miso", cluster_size=3, predictor="noisy", small_slice_model=(w2, w1))
    r1 = miso.simulate_batch(ctx, traces, same)
    assert np.array_equal(r0.metrics.view(np.uint8), r1.metrics.view(np.uint8))
    other = miso.SimOptions(policy="miso", cluster_size=3, predictor="noisy",
                            small_slice_model=([0, 0.5, 0.4, 0.0], [0, 0.1, 0.6, 0.0]))
    r2 = miso.simulate_batch(ctx, traces, other)
    assert not np.array_equal(r0.metrics["avg_jct_s"], r2.metrics["avg_jct_s"])


def test_max_events_counts_every_push(ctx, ref):
    """The budget is exceeded iff the pushed events (= the reference's pops, stale included)
    exceed max_events: at the reference's exact pop count the run completes, one below it
    fails (the reference's count comes from tools/dropin/sim_parity.cpp's search; here the
    device side of the same rule: budget = events pushed)."""
    tr = [miso.generate_trace(9301, 30, lambda_s=15.0)]
    opts = miso.SimOptions(policy="miso", cluster_size=2, predictor="noisy")
    full = miso.simulate_batch(ctx, tr, opts, rng_seeds=[9301])
    assert full.metrics["status"][0] == 0
    lo, hi = 1, 1 << 20
    while lo < hi:
        mid = (lo + hi) // 2
        opts.max_events = mid
        st = miso.simulate_batch(ctx, tr, opts, rng_seeds=[9301]).metrics["status"][0]
        if st == 0:
            hi = mid
        else:
            assert st == 4
            lo = mid + 1
    assert lo > full.metrics["events"][0]  # stale pops count too
