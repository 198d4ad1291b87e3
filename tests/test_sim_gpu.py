"""GPU parity tests for kernel (c), the batched event-step simulator (one warp per seed).

Bar (north_star): simulated event orders bit-exact -- the rendered event log must equal the
reference's text byte for byte -- and JCT statistics within 1e-5 (asserted bit-exact here,
since the engine keeps the reference's FP64 evaluation order, including the sequential STP sum).
The reference is run through oracle/_ref (the unmodified sim.hpp) on the same traces.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POL = {"nopart": 0, "oracle": 2, "miso": 3}


def ref_run(ref, tr, opts, rng_seed, want_log=True):
    out, log, _ = ref.simulate_trace(
        tr.arrival_s, tr.duration_s, tr.speeds5, tr.mem_gb, tr.qos_kind, seed=tr.seed,
        cluster_size=opts.cluster_size, policy=POL[opts.policy],
        mig_reconfig_s=opts.mig_reconfig_s, checkpoint_restart_s=opts.checkpoint_restart_s,
        mps_window_s=opts.mps_window_s, interference=opts.interference,
        noisy=opts.predictor == "noisy", target_mae=opts.target_mae, rng_seed=rng_seed,
        want_log=want_log)
    return out, log


def check_metrics(got, want):
    assert got["status"] == 0
    assert bool(got["completed"]) == bool(want.completed)
    assert got["completed_count"] == want.completed_count
    assert got["repartitions"] == want.repartitions
    assert got["mps_sessions"] == want.mps_sessions
    for f in ("avg_jct_s", "makespan_s", "stp_time_avg", "queue_frac", "mps_frac",
              "checkpoint_frac", "run_frac", "idle_frac"):
        g, w = float(got[f]), float(getattr(want, f))
        assert g == w or abs(g - w) <= 1e-12 * max(1.0, abs(w)), (f, g, w)
    assert got["stp_points"] == want.stp_points


def run_and_compare(ctx, ref, traces, opts, log_cap=1 << 16):
    import paper_2207_11428_b200 as m
    res = m.simulate_batch(ctx, traces, opts, log_cap=log_cap)
    for i, tr in enumerate(traces):
        want, wlog = ref_run(ref, tr, opts, tr.seed)
        got = res.report(i)
        assert got["log_records"] <= log_cap
        text = m.render_log(res.logs[i])
        assert wlog and wlog.count("\n") >= 3 * tr.n  # arrival + admit + complete per job at least
        if text != wlog:
            a, b = text.splitlines(), wlog.splitlines()
            k = next((q for q in range(min(len(a), len(b))) if a[q] != b[q]), min(len(a), len(b)))
            raise AssertionError(f"seed {tr.seed}: event logs diverge at line {k}: "
                                 f"got {a[k:k+3]} want {b[k:k+3]}")
        check_metrics(got, want)
    return res


@pytest.mark.parametrize("policy,predictor", [("miso", "noisy"), ("miso", "oracle"),
                                              ("oracle", "oracle"), ("nopart", "oracle")])
def test_event_log_parity_small(ctx, ref, policy, predictor):
    import paper_2207_11428_b200 as m
    traces = [m.generate_trace(seed, 100, lambda_s=60.0) for seed in (1, 2, 3, 1000)]
    opts = m.SimOptions(policy=policy, cluster_size=8, predictor=predictor)
    run_and_compare(ctx, ref, traces, opts)


def test_event_log_parity_config4_shape(ctx, ref):
    """Config 4: 100 GPUs, 1000-job Poisson trace (lambda 10 s), noisy predictor 0.017."""
    import paper_2207_11428_b200 as m
    traces = [m.generate_trace(seed, 1000, lambda_s=10.0) for seed in (0, 1)]
    opts = m.SimOptions(policy="miso", cluster_size=100, predictor="noisy")
    run_and_compare(ctx, ref, traces, opts, log_cap=1 << 16)


def test_clairvoyant_equivalence(ctx):
    """acceptance_test.cpp:141-177 / sim_test.cpp:161-221: zero overheads + oracle predictor
    -> miso and oracle policies produce byte-identical event logs and equal metrics."""
    import paper_2207_11428_b200 as m
    traces = [m.generate_trace(9000 + t, 100, lambda_s=60.0) for t in range(50)]
    kw = dict(cluster_size=8, mig_reconfig_s=0, checkpoint_restart_s=0, mps_window_s=0,
              predictor="oracle")
    a = m.simulate_batch(ctx, traces, m.SimOptions(policy="miso", **kw), log_cap=1 << 14)
    b = m.simulate_batch(ctx, traces, m.SimOptions(policy="oracle", **kw), log_cap=1 << 14)
    for i in range(len(traces)):
        la, lb = m.render_log(a.logs[i]), m.render_log(b.logs[i])
        assert la == lb and la
        assert a.metrics[i]["avg_jct_s"] == b.metrics[i]["avg_jct_s"]


def test_seven_parallel_friendly_jobs(ctx, ref):
    """sim_test.cpp:135-159: seven f(g)=(g/7)^0.5 jobs on one GPU -> STP sqrt(7), 13
    repartitions, no MPS sessions (zero overheads, oracle predictor)."""
    import paper_2207_11428_b200 as m
    g = np.array([1, 2, 3, 4, 7]) / 7.0
    sp = np.tile(g ** 0.5, (7, 1))
    tr = m.Trace(np.zeros(7), np.full(7, 100.0), sp, np.full(7, 5), None, 0)
    opts = m.SimOptions(policy="miso", cluster_size=1, mig_reconfig_s=0, checkpoint_restart_s=0,
                        mps_window_s=0, predictor="oracle")
    res = run_and_compare(ctx, ref, [tr], opts)
    r = res.report(0)
    rate = np.sqrt(1.0 / 7.0)
    assert r["completed"] == 1 and r["completed_count"] == 7
    assert abs(r["avg_jct_s"] - 100.0 / rate) < 1e-5
    assert abs(r["stp_time_avg"] - np.sqrt(7.0)) < 1e-9
    assert r["repartitions"] == 13 and r["mps_sessions"] == 0


def test_profiling_sessions_counted(ctx, ref):
    """sim_test.cpp:223-246: j0 profiles alone; j1..j3 queue and share one batched session."""
    import paper_2207_11428_b200 as m
    sp = np.tile([0.3, 0.5, 0.7, 0.8, 1.0], (4, 1))
    tr = m.Trace(np.arange(4) * 5.0, np.full(4, 300.0), sp, np.full(4, 5), None, 0)
    opts = m.SimOptions(policy="miso", cluster_size=1, predictor="noisy", target_mae=0.05)
    res = m.simulate_batch(ctx, [tr], opts, rng_seeds=[9], log_cap=4096)
    want, wlog = ref_run(ref, tr, opts, 9)
    assert m.render_log(res.logs[0]) == wlog
    r = res.report(0)
    assert r["mps_sessions"] == 2 and r["mps_frac"] > 0 and r["checkpoint_frac"] > 0
    check_metrics(r, want)


def test_memory_pinned_and_qos_jobs(ctx, ref):
    """Traces with 40 GB jobs (7g only) and QoS floors exercise effective_speed zeroing,
    spare-slice admission and head-of-line blocking."""
    import paper_2207_11428_b200 as m
    rng = np.random.default_rng(4)
    traces = []
    for s in range(4):
        t = m.generate_trace(500 + s, 120, lambda_s=30.0)
        t.mem_gb = np.where(rng.random(t.n) < 0.08, 40, t.mem_gb).astype(np.int32)
        t.qos_kind = np.where(rng.random(t.n) < 0.15, rng.integers(0, 4, t.n), -1).astype(np.int8)
        traces.append(t)
    for pol, pred in (("miso", "noisy"), ("oracle", "oracle")):
        run_and_compare(ctx, ref, traces, m.SimOptions(policy=pol, cluster_size=6, predictor=pred))


def test_invalid_sim_options(ctx):
    import paper_2207_11428_b200 as m
    tr = [m.generate_trace(1, 10)]
    for bad in (dict(cluster_size=0), dict(interference=0.0), dict(mig_reconfig_s=-1.0),
                dict(target_mae=0.7, predictor="noisy")):
        with pytest.raises(m.MisoError) as ei:
            m.simulate_batch(ctx, tr, m.SimOptions(**bad))
        assert ei.value.code == -2


def test_pruned_search_contract(ctx):
    """miso_b200_simulate_batch_pruned rejects what its bound cannot cover: another policy,
    no task_trace, multi-instance traces (the Python wrapper), per-job outputs."""
    import torch
    import paper_2207_11428_b200 as m
    tr = m.generate_traces(range(3), 40, lambda_s=20.0)
    bound = torch.full((3,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    part = [m.DEFAULT_CATALOG[8]] * 3
    with pytest.raises(m.MisoError) as ei:
        m.simulate_batch(ctx, tr, m.SimOptions(policy="nopart", cluster_size=4), task_trace=[0, 1, 2],
                         static_partitions=part, prune_bound=bound)
    assert ei.value.code == -2
    with pytest.raises(m.MisoError):
        m.simulate_batch(ctx, tr, m.SimOptions(policy="optsta", cluster_size=4),
                         static_partitions=part, prune_bound=bound)
    with pytest.raises(ValueError):
        m.simulate_batch(ctx, tr, m.SimOptions(policy="optsta", cluster_size=4), task_trace=[0, 1, 2],
                         static_partitions=part, prune_bound=bound, want_jct=True)
    # a completed candidate lowers its trace's bound to its exact JCT sum (us)
    res = m.simulate_batch(ctx, tr, m.SimOptions(policy="optsta", cluster_size=4), task_trace=[0, 1, 2],
                           static_partitions=part, prune_bound=bound, jct_only=True)
    full = m.simulate_batch(ctx, tr, m.SimOptions(policy="optsta", cluster_size=4),
                            static_partitions=part, want_jct=True)
    assert (res.metrics["status"] == 0).all()
    want = [int(np.asarray(j).sum()) for j in full.job_jct_us]
    assert bound.cpu().tolist() == want
    assert np.array_equal(res.metrics["avg_jct_s"].view(np.uint64), full.metrics["avg_jct_s"].view(np.uint64))


def test_optsta_event_log_parity(ctx, ref):
    """optsta policy (sim.hpp:493-572): fixed slots, largest-free-slot admission and
    small-to-large migrations with checkpoint restarts, byte-identical logs."""
    import paper_2207_11428_b200 as m
    from paper_2207_11428_b200.catalog import DEFAULT_CATALOG
    traces = [m.generate_trace(seed, 120, lambda_s=30.0) for seed in (11, 12)]
    for entry in (1, 8, 9, 24, 0):  # 4g+2g+1g, 3g+2g+2g, 3g+2g+1g+1g, 2g+1g*4, 7g
        opts = m.SimOptions(policy="optsta", cluster_size=6)
        res = m.simulate_batch(ctx, traces, opts, static_partitions=[DEFAULT_CATALOG[entry]] * 2,
                               log_cap=1 << 15)
        for i, tr in enumerate(traces):
            want, wlog = ref.simulate_trace(tr.arrival_s, tr.duration_s, tr.speeds5, tr.mem_gb,
                                            None, seed=tr.seed, cluster_size=6, policy=1,
                                            noisy=False, rng_seed=tr.seed, static_entry=entry,
                                            want_log=True)[:2]
            assert m.render_log(res.logs[i]) == wlog, (entry, tr.seed)
            got = res.report(i)
            assert got["migrations"] == want.migrations
            check_metrics(got, want)


def test_best_static_partition_matches_reference(ctx, ref):
    """best_static_partition (sim.hpp:1031-1066): all 36 candidates x 3 traces in one launch."""
    import paper_2207_11428_b200 as m
    traces = [m.generate_trace(seed, 150, lambda_s=20.0) for seed in (21, 22, 23)]
    got = m.best_static_partition(ctx, traces, cluster_size=8)
    for (entry, table), tr in zip(got, traces):
        we, wt = ref.best_static(tr.arrival_s, tr.duration_s, tr.speeds5, tr.mem_gb, cluster_size=8)
        assert entry == we
        assert np.array_equal(np.isinf(table), np.isinf(wt))
        fin = ~np.isinf(wt)
        assert np.array_equal(table[fin].view(np.uint64), wt[fin].view(np.uint64))


@pytest.mark.parametrize("spec", [
    dict(n=256, job_count=1000, lambda_s=10.0, cluster=100),   # config 4
    dict(n=96, job_count=300, lambda_s=40.0, cluster=8),       # light load: other winners
    dict(n=96, job_count=200, lambda_s=2.0, cluster=4),        # heavy queueing
    dict(n=64, job_count=150, lambda_s=15.0, cluster=6, dist="fixed", fixed_s=900.0),
])
def test_chosen_only_static_search_matches_full(ctx, spec):
    """best_static_partition(chosen_only=True) -- the pruned two-launch search used for
    run_trial_unit -- chooses the same entry as the full search, with the same avg JCT bits,
    and every candidate it did not stop has the full search's value."""
    import paper_2207_11428_b200 as m
    sp = dict(spec)
    n, cl = sp.pop("n"), sp.pop("cluster")
    traces = m.generate_traces(range(500, 500 + n), **sp)
    full = m.best_static_partition(ctx, traces, cluster_size=cl)
    fast = m.best_static_partition(ctx, traces, cluster_size=cl, chosen_only=True)
    stopped = 0
    for (e0, t0), (e1, t1) in zip(full, fast):
        assert e0 == e1
        assert t0[e0].view(np.uint64) == t1[e1].view(np.uint64)
        kept = np.isfinite(t1)
        assert np.array_equal(t1[kept].view(np.uint64), t0[kept].view(np.uint64))
        assert (t1[~kept] == np.inf).all()
        stopped += int((np.isfinite(t0) & ~kept).sum())
    if spec["job_count"] >= 300:
        assert stopped > 0  # the bound does stop candidates at these sizes


@pytest.mark.parametrize("spec", [
    dict(job_count=1000, lambda_s=10.0),                       # config 4
    dict(job_count=257, lambda_s=60.0, sigma=0.7),
    dict(job_count=1, lambda_s=5.0),
    dict(job_count=333, lambda_s=0.5, dist="fixed", fixed_s=1234.5),
    dict(job_count=500, lambda_s=30.0, dist="uniform", lo_s=60.0, hi_s=4000.0),
    dict(job_count=90, lambda_s=30.0, max_duration_s=900.0, sigma=3.0),
])
def test_device_trace_generation_bit_exact(ctx, spec):
    """generate_trace on the device (one warp per trace; glibc exp/pow/log1p/log/cos restated
    from the FMA variants) == the host generator (itself bit-identical to the reference's)."""
    import torch
    import paper_2207_11428_b200 as m
    seeds = [0, 1, 7, 99, 2**40 + 3, 2**63 + 11] + list(range(1000, 1058))
    db = m.generate_traces_device(ctx, seeds, **spec)
    a, d, sp, mem = db.arrival_s, db.duration_s, db.speeds5, db.mem_gb
    torch.cuda.synchronize()
    host = m.generate_traces(seeds, **spec)
    for i, t in enumerate(host):
        assert np.array_equal(a[i].cpu().numpy().view(np.uint64), t.arrival_s.view(np.uint64)), (spec, i, "arrival")
        assert np.array_equal(d[i].cpu().numpy().view(np.uint64), t.duration_s.view(np.uint64)), (spec, i, "duration")
        assert np.array_equal(sp[i].cpu().numpy().view(np.uint64), t.speeds5.view(np.uint64)), (spec, i, "speeds")
        assert np.array_equal(mem[i].cpu().numpy(), t.mem_gb), (spec, i, "mem")


def test_device_trace_batch_feeds_the_simulator(ctx):
    """A device-resident trace batch goes straight into simulate_batch / best_static_partition:
    same metrics (bits) as the host traces."""
    import paper_2207_11428_b200 as m
    seeds = list(range(40))
    db = m.generate_traces_device(ctx, seeds, 300, lambda_s=20.0)
    hb = m.generate_traces(seeds, 300, lambda_s=20.0)
    for pol in ("nopart", "miso"):
        o = m.SimOptions(policy=pol, cluster_size=16, predictor="noisy")
        a = m.simulate_batch(ctx, db, o).metrics
        b = m.simulate_batch(ctx, hb, o).metrics
        assert a.tobytes() == b.tobytes(), pol
    sa = m.best_static_partition(ctx, db, cluster_size=16)
    sb = m.best_static_partition(ctx, hb, cluster_size=16)
    assert [e for e, _ in sa] == [e for e, _ in sb]
    assert all(np.array_equal(x.view(np.uint64), y.view(np.uint64)) for (_, x), (_, y) in zip(sa, sb))


def test_device_trace_batch_stream_order(ctx):
    """Stream order of device-resident traces: traces generated on one stream behind a long
    spin, then simulated at once on other streams (and a slice of them, and the chosen-only
    static search) without any host synchronisation -- every launch waits for the generator,
    so the results equal the host traces' bit for bit."""
    import torch
    import paper_2207_11428_b200 as m
    seeds = list(range(24))
    hb = m.generate_traces(seeds, 200, lambda_s=20.0)
    o = m.SimOptions(policy="nopart", cluster_size=16)
    want = m.simulate_batch(ctx, hb, o).metrics
    gen, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(gen):
        torch.cuda._sleep(50_000_000)  # ~25 ms: the generator finishes long after the launches
    db = m.generate_traces_device(ctx, seeds, 200, lambda_s=20.0, stream=gen)
    c2 = m.Context(0)
    try:
        r1 = m.simulate_batch(ctx, db, o, stream=s1, defer=True)
        r2 = m.simulate_batch(c2, db[8:24], o, stream=s2, defer=True)
        got1, got2 = r1().metrics, r2().metrics
        assert got1.tobytes() == want.tobytes()
        assert got2.tobytes() == want[8:24].tobytes()
        torch.cuda.synchronize()
        with torch.cuda.stream(gen):
            torch.cuda._sleep(50_000_000)
        db2 = m.generate_traces_device(ctx, seeds, 200, lambda_s=20.0, stream=gen)
        st = m.best_static_partition(c2, db2, cluster_size=16, stream=s2, chosen_only=True)
        sh = m.best_static_partition(ctx, hb, cluster_size=16)
        assert [e for e, _ in st] == [e for e, _ in sh]
    finally:
        c2.close()


def test_async_stp_matches_sync():
    """The asynchronous-STP kernels (an STP helper warp per task; the default for batches
    that fit one wave) against the synchronous ones, forced per process with
    MISO_B200_SIM_ASYNC_STP: miso and oracle metrics and STP series byte-identical
    (tools/async_stp_check.py on 256 config-4 seeds)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    p = subprocess.run([sys.executable, str(root / "tools" / "async_stp_check.py"), "256"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert p.returncode == 0, p.stdout + p.stderr
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert all(res["identical"].values()), res


def test_sm_partition_streams_same_results(ctx):
    """paper_2207_11428_b200.partition.SmPartition (green contexts): simulations launched on
    either SM group's streams -- miso on one, nopart and the chosen-only static search on the
    other, concurrently -- give the bytes of the shared-GPU runs."""
    import paper_2207_11428_b200 as m
    from paper_2207_11428_b200.partition import SmPartition
    tr = m.generate_traces_device(ctx, np.arange(48, dtype=np.uint64), 300, lambda_s=20.0)
    om = m.SimOptions(policy="miso", cluster_size=16, predictor="noisy")
    on = m.SimOptions(policy="nopart", cluster_size=16)
    want_m = m.simulate_batch(ctx, tr, om).metrics
    want_n = m.simulate_batch(ctx, tr, on).metrics
    want_s = m.best_static_partition(ctx, tr, cluster_size=16, chosen_only=True)
    part = SmPartition(0, 56)
    c2, c3 = m.Context(0), m.Context(0)
    try:
        (s_m,), (s_n, s_s) = part.streams(0, 1), part.streams(1, 2)
        assert part.sms[0] >= 8 and part.sms[1] >= 8
        pm = m.simulate_batch(ctx, tr, om, stream=s_m, defer=True)
        pn = m.simulate_batch(c2, tr, on, stream=s_n, defer=True)
        st = m.best_static_partition(c3, tr, cluster_size=16, stream=s_s, chosen_only=True)
        assert pm().metrics.tobytes() == want_m.tobytes()
        assert pn().metrics.tobytes() == want_n.tobytes()
        assert [e for e, _ in st] == [e for e, _ in want_s]
    finally:
        c2.close()
        c3.close()
        part.close()
