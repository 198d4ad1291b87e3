"""GPU parity tests for kernel (a), the batched MPS->MIG predictor, and the fused
predictor -> effective_speed -> search decision kernel.

Bars (north_star): predicted speeds within 1e-5 relative of the reference, partition
decisions bit-exact. The kernel restates glibc 2.39's FMA-variant log/cos bit-exactly
(glibc_math.cuh), so the predicted speeds are asserted bit-identical as well.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MEM = np.array([5, 10, 20, 20, 40])
GPC = np.array([1, 2, 3, 4, 7])


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def zero_eff(est, mem, qos):
    """effective_speed (profiles.hpp:60-65) on (n,5) tables."""
    out = est.copy()
    out[MEM[None, :] < mem[:, None]] = 0.0
    q = np.where(qos >= 0, GPC[np.maximum(qos, 0)], 0)
    out[GPC[None, :] < q[:, None]] = 0.0
    return out


def test_oracle_mode_bit_exact(ctx, golden):
    g = np.load(golden / "predict_seed7.npz")
    out = ctx.predict_batch(g["truth3"], 7, 1, 7, 0, 0.017).cpu().numpy().reshape(-1)
    assert np.array_equal(bits(out), bits(g["out_n0_0.017"]))


@pytest.mark.parametrize("mae", [0.017, 0.05, 0.09])
def test_noisy_mode_vs_reference_golden(ctx, golden, mae):
    g = np.load(golden / "predict_seed7.npz")
    out = ctx.predict_batch(g["truth3"], 7, 1, 7, 1, mae).cpu().numpy().reshape(-1)
    want = g[f"out_n1_{mae}"]
    assert np.array_equal(bits(out), bits(want))


def test_noisy_cpg3_golden(ctx, golden):
    g = np.load(golden / "predict_seed7.npz")
    out = ctx.predict_batch(g["truth3"][: 3 * 99], 3, 41, 12345, 1, 0.017).cpu().numpy().reshape(-1)
    assert np.array_equal(bits(out), bits(g["out_cpg3"]))


def test_noisy_mode_million_vs_oracle(ctx, oracle):
    """Config-3 stream at 1M profiles: report the ulp-mismatch rate, bound the error."""
    t, _ = oracle.gen_profiles(3, 1_000_000)
    want = oracle.predict_batch(t, 7, 1, 3, 1, 0.017)
    out = ctx.predict_batch(t, 7, 1, 3, 1, 0.017).cpu().numpy().reshape(-1)
    mism = int((bits(out) != bits(want)).sum())
    print(f"noisy predictor: {mism} of {out.size} entries differ from the glibc-based oracle")
    assert mism == 0
    oracle_mode = ctx.predict_batch(t, 7, 1, 3, 0, 0.017).cpu().numpy().reshape(-1)
    assert np.array_equal(bits(oracle_mode), bits(oracle.predict_batch(t, 7, 1, 3, 0, 0.017)))


def test_zero_mae_equals_oracle(ctx, oracle):
    """profiles_test.cpp:233-248: target_mae 0 in noisy mode == oracle mode."""
    t, _ = oracle.gen_profiles(11, 7000)
    a = ctx.predict_batch(t, 7, 1, 5, 1, 0.0).cpu().numpy()
    b = ctx.predict_batch(t, 7, 1, 5, 0, 0.0).cpu().numpy()
    assert np.array_equal(bits(a), bits(b))


def test_determinism_and_nonce_decorrelation(ctx, oracle):
    """profiles_test.cpp:163-195: same (seed, nonce) -> same output; anchor row stays 1."""
    t, _ = oracle.gen_profiles(12, 700)
    a = ctx.predict_batch(t, 7, 5, 9, 1, 0.05).cpu().numpy()
    b = ctx.predict_batch(t, 7, 5, 9, 1, 0.05).cpu().numpy()
    c = ctx.predict_batch(t, 7, 6, 9, 1, 0.05).cpu().numpy()
    assert np.array_equal(bits(a), bits(b))
    assert not np.array_equal(a[:, 3], c[:, 3])
    assert np.all(a[:, 4] == 1.0)
    assert np.all((a > 0) & (a <= 1.0))
    assert np.all(a[:, 0] <= a[:, 1]) and np.all(a[:, 1] <= a[:, 2])  # f1 <= f2 <= f3


@pytest.mark.parametrize("mae", [0.017, 0.05, 0.09])
def test_mae_calibration(ctx, oracle, mae):
    """profiles_test.cpp:199-231: empirical MAE of the 4g/3g entries within 2 SE of target."""
    t, _ = oracle.gen_profiles(21, 7 * 1500)
    out = ctx.predict_batch(t, 7, 1, 77, 1, mae).cpu().numpy()
    tt = t.reshape(-1, 3)
    err = np.concatenate([np.abs(out[:, 3] - tt[:, 1]), np.abs(out[:, 2] - tt[:, 2])])
    se = err.std(ddof=1) / np.sqrt(len(err))
    assert abs(err.mean() - mae) <= 2 * se + 1e-3, (err.mean(), se)


def test_invalid_predictor_spec(ctx):
    import paper_2207_11428_b200 as m
    t = np.ones(3 * 7)
    for mode, mae in ((1, -0.1), (1, 0.6), (3, 0.017)):
        with pytest.raises(m.MisoError) as ei:
            ctx.predict_batch(t, 7, 1, 0, mode, mae)
        assert ei.value.code == -2


def test_config1_anchor_through_dropin(ctx, golden):
    """Config 1 (the reference CPU example): 3 jobs -> noisy predictor (seed 7, nonce 1)
    -> default model -> effective_speed -> optimize_partition == 3g+2g+2g, 1.6533152344307642."""
    a = json.loads((golden / "c1_anchor.json").read_text())
    t = np.array(a["truth3"]).reshape(3, 3)
    jobs = [(f"j{i}", t[i], a["mem"][i], None) for i in range(3)]
    r, est = ctx.decide(jobs, nonce=1, rng_seed=7, mode=1, target_mae=0.017)
    assert r.partition_name == "3g+2g+2g"
    assert float(r.objective).hex() == a["obj_hex"]
    assert [x.slice for x in r.assignments] == a["place"]
    want = np.array(a["est5"]).reshape(3, 5)
    assert np.array_equal(bits(est), bits(want))


def test_decide_batch_vs_oracle_chain(ctx, oracle):
    """Fused kernel == oracle predictor + effective_speed + oracle optimizer on random rosters
    (decisions bit-exact; sizes 1..7, memory 5/10/20/40 GB, QoS floors)."""
    rng = np.random.default_rng(8)
    n = 20000
    m = rng.integers(1, 8, n)
    offs = np.concatenate([[0], np.cumsum(m)]).astype(np.uint32)
    J = int(offs[-1])
    t, _ = oracle.gen_profiles(31, J)
    mem = rng.choice([5, 10, 20, 40], J, p=[0.45, 0.3, 0.2, 0.05]).astype(np.uint8)
    qos = np.where(rng.random(J) < 0.15, rng.integers(0, 5, J), -1).astype(np.int8)
    nonce = rng.integers(1, 1 << 40, n).astype(np.uint64)
    seed = 1234
    # oracle chain
    w2, w1 = oracle.default_model()
    est = np.zeros((J, 5))
    import ctypes as C
    for i in range(n):
        o, mm = int(offs[i]), int(m[i])
        est[o:o + mm] = oracle.predict_batch(t[3 * o: 3 * (o + mm)], mm, int(nonce[i]), seed, 1,
                                             0.017, w2, w1).reshape(mm, 5)
    est = zero_eff(est, mem.astype(int), qos.astype(int))
    e, p, ob = oracle.optimize_batch(est.reshape(-1), offs)
    cand, obj, dest = ctx.decide_batch(t, mem, qos, offs, nonce, seed, 1, 0.017, want_est=True)
    dest = dest.cpu().numpy().reshape(-1, 5)
    assert np.array_equal(bits(dest), bits(est))
    ge, gp = ctx.decode(cand.cpu().numpy(), offs)
    assert np.array_equal(ge, e.astype(np.int32))
    feas = np.repeat(e >= 0, m)
    assert np.array_equal(gp[feas], p[feas])
    assert np.array_equal(bits(obj.cpu().numpy()), bits(ob))


def test_decide_server_matches_launch_mode(ctx, oracle):
    """miso_b200_decide through the resident server == one launch per call == the oracle chain,
    with and without the server's draw-ahead (consecutive / random nonces), across server idle-outs (relaunch with a pending request), catalog changes between calls
    and host-pipeline calls that stop the server."""
    import time
    rng = np.random.default_rng(11)
    w2, w1 = oracle.default_model()
    cases = []
    for i in range(60):
        m = int(rng.integers(1, 8))
        t, _ = oracle.gen_profiles(100 + i, m)
        mem = rng.choice([5, 10, 20, 40], m).astype(np.uint8)
        qos = np.where(rng.random(m) < 0.2, rng.integers(0, 5, m), -1).astype(np.int8)
        jobs = [(f"j{c}", tuple(t[3 * c:3 * c + 3]), int(mem[c]), None if qos[c] < 0 else int(qos[c]))
                for c in range(m)]
        # runs of consecutive call nonces (the server's draw-ahead hits) broken by random ones
        cases.append((jobs, 5000 + i if i % 3 else int(rng.integers(1, 1 << 40))))

    from paper_2207_11428_b200.catalog import DEFAULT_CATALOG
    full = [list(c) for c in DEFAULT_CATALOG]

    def run(idle_us, pause_every=0, poke=False, catalog=None):
        ctx.decide_server(idle_us)
        out = []
        for k, (jobs, nonce) in enumerate(cases):
            if pause_every and k % pause_every == pause_every - 1:
                time.sleep(0.01)  # longer than the idle window: the server exits meanwhile
            if catalog is not None:
                ctx.set_catalog(catalog if k % 2 else full)
            if poke and k % 7 == 3:  # growing host batches: scratch is reallocated (cudaFree)
                n = 5000 * (k + 1)
                ctx.optimize_batch(np.ones((n, 5)), np.arange(n + 1, dtype=np.uint32))
            r, est = ctx.decide(jobs, nonce=nonce, rng_seed=5, mode=1, target_mae=0.017)
            out.append((None if r is None else (r.entry, tuple(a.slice for a in r.assignments),
                                                 np.float64(r.objective).view(np.uint64)),
                        bits(est)))
        return out

    sub = [c for c in full if c[4] == 0][::2]  # a catalog without 7g, changed between calls
    try:
        launched = run(0)
        served = run(2000)
        idled = run(200, pause_every=5)
        poked = run(2000, poke=True)
        sub_launched = run(0, catalog=sub)
        sub_served = run(2000, catalog=sub)
    finally:
        ctx.decide_server(2000)
        ctx.set_catalog(full)
    for a, b, c, d in zip(launched, served, idled, poked):
        assert a[0] == b[0] == c[0] == d[0]
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[1], c[1]) and np.array_equal(a[1], d[1])
    for a, b in zip(sub_launched, sub_served):
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
    assert any(a[0] != b[0] for a, b in zip(launched, sub_launched))
    # the chain itself against the oracle for the served results
    for (jobs, nonce), (res, est_bits) in zip(cases, served):
        m = len(jobs)
        t3 = np.array([j[1] for j in jobs], np.float64).reshape(-1)
        est = oracle.predict_batch(t3, m, nonce, 5, 1, 0.017, w2, w1).reshape(m, 5)
        est = zero_eff(est, np.array([j[2] for j in jobs]), np.array([-1 if j[3] is None else j[3] for j in jobs]))
        assert np.array_equal(bits(est), est_bits)


def test_decide_server_option_checked(ctx):
    import paper_2207_11428_b200 as m
    with pytest.raises(m.MisoError) as ei:
        ctx.decide_server(-1)
    assert ei.value.code == -2
