"""GPU parity tests for kernel (b), the batched partition search, through the C ABI.

Bar: bit-exact candidate, placement and FP64 objective versus the oracle (oracle/, itself
pinned to the reference's golden vectors in test_oracle.py) and the golden fixtures.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def check_against(ctx, speeds, offsets, entry, place, obj, cand=None, got_obj=None):
    if cand is None:
        cand, got_obj = ctx.optimize_batch(speeds, offsets)
    e, p = ctx.decode(cand, offsets)
    assert np.array_equal(e, entry.astype(np.int32)), np.nonzero(e != entry)[0][:10]
    feas = np.repeat(entry >= 0, np.diff(offsets.astype(np.int64)))
    assert np.array_equal(p[feas], place[: len(feas)][feas])
    assert np.array_equal(bits(got_obj), bits(obj))


@pytest.mark.parametrize("name", ["opt_random_0b5e55ed", "opt_accept_acce91", "opt_ties_71e5"])
def test_golden_host_path(ctx, golden, name):
    g = np.load(golden / f"{name}.npz")
    check_against(ctx, g["speeds"], g["offsets"], g["entry"], g["place"], g["obj"])


@pytest.mark.parametrize("name", ["opt_random_0b5e55ed", "opt_ties_71e5"])
def test_golden_device_path(ctx, golden, name):
    import torch
    g = np.load(golden / f"{name}.npz")
    s = torch.from_numpy(g["speeds"]).cuda()
    o = torch.from_numpy(g["offsets"].astype(np.int32)).cuda()
    cand, obj = ctx.optimize_batch(s, o)
    torch.cuda.synchronize()
    check_against(ctx, g["speeds"], g["offsets"], g["entry"], g["place"], g["obj"],
                  cand.cpu().numpy(), obj.cpu().numpy())


def test_literal_cases_dropin(ctx, golden):
    """optimizer_test.cpp:29-106 through the reference-shaped single-instance API."""
    lit = json.loads((golden / "opt_literal.json").read_text())
    for name, case in lit.items():
        sp = np.array(case["speeds"]).reshape(-1, 5)
        jobs = [(f"j{i}", sp[i]) for i in range(len(sp))]
        r = ctx.optimize_partition(jobs)
        if case["entry"] < 0:
            assert r is None, name
            continue
        assert r.entry == case["entry"], name
        assert [a.slice for a in r.assignments] == case["place"], name
        assert float(r.objective).hex() == case["obj_hex"], name
        for i, a in enumerate(r.assignments):
            assert a.job_id == f"j{i}" and a.speed == sp[i, a.slice]
    r = ctx.optimize_partition([("j1", [0.3, 0.5, 0.85, 0.9, 1.0]), ("j2", [0.35, 0.4, 0.5, 0.6, 1.0])])
    assert r.partition_name == "3g+3g" and abs(r.objective - 1.35) < 1e-12


@pytest.mark.parametrize("server", [True, False])
@pytest.mark.parametrize("name", ["opt_accept_acce91", "opt_ties_71e5"])
def test_scalar_optimize_golden(ctx, golden, oracle, name, server):
    """miso_b200_optimize (the scalar optimize_partition drop-in: one search-only request per
    call to the resident decision server, or one decide_one_kernel launch per call with the
    server disabled) instance by instance against the golden decisions, then against the oracle
    on instances with NaN / inf / -0 / subnormal / > 1 speeds in every slot."""
    import paper_2207_11428_b200 as m
    g = np.load(golden / f"{name}.npz")
    off = g["offsets"].astype(np.int64)
    sp = g["speeds"].reshape(-1, 5)
    m.lib.miso_b200_decide_server(ctx._h, 2000 if server else 0)
    try:
        n = min(len(off) - 1, 600)
        for i in range(n):
            jobs = [(f"j{j}", sp[off[i] + j]) for j in range(off[i + 1] - off[i])]
            r = ctx.optimize_partition(jobs)
            if g["entry"][i] < 0:
                assert r is None, i
                continue
            assert r.entry == g["entry"][i], i
            assert [a.slice for a in r.assignments] == list(g["place"][off[i]:off[i + 1]]), i
            assert bits(r.objective) == bits(g["obj"][i]), i
        rng = np.random.default_rng(5)
        specials = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 5e-324, 1.5, 1e300, -1.0])
        for t in range(300):
            mm = int(rng.integers(1, 8))
            s5 = rng.uniform(0.05, 1.0, (mm, 5))
            hit = rng.random((mm, 5)) < 0.15
            s5[hit] = rng.choice(specials, int(hit.sum()))
            e, p, o = oracle.optimize_batch(s5.reshape(-1), np.array([0, mm], np.uint32))
            r = ctx.optimize_partition([(f"j{j}", s5[j]) for j in range(mm)])
            if e[0] < 0:
                assert r is None, t
                continue
            assert r.entry == e[0] and [a.slice for a in r.assignments] == list(p[:mm]), t
            assert bits(r.objective) == bits(o[0]), t
    finally:
        m.lib.miso_b200_decide_server(ctx._h, 2000)


def test_job_count_out_of_range(ctx):
    with pytest.raises(ValueError):
        ctx.optimize_partition([])
    with pytest.raises(ValueError):
        ctx.optimize_partition([("x", [1, 1, 1, 1, 1])] * 8)
    cand, obj = ctx.optimize_batch(np.ones(8 * 5), np.array([0, 0, 8, 8], np.uint32))
    assert list(cand) == [0xFE, 0xFE, 0xFE] and list(obj) == [0, 0, 0]


def test_host_path_rejects_malformed_offsets(ctx, oracle):
    """miso_b200_optimize_batch_host validates offsets chunk by chunk (131072 instances per
    chunk): a decrease or an offset beyond offsets[n] anywhere -- first chunk, a later chunk,
    the last entry -- fails with MISO_B200_E_MALFORMED and copies nothing out of bounds; a
    valid batch afterwards is still exact."""
    import paper_2207_11428_b200 as m
    n = 300_000
    rng = np.random.default_rng(3)
    mm = rng.integers(1, 8, n)
    offs = np.concatenate([[0], np.cumsum(mm)]).astype(np.uint32)
    sp = rng.random((int(offs[-1]), 5))
    for pos, val in ((5, None), (200_000, None), (n, None), (10, int(offs[-1]) + 100)):
        bad = offs.copy()
        bad[pos] = bad[pos - 1] - 1 if val is None else val
        with pytest.raises(m.MisoError) as ei:
            ctx.optimize_batch(sp[: int(max(bad[-1], 1))] if bad[-1] < offs[-1] else sp, bad)
        assert ei.value.code == -3
    cand, obj = ctx.optimize_batch(sp, offs)
    e, p, ob = oracle.optimize_batch(sp.reshape(-1), offs)
    ge, _ = ctx.decode(cand, offs)
    assert np.array_equal(ge, e.astype(np.int32))
    assert np.array_equal(obj.view(np.uint64), ob.view(np.uint64))


def test_empty_batch(ctx):
    cand, obj = ctx.optimize_batch(np.zeros(0), np.array([0], np.uint32))
    assert len(cand) == 0 and len(obj) == 0


def test_config2_million_vs_oracle(ctx, oracle):
    """Config 2 (1M acceptance-generator mixes) bit-exact against the oracle."""
    s, f = oracle.gen_mixes(0xACCE91, 1_000_000)
    e, p, o = oracle.optimize_batch(s, f)
    check_against(ctx, s, f, e, p, o)


def test_special_values(ctx, oracle):
    """NaN, +-inf, -0.0, subnormals, negatives: validity is exactly `v > 0`."""
    rng = np.random.default_rng(3)
    vals = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 5e-324, -1.0, 0.5, 1.0, 1e308, 0.25])
    sizes = rng.integers(1, 8, 20000)
    f = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    s = vals[rng.integers(0, len(vals), int(f[-1]) * 5)]
    e, p, o = oracle.optimize_batch(s, f)
    check_against(ctx, s, f, e, p, o)


def test_all_m7_and_all_m1_tiles(ctx, oracle):
    """Tiles at the maximum staged size (every instance m=7) and the minimum."""
    rng = np.random.default_rng(5)
    for m in (7, 1, 4):
        n = 3000
        f = (np.arange(n + 1) * m).astype(np.uint32)
        s = rng.uniform(0.01, 1.0, n * m * 5)
        e, p, o = oracle.optimize_batch(s, f)
        check_against(ctx, s, f, e, p, o)


def test_misaligned_device_base(ctx, oracle):
    """Speeds base pointer only 8-byte aligned (a view one row-element in)."""
    import torch
    s, f = oracle.gen_mixes(99, 5000)
    e, p, o = oracle.optimize_batch(s, f)
    buf = torch.zeros(len(s) + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(s).cuda()
    cand, obj = ctx.optimize_batch(buf[1:], torch.from_numpy(f.astype(np.int32)).cuda())
    torch.cuda.synchronize()
    check_against(ctx, s, f, e, p, o, cand.cpu().numpy(), obj.cpu().numpy())


def test_catalog_subset(ctx, oracle):
    """A file-loaded catalog (topology.hpp:276-326) is any subset of the 36 entries."""
    from oracle_lib import OrcCatalog
    import ctypes as C
    rng = np.random.default_rng(11)
    full = oracle.catalog_counts()
    s, f = oracle.gen_mixes(4242, 20000)
    try:
        for trial in range(4):
            keep = np.sort(rng.choice(36, size=int(rng.integers(3, 30)), replace=False))
            sub = full[keep]
            ctx.set_catalog(sub)
            cat = OrcCatalog()
            cat.n_entries = len(sub)
            for i, row in enumerate(sub):
                for k in range(5):
                    cat.counts[i][k] = int(row[k])
            n = len(f) - 1
            e = np.zeros(n, np.int16); p = np.zeros(int(f[-1]), np.uint8); o = np.zeros(n)
            oracle.lib.orc_optimize_batch(C.byref(cat), s, f, n, e, p, o)
            check_against(ctx, s, f, e, p, o)
    finally:
        ctx.set_catalog(full)


def test_invalid_catalog_rejected(ctx):
    import paper_2207_11428_b200 as m
    with pytest.raises(m.MisoError) as ei:
        ctx.set_catalog([[0, 0, 1, 1, 0]])  # 4g + 3g cannot co-exist
    assert ei.value.code == -2
    with pytest.raises(m.MisoError):
        ctx.set_catalog([[1, 0, 0, 0, 0], [1, 0, 0, 0, 0]])  # duplicate


def test_full_size_properties(ctx, oracle):
    """At 8M instances: every decision is consistent with its own inputs (placement speeds
    > 0, objective == job-order sum, partition size == m), and a sampled slice matches the
    oracle exactly."""
    import torch
    s, f = oracle.gen_mixes(0xB200, 8_000_000)
    ds = torch.from_numpy(s).cuda()
    df = torch.from_numpy(f.astype(np.int32)).cuda()
    cand, obj = ctx.optimize_batch(ds, df)
    cand = cand.cpu().numpy(); obj = obj.cpu().numpy()
    ent, ms, pl = ctx.candidate_table()
    m = np.diff(f.astype(np.int64))
    ok = cand < 111
    assert np.all(cand[~ok] == 0xFF)
    assert np.array_equal(ms[cand[ok]], m[ok])
    sp = s.reshape(-1, 5)
    acc = np.zeros(ok.sum())
    idx = np.nonzero(ok)[0]
    for j in range(7):
        has = m[idx] > j
        rows = f[idx[has]].astype(np.int64) + j
        v = sp[rows, pl[cand[idx[has]], j]]
        assert np.all(v > 0)
        acc[has] = acc[has] + v
    assert np.array_equal(bits(acc), bits(obj[ok]))
    sl = slice(3_000_000, 3_050_000)
    sub_f = (f[sl.start: sl.stop + 1] - f[sl.start]).astype(np.uint32)
    sub_s = s[int(f[sl.start]) * 5: int(f[sl.stop]) * 5]
    e, p, o = oracle.optimize_batch(sub_s, sub_f)
    check_against(ctx, sub_s, sub_f, e, p, o, cand[sl], obj[sl])


def test_simple_tile_path_subprocess(golden):
    """The one-shot tile kernel (unaligned inputs / MISO_B200_SIMPLE_SEARCH=1) stays exact."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2207_11428_b200 as m
ctx = m.Context(0)
for name in ("opt_random_0b5e55ed", "opt_accept_acce91", "opt_ties_71e5"):
    g = np.load(f"tests/golden/{name}.npz")
    cand, obj = ctx.optimize_batch(g["speeds"], g["offsets"])
    e, p = ctx.decode(cand, g["offsets"])
    assert np.array_equal(e, g["entry"].astype(np.int32)), name
    assert np.array_equal(obj.view(np.uint64), g["obj"].view(np.uint64)), name
print("ok")
'''
    root = golden.parent.parent
    env = dict(os.environ, MISO_B200_SIMPLE_SEARCH="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_spare_slice_table_matches_oracle(ctx, oracle):
    """miso_b200_max_spare_slice -- the spare-slice table the simulator's placement reads --
    equals the oracle's max_spare_slice_for for every roster of up to 7 pinned kinds."""
    import itertools
    for n in range(8):
        for kinds in itertools.combinations_with_replacement(range(5), n):
            want = oracle.max_spare(list(kinds))
            got = ctx.max_spare_slice(list(kinds))
            assert (got if got is not None else -1) == want, (kinds, got, want)


def test_optimize_batches_equal_per_batch_calls(ctx, oracle):
    """miso_b200_optimize_batches: 40 batches (two launches of <= 32), empty batches, a batch
    whose speeds are only 8-byte aligned (one-shot tile kernel), sizes that are not multiples
    of the 256-instance tile, and one batch of 300k instances -- every batch's decisions and
    objective bits equal a separate optimize_batch call, and a sample equals the oracle."""
    import torch
    rng = np.random.default_rng(11)
    sizes = [int(x) for x in rng.integers(1, 5000, 37)] + [0, 300_000, 0]
    rng.shuffle(sizes)
    batches, want = [], []
    for i, n in enumerate(sizes):
        sp, off = oracle.gen_mixes(0x5EA + i, max(n, 1))
        if n == 0:
            sp, off = sp[:0], off[:1] * 0
        d_sp = torch.from_numpy(sp).cuda()
        if i == 5 and n:  # misaligned: an 8-byte offset view of a copy
            buf = torch.zeros(len(sp) + 1, dtype=torch.float64, device="cuda")
            buf[1:] = d_sp
            d_sp = buf[1:]
        d_off = torch.from_numpy(off.astype(np.int32)).cuda()
        c, o = ctx.optimize_batch(d_sp, d_off)
        want.append((c, o))
        batches.append((d_sp, d_off, torch.full((max(n, 1),), 0xAB, dtype=torch.uint8, device="cuda"),
                        torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")))
    ctx.optimize_batches(batches)
    torch.cuda.synchronize()
    for i, ((sp, off, c, o), (wc, wo)) in enumerate(zip(batches, want)):
        n = len(off) - 1
        assert torch.equal(c[:n], wc[:n]), i
        assert torch.equal(o[:n].view(torch.int64), wo[:n].view(torch.int64)), i
        if n == 0:
            assert int(c[0]) == 0xAB  # nothing written for an empty batch
    i = next(j for j, n in enumerate(sizes) if n > 100 and j != 5)
    sp, off = oracle.gen_mixes(0x5EA + i, sizes[i])
    e, p, obj = oracle.optimize_batch(sp, off)
    check_against(ctx, sp, off, e, p, obj, batches[i][2].cpu().numpy(), batches[i][3].cpu().numpy())


def test_optimize_batches_catalog_subset(oracle):
    """The queued entry on a context with a catalog subset (the kernel's masked-candidate
    instantiation): each batch equals its own optimize_batch call."""
    import torch
    import paper_2207_11428_b200 as m
    c = m.Context(0)
    try:
        full = c.catalog()
        c.set_catalog(full[::3])
        batches, want = [], []
        for i, n in enumerate([3000, 1, 257, 4096]):
            sp, off = oracle.gen_mixes(0x5B + i, n)
            d_sp, d_off = torch.from_numpy(sp).cuda(), torch.from_numpy(off.astype(np.int32)).cuda()
            want.append(c.optimize_batch(d_sp, d_off))
            batches.append((d_sp, d_off, torch.empty(n, dtype=torch.uint8, device="cuda"),
                            torch.empty(n, dtype=torch.float64, device="cuda")))
        c.optimize_batches(m.BatchList(batches))
        torch.cuda.synchronize()
        for (_, _, cc, oo), (wc, wo) in zip(batches, want):
            assert torch.equal(cc, wc) and torch.equal(oo.view(torch.int64), wo.view(torch.int64))
    finally:
        c.close()
