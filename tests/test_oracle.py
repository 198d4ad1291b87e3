"""CPU tests: the C restatement (oracle/) pinned against the reference's golden vectors.

Golden fixtures in tests/golden/ were produced by the unmodified reference (oracle/_ref, see
tests/golden/make_golden.py). The oracle must reproduce them bit-for-bit before it is trusted
as the checker of the CUDA path.
"""
import json

import numpy as np
import pytest


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def test_catalog_matches_reference(oracle, golden):
    cat = oracle.catalog_counts()
    assert cat.shape == (36, 5)
    assert np.array_equal(cat, np.load(golden / "catalog.npy"))
    # topology_test.cpp:148-156: first 7g, last 1g
    assert list(cat[0]) == [0, 0, 0, 0, 1] and list(cat[-1]) == [1, 0, 0, 0, 0]


def test_candidate_counts(oracle):
    c = oracle.candidates()
    assert c.n == 111
    per_m = [c.base[m + 1] - c.base[m] for m in range(1, 8)]
    assert per_m == [5, 13, 29, 35, 21, 7, 1]


@pytest.mark.parametrize("name", ["opt_random_0b5e55ed", "opt_accept_acce91", "opt_ties_71e5"])
def test_optimizer_golden(oracle, golden, name):
    g = np.load(golden / f"{name}.npz")
    e, p, o = oracle.optimize_batch(g["speeds"], g["offsets"])
    assert np.array_equal(e, g["entry"])
    feas = np.repeat(g["entry"] >= 0, np.diff(g["offsets"].astype(np.int64)))
    assert np.array_equal(p[: len(feas)][feas], g["place"][: len(feas)][feas])
    assert np.array_equal(bits(o), bits(g["obj"]))


def test_optimizer_golden_feasible_fraction(golden):
    # optimizer_test.cpp:156-159: 500 < feasible < 950 for seed 0x0b5e55ed
    g = np.load(golden / "opt_random_0b5e55ed.npz")
    assert 500 < int((g["entry"] >= 0).sum()) < 950
    # acceptance_test.cpp:115: feasible > 700
    g = np.load(golden / "opt_accept_acce91.npz")
    assert int((g["entry"] >= 0).sum()) > 700


def test_optimizer_literal_cases(oracle, golden):
    lit = json.loads((golden / "opt_literal.json").read_text())
    cat = oracle.catalog_counts()
    names = {tuple(c): i for i, c in enumerate(cat)}
    for name, case in lit.items():
        sp = np.array(case["speeds"])
        m = len(sp) // 5
        e, p, o = oracle.optimize_batch(sp, np.array([0, m], np.uint32))
        assert e[0] == case["entry"], name
        if e[0] >= 0:
            assert list(p[:m]) == case["place"], name
            assert float(o[0]).hex() == case["obj_hex"], name
    # optimizer_test.cpp expectations restated
    assert lit["pair_3g3g"]["entry"] == names[(0, 0, 2, 0, 0)]
    assert lit["single_7g"]["entry"] == names[(0, 0, 0, 0, 1)]
    assert lit["flat_1g"]["entry"] == names[(1, 0, 0, 0, 0)]
    assert lit["seven_linear"]["entry"] == names[(7, 0, 0, 0, 0)]
    assert lit["all_infeasible"]["entry"] == -1


def test_optimizer_bad_m(oracle):
    sp = np.ones(8 * 5)
    e, _, _ = oracle.optimize_batch(sp, np.array([0, 0, 8], np.uint32))
    assert list(e) == [-2, -2]


def test_default_model(oracle, golden):
    g = np.load(golden / "predict_seed7.npz")
    w2, w1 = oracle.default_model()
    assert np.array_equal(bits(w2), bits(g["w2"])) and np.array_equal(bits(w1), bits(g["w1"]))
    # SURVEY.md 8(a) a10 probe values
    assert w2[1] == 0.26129028483659655 and w1[2] == 1.2887601594439484


def test_profiles_stream(oracle, golden):
    g = np.load(golden / "predict_seed7.npz")
    t, s = oracle.gen_profiles(7, 700)
    assert np.array_equal(bits(t), bits(g["truth3"])) and np.array_equal(bits(s), bits(g["small2"]))


@pytest.mark.parametrize("key,noisy,mae", [("out_n0_0.017", 0, 0.017), ("out_n1_0.017", 1, 0.017),
                                           ("out_n1_0.05", 1, 0.05), ("out_n1_0.09", 1, 0.09)])
def test_predictor_golden(oracle, golden, key, noisy, mae):
    g = np.load(golden / "predict_seed7.npz")
    out = oracle.predict_batch(g["truth3"], 7, 1, 7, noisy, mae)
    assert np.array_equal(bits(out), bits(g[key]))


def test_predictor_golden_cpg3(oracle, golden):
    g = np.load(golden / "predict_seed7.npz")
    out = oracle.predict_batch(g["truth3"][: 3 * 99], 3, 41, 12345, 1, 0.017)
    assert np.array_equal(bits(out), bits(g["out_cpg3"]))


def test_predictor_oracle_mode_is_truth(oracle, golden):
    # profiles_test.cpp:137-161: oracle predictor returns the truth rows
    g = np.load(golden / "predict_seed7.npz")
    out = oracle.predict_batch(g["truth3"], 7, 1, 7, 0, 0.017).reshape(-1, 5)
    t = g["truth3"].reshape(-1, 3)
    assert np.array_equal(out[:, 4], t[:, 0]) and np.array_equal(out[:, 3], t[:, 1])
    assert np.array_equal(out[:, 2], t[:, 2])


def test_spare_lut_golden(oracle, golden):
    g = np.load(golden / "spare_lut.npz")
    for ks, want in zip(g["kinds"], g["spare"]):
        k = [int(x) for x in ks if x >= 0]
        assert oracle.max_spare(k[::-1]) == want


def test_c1_anchor(oracle, golden):
    """Config 1: 3 jobs -> noisy predictor -> extrapolate -> effective_speed -> optimize."""
    a = json.loads((golden / "c1_anchor.json").read_text())
    assert a["partition"] == "3g+2g+2g" and a["obj_hex"] == (1.6533152344307642).hex()
    t = np.array(a["truth3"])
    pred = oracle.predict_batch(t, 3, 1, 7, 1, 0.017).reshape(-1, 5)
    mem = a["mem"]
    memgb = [5, 10, 20, 20, 40]
    est = np.array([[pred[j, k] if memgb[k] >= mem[j] else 0.0 for k in range(5)] for j in range(3)])
    assert np.array_equal(bits(est.reshape(-1)), bits(a["est5"]))
    e, p, o = oracle.optimize_batch(est.reshape(-1), np.array([0, 3], np.uint32))
    assert e[0] == a["entry"] and list(p[:3]) == a["place"] and float(o[0]).hex() == a["obj_hex"]


def test_oracle_vs_reference_large(oracle, ref):
    """Beyond the fixtures: 200k config-2 mixes, oracle == reference bit-for-bit."""
    s, f = ref.gen_mixes(0x5EED5, 200_000)
    s2, f2 = oracle.gen_mixes(0x5EED5, 200_000)
    assert np.array_equal(bits(s), bits(s2)) and np.array_equal(f, f2)
    a = oracle.optimize_batch(s, f)
    b = ref.optimize_batch(s, f, threads=4)
    assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[2]), bits(b[2]))
    feas = np.repeat(a[0] >= 0, np.diff(f.astype(np.int64)))
    assert np.array_equal(a[1][feas], b[1][feas])
