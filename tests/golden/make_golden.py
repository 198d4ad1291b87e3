#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run here (where /root/reference exists): `python tests/golden/make_golden.py`. Every output
value below comes from oracle/_ref/libmiso_ref.so, i.e. the unmodified reference headers
(optimize_partition, predict_mig_speeds, extrapolate_small_slices, max_spare_slice_for,
default_catalog, fit_small_slice_model, run_simulation). Inputs come from the reference's own
generators (DetRng streams) or from its tests' literal cases. The fixtures travel to the GPU
box, where /root/reference does not exist.

Host facts recorded in meta.json: glibc version and whether the FMA libm variants were active
(noisy-predictor bits depend on them at the ulp level, SURVEY.md 7.4 hard part 3).
"""
from __future__ import annotations

import itertools
import json
import os
import platform
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import PyDetRng, Ref  # noqa: E402


def pack(instances):
    offs = [0]
    rows = []
    for jobs in instances:
        rows.extend(jobs)
        offs.append(len(rows))
    return np.array(rows, np.float64).reshape(-1), np.array(offs, np.uint32)


def optimizer_random_jobs(ref: Ref, seed: int, trials: int):
    """optimizer_test.cpp:110-130 random_jobs stream."""
    rng = PyDetRng(ref.rng_raw(seed, trials * 7 * 6 + 16))
    out = []
    for _ in range(trials):
        m = 1 + rng.index(7)
        jobs = []
        for _ in range(m):
            f4 = rng.uniform(0.2, 1.0)
            f3 = rng.uniform(0.15, f4)
            f2 = rng.uniform(0.1, f3)
            f1 = rng.uniform(0.05, f2)
            u = rng.uniform01()
            if u < 0.18:
                f1 = 0.0
            elif u < 0.33:
                f1 = 0.0
                f2 = 0.0
            jobs.append([f1, f2, f3, f4, 1.0])
        out.append(jobs)
    return out


def tie_heavy_jobs(ref: Ref, seed: int, trials: int):
    """Speeds from a tiny value set so exact objective ties are common (tie-break stress)."""
    rng = PyDetRng(ref.rng_raw(seed, trials * 7 * 6 + 16))
    vals = [0.0, 0.25, 0.5, 0.75, 1.0]
    out = []
    for _ in range(trials):
        m = 1 + rng.index(7)
        out.append([[vals[rng.index(5)] for _ in range(5)] for _ in range(m)])
    return out


def literal_cases():
    """optimizer_test.cpp:29-106 fixed inputs (speeds listed 7g,4g,3g,2g,1g there)."""
    def desc(s):
        return [s[4], s[3], s[2], s[1], s[0]]
    return {
        "seven_linear": [desc([1.0, 4 / 7, 3 / 7, 2 / 7, 1 / 7])] * 7,
        "pair_3g3g": [desc([1.0, 0.9, 0.85, 0.5, 0.3]), desc([1.0, 0.6, 0.5, 0.4, 0.35])],
        "single_7g": [desc([1.0, 0.8, 0.7, 0.5, 0.3])],
        "flat_1g": [desc([1, 1, 1, 1, 1])],
        "zero_avoid": [desc([1.0, 0.9, 0.8, 0.6, 0.0]), desc([1.0, 0.5, 0.4, 0.3, 0.25])],
        "all_infeasible": [desc([1, 0, 0, 0, 0]), desc([1, 0, 0, 0, 0])],
    }


def main():
    ref = Ref()
    meta = {
        "generated_by": "tests/golden/make_golden.py via oracle/_ref (reference headers)",
        "glibc": platform.libc_ver()[1],
        "host_fma": "fma" in open("/proc/cpuinfo").read(),
        "machine": platform.machine(),
    }
    cat = ref.catalog_counts()
    np.save(HERE / "catalog.npy", cat)

    # optimizer fixtures -------------------------------------------------------------
    sets = {
        "opt_random_0b5e55ed": optimizer_random_jobs(ref, 0x0B5E55ED, 1000),
        "opt_ties_71e5": tie_heavy_jobs(ref, 0x71E5, 2000),
    }
    for name, inst in sets.items():
        speeds, offs = pack(inst)
        e, p, o = ref.optimize_batch(speeds, offs)
        np.savez_compressed(HERE / f"{name}.npz", speeds=speeds, offsets=offs, entry=e, place=p,
                            obj=o)
    speeds, offs = ref.gen_mixes(0xACCE91, 1000)
    e, p, o = ref.optimize_batch(speeds, offs)
    np.savez_compressed(HERE / "opt_accept_acce91.npz", speeds=speeds, offsets=offs, entry=e,
                        place=p, obj=o)
    lit = {}
    for name, jobs in literal_cases().items():
        speeds, offs = pack([jobs])
        e, p, o = ref.optimize_batch(speeds, offs)
        lit[name] = dict(speeds=speeds.tolist(), entry=int(e[0]), place=p[: len(jobs)].tolist(),
                         obj=float(o[0]), obj_hex=float(o[0]).hex())
    (HERE / "opt_literal.json").write_text(json.dumps(lit, indent=1))

    # predictor fixtures -------------------------------------------------------------
    w2, w1 = ref.default_model()
    truth3, small2 = ref.gen_profiles(7, 700)
    pred = {}
    for noisy in (0, 1):
        for mae in ((0.017, 0.05, 0.09) if noisy else (0.017,)):
            pred[f"out_n{noisy}_{mae}"] = ref.predict_batch(truth3, 7, 1, 7, noisy, mae)
    # cols-per-group 3 (a 3-job roster padded with 4 dummies), nonce base 41
    pred["out_cpg3"] = ref.predict_batch(truth3[: 3 * 99], 3, 41, 12345, 1, 0.017)
    np.savez_compressed(HERE / "predict_seed7.npz", truth3=truth3, small2=small2, w2=w2, w1=w1,
                        **pred)

    # spare-slice LUT over every sorted multiset of <= 6 min kinds ---------------------
    keys, vals = [], []
    for m in range(7):
        for ks in itertools.combinations_with_replacement(range(5), m):
            keys.append(list(ks) + [-1] * (6 - m))
            vals.append(ref.lib.ref_max_spare_slice_for(np.array(ks, np.int32), m))
    np.savez_compressed(HERE / "spare_lut.npz", kinds=np.array(keys, np.int8),
                        spare=np.array(vals, np.int8))

    # config 1 anchor ----------------------------------------------------------------
    c1 = ref.c1_chain()
    (HERE / "c1_anchor.json").write_text(json.dumps(
        {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in c1.items()} |
        {"obj_hex": float(c1["obj"]).hex(),
         "partition": "+".join(["1g", "2g", "3g", "4g", "7g"][k] for k in range(4, -1, -1)
                               for _ in range(int(cat[c1["entry"]][k])))}, indent=1))

    (HERE / "meta.json").write_text(json.dumps(meta, indent=1))
    for f in sorted(HERE.iterdir()):
        if f.suffix in (".npz", ".npy", ".json"):
            print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
