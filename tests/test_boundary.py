"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every symbol that
include/miso_b200.h declares; the generated candidate table agrees with the oracle; the
product path fails loudly without a GPU (no CPU fallback)."""
import ctypes as C
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "miso_b200.h"
LIB = ROOT / "paper_2207_11428_b200" / "_lib" / "libmiso_b200.so"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(miso_b200_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("miso_b200_create", "miso_b200_optimize_batch", "miso_b200_optimize_batch_host",
              "miso_b200_set_catalog"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "build the CUDA library first (__graft_entry__.build())"
    lib = C.CDLL(str(LIB))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (miso_b200_\w+)", out))
    assert exported == set(declared_symbols()), exported ^ set(declared_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_dfma_in_search_kernels():
    """FP64 parity needs un-contracted DMUL/DADD (SURVEY.md 7.4 hard part 1). The search
    kernels are pure DADD; elsewhere DFMA may only come from libdevice math (log/cos)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    search = [f for f in funcs if "optimize_" in f.split("\n")[0]]
    assert search, "no search kernels found"
    for f in search:
        assert "DADD" in f
        assert "DFMA" not in f, f.split("\n")[0]


def test_generated_candidates_up_to_date(tmp_path):
    dst = tmp_path / "c.cuh"
    subprocess.run([sys.executable, str(ROOT / "tools" / "gen_candidates.py"), str(dst)], check=True,
                   capture_output=True)
    cur = (ROOT / "paper_2207_11428_b200" / "csrc" / "candidates_gen.cuh").read_text()
    assert dst.read_text() == cur


def test_generated_candidates_match_oracle(oracle):
    sys.path.insert(0, str(ROOT / "tools"))
    import gen_candidates as g
    cands = g.candidates()
    c = oracle.candidates()
    assert len(cands) == c.n == 111
    for i, d in enumerate(cands):
        assert d["entry"] == c.entry[i] and d["m"] == c.m[i]
        assert d["place"] == list(c.place[i])[: d["m"]]
    assert [tuple(x) for x in g.catalog()] == [tuple(x) for x in oracle.catalog_counts()]


def test_python_catalog_mirror(oracle):
    from paper_2207_11428_b200.catalog import DEFAULT_CATALOG, partition_name
    assert np.array_equal(np.array(DEFAULT_CATALOG, np.uint8), oracle.catalog_counts())
    assert partition_name((0, 2, 1, 0, 0)) == "3g+2g+2g"


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2207_11428_b200 as m
    with pytest.raises(m.MisoError) as ei:
        m.Context(0)
    assert ei.value.code == -1


def test_default_model_host_fit_matches_reference(golden):
    """miso_b200_default_model is host code (no GPU): bit-exact with the reference fit."""
    import paper_2207_11428_b200 as m
    g = np.load(golden / "predict_seed7.npz")
    w2, w1 = m.default_model()
    assert np.array_equal(w2.view(np.uint64), g["w2"].view(np.uint64))
    assert np.array_equal(w1.view(np.uint64), g["w1"].view(np.uint64))


def test_dropin_sim_binaries_never_reach_the_reference_engine(tmp_path):
    """The reference's sim / experiment / acceptance test files, compiled with -fno-inline
    against the B200 binding (tools/dropin), carry no symbol of the reference's CPU engine
    (SimEngine members, run_simulation, best_static_partition, run_experiment[_in_memory],
    optsta_search, run_trial_unit): every simulation they run goes to the device. Positive
    control: the same flags on a file that calls the reference's run_simulation do emit them."""
    import re
    import shutil
    import subprocess
    bins = ROOT / "tools" / "dropin" / "_bin"
    if not (bins / "sim_test_b200").exists() or not shutil.which("nm"):
        pytest.skip("drop-in binaries not built")
    pat = re.compile(r" miso::(SimEngine::|(run_simulation|best_static_partition|"
                     r"run_experiment_in_memory|run_experiment|optsta_search|run_trial_unit)\()")
    for name in ("sim", "experiment", "acceptance"):
        syms = subprocess.run(["nm", "-C", str(bins / f"{name}_test_b200")], capture_output=True,
                              text=True, check=True).stdout
        hits = [ln for ln in syms.splitlines() if pat.search(ln)]
        assert not hits, (name, hits[:5])
        assert "miso::b200::" in syms, name
    ref = Path("/root/reference/proj/include")
    if ref.is_dir() and shutil.which("g++"):
        src = tmp_path / "ctl.cpp"
        src.write_text('#include "miso/sim.hpp"\nmiso::MetricsReport f(const miso::JobTrace& t) '
                       '{ miso::SimOptions o; return miso::run_simulation(t, o); }\n')
        obj = tmp_path / "ctl.o"
        subprocess.run(["g++", "-std=c++20", "-O2", "-fno-inline", f"-I{ref}", "-c", str(src),
                        "-o", str(obj)], check=True)
        syms = subprocess.run(["nm", "-C", str(obj)], capture_output=True, text=True).stdout
        assert pat.search(syms), "positive control: the reference engine's symbols must show"
