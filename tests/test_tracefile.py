"""CPU tests: trace files ("miso-trace v1", workload.hpp:122-245). save_trace output is
byte-identical to the reference's save_trace for the same generated trace; load_trace reads the
reference's files back to the exact arrays; malformed files fail with the reference reader's
ParseError line and message."""
import numpy as np
import pytest


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("seed,n,lam", [(0, 50, 60.0), (7, 300, 10.0), (2**40 + 3, 20, 5.0)])
def test_save_trace_byte_identical(ref, seed, n, lam):
    import paper_2207_11428_b200 as m
    from paper_2207_11428_b200 import tracefile as tf
    t = m.generate_trace(seed, n, lambda_s=lam)
    ours = tf.dumps(t, tf.TraceSpec(job_count=n, lambda_s=lam, seed=seed))
    assert ours == ref.trace_text(seed, n, lam)


def test_load_trace_roundtrip(ref, tmp_path):
    import paper_2207_11428_b200 as m
    from paper_2207_11428_b200 import tracefile as tf
    text = ref.trace_text(11, 120, 30.0)
    p = tmp_path / "t.trace"
    p.write_text(text)
    f = tf.load_trace(str(p))
    g = m.generate_trace(11, 120, lambda_s=30.0)
    assert f.spec.job_count == 120 and f.spec.lambda_s == 30.0 and f.spec.seed == 11
    assert f.job_ids == [f"j{i}" for i in range(120)]
    for a in ("arrival_s", "duration_s", "speeds5"):
        assert np.array_equal(bits(getattr(f.trace, a)), bits(getattr(g, a))), a
    assert np.array_equal(f.trace.mem_gb, g.mem_gb) and f.trace.qos_kind is None
    assert tf.dumps(f.trace, f.spec, job_ids=f.job_ids, mps_rates=f.mps_rates) == text


def _mutations(text):
    lines = text.split("\n")
    yield "\n".join(["miso-trace v2"] + lines[1:])
    yield "\n".join(lines[:1] + ["spek job_count=3"] + lines[2:])
    yield "\n".join(lines[:1] + [lines[1] + " colour=blue"] + lines[2:])
    yield "\n".join(lines[:1] + [lines[1].replace("dist=lognormal", "dist=gamma")] + lines[2:])
    yield "\n".join(lines[:1] + [lines[1].replace("lambda_s=10", "lambda_s=-1")] + lines[2:])
    yield "\n".join(lines[:2])
    yield "\n".join(lines[:2] + [lines[2].replace("f7", "f8")] + lines[3:])
    row = lines[5].split(",")
    for i, bad in [(1, "x"), (2, "1e999x"), (3, "12.5"), (4, "5"), (5, "0.9"), (6, "1.5"),
                   (2, "-3"), (3, "0"), (10, "0"), (0, ""), (1, "-1")]:
        r = list(row)
        r[i] = bad
        yield "\n".join(lines[:5] + [",".join(r)] + lines[6:])
    yield "\n".join(lines[:5] + [",".join(row[:12])] + lines[6:])
    yield "\n".join(lines[:5] + [lines[4]] + lines[6:])          # duplicate id
    yield "\n".join(lines[:3] + [lines[4], lines[3]] + lines[5:])  # first arrival != 0
    yield "\n".join(lines[:-2])                                      # job count mismatch
    yield "\n".join(lines[:4] + lines[5:]).replace(",", ",", 1)


def test_load_trace_errors_match_reference(ref):
    from paper_2207_11428_b200 import tracefile as tf
    text = ref.trace_text(3, 8, 10.0)
    assert ref.load_trace(text)[0] == 0
    n = 0
    for bad in _mutations(text):
        r_line, _, r_msg = ref.load_trace(bad)
        if r_line == 0:
            tf.loads(bad)  # both accept
            continue
        with pytest.raises(tf.ParseError) as ei:
            tf.loads(bad)
        assert str(ei.value) == r_msg, (bad.split("\n")[:6], r_msg)
        assert ei.value.line == r_line
        n += 1
    assert n >= 15
