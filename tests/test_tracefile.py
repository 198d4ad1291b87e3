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


def _profile_lines(ref):
    """Valid records (every line of a reference trace, minus its arrival field) and mutations
    that trip each of parse_profile_body's and validate_profile's checks."""
    text = ref.trace_text(5, 12, 10.0).split("\n")
    rows = [ln.split(",") for ln in text[3:] if ln]
    good = [",".join([r[0]] + r[2:]) for r in rows]
    yield from good
    base = good[3].split(",")
    for i, bad in [(1, "x"), (1, "0"), (1, "-2"), (1, " 3"), (1, "3 "), (1, "nan"), (1, "inf"),
                   (2, "0"), (2, "41"), (2, "7.5"), (2, "+5"), (2, "0x10"), (3, "5"), (3, "-1"),
                   (3, "2"), (4, "1.0000001"), (4, "0.5"), (5, "1.5"), (6, "0"), (7, "-0.1"),
                   (8, "1e-320"), (9, "0"), (10, "2"), (11, "nan"), (0, ""), (0, "a\rb"),
                   (5, "1e999"), (5, "0x1p-1"), (2, "99999999999"), (1, "nan(1)"), (2, " 5"),
                   (1, "1e-310"), (7, "0x1.8p-1"), (1, "INFINITY"), (2, "-0"), (3, "+4")]:
        r = list(base)
        r[i] = bad
        yield ",".join(r)
    yield ",".join(base[:11])
    yield ",".join(base + ["1"])
    yield ",".join(base) + "\r"
    yield ""


@pytest.mark.parametrize("lineno", [0, 7])
def test_profile_records_match_reference(ref, lineno):
    """parse_profile_record / format_profile_record (profiles.hpp:484-568) against the
    reference's: the same text back for every accepted line, the same ParseError line and
    message (or std::invalid_argument from validate_profile when lineno is 0) otherwise."""
    from paper_2207_11428_b200 import tracefile as tf
    n_ok = n_err = 0
    for line in _profile_lines(ref):
        r, want = ref.profile_record(line, lineno)
        if r == 0:
            assert tf.format_profile_record(tf.parse_profile_record(line, lineno)) == want, line
            n_ok += 1
            continue
        exc = ValueError if r == -2 else tf.ParseError
        with pytest.raises(exc) as ei:
            tf.parse_profile_record(line, lineno)
        if r != -2:
            assert isinstance(ei.value, tf.ParseError) and ei.value.line == (r if r > 0 else 0)
        else:
            assert not isinstance(ei.value, tf.ParseError)
        assert str(ei.value) == want, (line, want)
        n_err += 1
    assert n_ok >= 12 and n_err >= 25
