"""Drop-in proof (GPU): the reference's own optimizer test file (proj/tests/optimizer_test.cpp,
compiled unmodified against include/miso_b200_ref.hpp by tools/dropin/Makefile) passes with
`optimize_partition` routed to the B200 kernels: fixed answers, 1000 random instances vs the
reference's brute-force oracle, scale invariance, 2-opt optimality, and the < 1 ms per call
budget."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent.parent / "tools" / "dropin" / "_bin" / "optimizer_test_b200"


def test_reference_optimizer_tests_against_b200():
    if not BIN.exists():
        pytest.skip("drop-in binary not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "11 tests, 0 failed" in r.stdout
