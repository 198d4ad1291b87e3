"""CPU tests: the device restatement of glibc 2.39's FMA-variant log()/cos()
(paper_2207_11428_b200/csrc/glibc_math.cuh) is bit-identical to the host libm on the
arguments DetRng::normal01 produces (common.hpp:103-108). Compiled for the host with g++ from
the same header the kernels use."""
import hashlib
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

CSRC = ROOT / "paper_2207_11428_b200" / "csrc"
LIBM = Path("/lib/x86_64-linux-gnu/libm.so.6")

PROG = r'''
#define __device__
#include <cstdio>
#include <cmath>
#include <random>
#include "glibc_math.cuh"
namespace miso_b200 { namespace glibc {
const uint64_t* host_log_tab = k_log_tab;
const uint64_t* host_sincostab = k_sincostab;
}}
using namespace miso_b200::glibc;
int main(int argc, char** argv) {
  std::mt19937_64 rng(std::stoull(argv[1]));
  long n = std::stol(argv[2]), bad = 0;
  for (long i = 0; i < n; ++i) {
    double u = (double)(rng() >> 11) * 0x1.0p-53;
    if (u <= 0) u = 0x1.0p-53;
    if (std::log(u) != log_fma(u)) ++bad;
    double x = 6.283185307179586476925287 * ((double)(rng() >> 11) * 0x1.0p-53);
    if (std::cos(x) != cos_fma(x)) ++bad;
    double v = 1.0 - (double)(rng() % 100000000) * 0x1.0p-53;  // log near-1 path
    if (std::log(v) != log_fma(v)) ++bad;
  }
  printf("%ld\n", bad);
  return 0;
}
'''


def host_has_fma_avx2() -> bool:
    flags = Path("/proc/cpuinfo").read_text()
    return " fma " in flags and " avx2 " in flags


@pytest.fixture(scope="module")
def prog(tmp_path_factory):
    if not host_has_fma_avx2():
        pytest.skip("host libm would select a non-FMA variant")
    d = tmp_path_factory.mktemp("gm")
    (d / "t.cpp").write_text(PROG)
    exe = d / "t"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", f"-I{CSRC}", str(d / "t.cpp"),
                    "-o", str(exe), "-lm"], check=True)
    return exe


@pytest.mark.parametrize("seed", [1, 2])
def test_log_cos_bit_exact_vs_host_libm(prog, seed):
    out = subprocess.run([str(prog), str(seed), "2000000"], capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "0"


def test_glibc_tables_up_to_date(tmp_path):
    if hashlib.md5(LIBM.read_bytes()).hexdigest() != "f8e590c62ca7258e57ee58b356a68ef6":
        pytest.skip("different libm build")
    dst = tmp_path / "g.cuh"
    subprocess.run([sys.executable, str(ROOT / "tools" / "extract_glibc_math.py"), str(dst)], check=True,
                   capture_output=True)
    assert dst.read_text() == (CSRC / "glibc_math_gen.cuh").read_text()
