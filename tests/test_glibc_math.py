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


PROG2 = r'''
#define __device__
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <random>
#include "glibc_math2.cuh"
namespace miso_b200 { namespace glibc {
const uint64_t* host_log_tab = k_log_tab;
const uint64_t* host_sincostab = k_sincostab;
const uint64_t* host_exp_tab = k_exp_tab;
const uint64_t* host_pow_tab = k_pow_tab;
}}
using namespace miso_b200::glibc;
static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0 || (std::isnan(a) && std::isnan(b)); }
int main(int argc, char** argv) {
  std::mt19937_64 rng(std::stoull(argv[1]));
  long n = std::stol(argv[2]);
  long bad_e = 0, bad_p = 0, bad_l = 0;
  auto u01 = [&]() { return (double)(rng() >> 11) * 0x1.0p-53; };
  for (long i = 0; i < n; ++i) {
    // exp: lognormal domain, wide range, tiny, large
    double xs[5] = {8.88 - 1.92 + 1.5 * (u01() * 17 - 8.5), (u01() - 0.5) * 1400, (u01() - 0.5) * 1e-15,
                    (u01() - 0.5) * 60, 500 + u01() * 240};
    for (double x : xs) if (!same(std::exp(x), exp_fma(x))) { if (bad_e < 5) printf("exp %a: %a vs %a\n", x, std::exp(x), exp_fma(x)); ++bad_e; }
    // pow: generator's (g/7)^alpha, plus random positive bases
    const double gs[5] = {1, 2, 3, 4, 7};
    double al = 0.1 + (1.0 - 0.1) * u01();
    for (double g : gs) { double x = g / 7.0; if (!same(std::pow(x, al), pow_fma(x, al))) { if (bad_p < 5) printf("pow %a %a\n", x, al); ++bad_p; } }
    double x = u01() * 20, y = (u01() - 0.5) * 40;
    if (!same(std::pow(x, y), pow_fma(x, y))) { if (bad_p < 5) printf("pow %a %a: %a vs %a\n", x, y, std::pow(x, y), pow_fma(x, y)); ++bad_p; }
    // log1p: the generator's -u, plus wide / tiny / near -1 / large
    double ls[6] = {-u01(), (u01() - 0.5) * 1e-12, -1 + u01() * 1e-6, u01() * 100, (u01()) * 0.9 - 0.45, u01() * 1e20};
    for (double v : ls) if (!same(std::log1p(v), log1p_fma(v))) { if (bad_l < 5) printf("log1p %a: %a vs %a\n", v, std::log1p(v), log1p_fma(v)); ++bad_l; }
  }
  printf("exp %ld pow %ld log1p %ld mismatches over %ld rounds\n", bad_e, bad_p, bad_l, n);
  return (bad_e || bad_p || bad_l) ? 1 : 0;
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


@pytest.fixture(scope="module")
def prog2(tmp_path_factory):
    if not host_has_fma_avx2():
        pytest.skip("host libm would select a non-FMA variant")
    d = tmp_path_factory.mktemp("gm2")
    (d / "t.cpp").write_text(PROG2)
    exe = d / "t"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", f"-I{CSRC}", str(d / "t.cpp"),
                    "-o", str(exe), "-lm"], check=True)
    return exe


@pytest.mark.parametrize("seed", [11, 12])
def test_exp_pow_log1p_bit_exact_vs_host_libm(prog2, seed):
    """glibc_math2.cuh (the device trace generator's exp / pow / log1p) == host libm's
    __exp_fma / __pow_fma / __log1p_fma on the generator's domains and wide random ranges
    (every branch: tiny, |x| in [512, 1024), k = 0 / k != 0 log1p paths, x >= 2^53)."""
    out = subprocess.run([str(prog2), str(seed), "1000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "exp 0 pow 0 log1p 0 mismatches" in out.stdout


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
    assert (tmp_path / "glibc_math2_gen.cuh").read_text() == (CSRC / "glibc_math2_gen.cuh").read_text()
