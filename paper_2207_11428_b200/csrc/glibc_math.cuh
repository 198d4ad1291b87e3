// glibc_math.cuh -- bit-exact restatements of glibc 2.39's x86_64 FMA variants of log() and
// cos(), for the arguments DetRng::normal01 (common.hpp:103-108) feeds them:
//   log(u1), u1 in [2^-53, 1)   and   cos(2*pi*u2), 2*pi*u2 in [0, 2*pi).
// The reference calls glibc through libm's ifunc, which on an FMA+AVX2 host (every current
// x86 server, incl. this image's hosts) selects __log_fma / __cos_fma. Their numbers come from
// glibc_math_gen.cuh (tools/extract_glibc_math.py); their operation order -- in particular
// which products GCC contracted into FMAs -- is restated here from the disassembly of those
// functions. Every fma() below is one vfmadd/vfnmadd/vfmsub there; every other product and
// sum is a separately rounded DMUL/DADD (TU compiled with --fmad=false / -ffp-contract=off).
//
// Paths not reachable from normal01 (x <= 0, subnormals, inf/nan for log; |x| >= 105414350
// for cos, which needs the multi-precision __branred) fall back to the platform log/cos.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "glibc_math_gen.cuh"

namespace miso_b200 {
namespace glibc {

#if defined(__CUDA_ARCH__)
#define MISO_HD __device__ __forceinline__
__device__ __forceinline__ double d_of(uint64_t b) { return __longlong_as_double(static_cast<long long>(b)); }
__device__ __forceinline__ uint64_t bits_of(double d) { return static_cast<uint64_t>(__double_as_longlong(d)); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double tab_log(int i) { return d_of(__ldg(reinterpret_cast<const unsigned long long*>(k_log_tab) + i)); }
__device__ __forceinline__ double tab_sc(int i) { return d_of(__ldg(reinterpret_cast<const unsigned long long*>(k_sincostab) + i)); }
#else
#define MISO_HD inline
inline double d_of(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }
inline uint64_t bits_of(double d) { uint64_t b; std::memcpy(&b, &d, 8); return b; }
inline double fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
extern const uint64_t* host_log_tab;
extern const uint64_t* host_sincostab;
inline double tab_log(int i) { return d_of(host_log_tab[i]); }
inline double tab_sc(int i) { return d_of(host_sincostab[i]); }
#endif

// ---- log: sysdeps/ieee754/dbl-64/e_log.c as compiled into __log_fma ------------------------
MISO_HD double log_fma(double x) {
  const uint64_t ix = bits_of(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  constexpr uint64_t LO = 0x3fee000000000000ull;  // asuint64(1.0 - 0x1p-4)
  if (ix - LO < 0x0003090000000000ull) {           // |x - 1| < 0x1.09p-4 (HI - LO)
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = x - 1.0;
    const double B2 = d_of(k_log_B2), B1 = d_of(k_log_B1), B5 = d_of(k_log_B5),
                 B4 = d_of(k_log_B4), B8 = d_of(k_log_B8), B7 = d_of(k_log_B7),
                 B3 = d_of(k_log_B3), B6 = d_of(k_log_B6), B9 = d_of(k_log_B9),
                 B10 = d_of(k_log_B10), B0 = d_of(k_log_B0);
    const double p12 = fma_rn(r, B2, B1);
    const double p45 = fma_rn(r, B5, B4);
    const double r2 = r * r;
    const double p78 = fma_rn(r, B8, B7);
    const double p123 = fma_rn(r2, B3, p12);
    const double p456 = fma_rn(r2, B6, p45);
    const double r3 = r * r2;
    double q = fma_rn(r2, B9, p78);
    q = fma_rn(r3, B10, q);
    q = fma_rn(q, r3, p456);
    const double two27 = 134217728.0;
    q = fma_rn(q, r3, p123);                       // y / r3
    const double rw = fma_rn(r, two27, r);         // r + w, w = r * 0x1p27
    const double rhi = fma_rn(-two27, r, rw);      // r + w - w
    const double rhi2 = rhi * rhi;
    const double rlo = r - rhi;
    const double hi = fma_rn(rhi2, B0, r);         // r + rhi*rhi*B0
    const double rmh = r - hi;
    const double rpr = r + rhi;
    double lo = fma_rn(rhi2, B0, rmh);             // r - hi + w
    const double b0rlo = B0 * rlo;
    lo = fma_rn(b0rlo, rpr, lo);                   // lo += B0 * rlo * (rhi + r)
    const double y = fma_rn(q, r3, lo);            // y = r3 * poly; y += lo
    return hi + y;                                 // y += hi
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) return ::log(x);  // subnormal, <= 0, inf, nan
  const uint64_t tmp = ix - 0x3fe6000000000000ull;           // ix - OFF
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const int64_t k = static_cast<int64_t>(tmp) >> 52;
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = tab_log(2 * i), logc = tab_log(2 * i + 1);
  const double z = d_of(iz);
  const double kd = static_cast<double>(k);
  const double w = fma_rn(kd, d_of(k_log_ln2hi), logc);     // kd*Ln2hi + logc
  const double r = fma_rn(z, invc, -1.0);
  const double a12 = fma_rn(r, d_of(k_log_A2), d_of(k_log_A1));
  const double hi = r + w;
  const double r2 = r * r;
  double lo = w - hi;
  lo = lo + r;
  lo = fma_rn(kd, d_of(k_log_ln2lo), lo);                   // w - hi + r + kd*Ln2lo
  const double rr2 = r * r2;
  const double a34 = fma_rn(r, d_of(k_log_A4), d_of(k_log_A3));
  lo = fma_rn(r2, d_of(k_log_A0), lo);                      // lo + r2*A0
  const double p = fma_rn(a34, r2, a12);
  const double y = fma_rn(rr2, p, lo);
  return y + hi;
}

// ---- cos: sysdeps/ieee754/dbl-64/s_sin.c as compiled into __cos_fma -------------------------
// do_cos (x, dx)
MISO_HD double do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double big = d_of(k_cos_big);
  const double ax = fabs(x);
  const double u = ax + big;
  const int k = static_cast<int>(static_cast<uint32_t>(bits_of(u)) << 2);
  x = (ax - (u - big)) + dx;
  const double xx = x * x;
  const double sp = fma_rn(xx, d_of(k_cos_sn5), d_of(k_cos_sn3));
  const double s = fma_rn(x * xx, sp, x);                   // x + x*xx*(sn3 + xx*sn5)
  double cp = fma_rn(xx, d_of(k_cos_cs6), d_of(k_cos_cs4));
  cp = fma_rn(xx, cp, d_of(k_cos_cs2));
  const double c = xx * cp;                                 // xx*(cs2 + xx*(cs4 + xx*cs6))
  const double sn = tab_sc(k), ssn = tab_sc(k + 1), cs = tab_sc(k + 2), ccs = tab_sc(k + 3);
  double cor = fma_rn(-s, ssn, ccs);                        // ccs - s*ssn
  cor = fma_rn(-c, cs, cor);                                // - cs*c
  cor = fma_rn(-s, sn, cor);                                // - sn*s
  return cs + cor;
}

// TAYLOR_SIN (xx, a, da)
MISO_HD double taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = fma_rn(xx, d_of(k_cos_s5), d_of(k_cos_s4));
  p = fma_rn(xx, p, d_of(k_cos_s3));
  p = fma_rn(xx, p, d_of(k_cos_s2));
  p = fma_rn(xx, p, d_of(k_cos_s1));
  const double hda = da * 0.5;
  const double t1 = fma_rn(p, a, -hda);                     // POLY*a - 0.5*da
  const double t = fma_rn(xx, t1, da);
  return a + t;
}

// do_sin (x, dx)
MISO_HD double do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < d_of(k_cos_t0126)) return taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  const double big = d_of(k_cos_big);
  const double ax = fabs(x);
  const double u = ax + big;
  const int k = static_cast<int>(static_cast<uint32_t>(bits_of(u)) << 2);
  x = ax - (u - big);
  const double xx = x * x;
  const double sp = fma_rn(xx, d_of(k_cos_sn5), d_of(k_cos_sn3));
  const double s = x + fma_rn(x * xx, sp, dx);              // x + (dx + x*xx*(sn3 + xx*sn5))
  double cp = fma_rn(xx, d_of(k_cos_cs6), d_of(k_cos_cs4));
  cp = fma_rn(xx, cp, d_of(k_cos_cs2));
  const double c = fma_rn(x, dx, xx * cp);                  // x*dx + xx*(cs2 + ...)
  const double sn = tab_sc(k), ssn = tab_sc(k + 1), cs = tab_sc(k + 2), ccs = tab_sc(k + 3);
  double cor = fma_rn(s, ccs, ssn);                         // ssn + s*ccs
  cor = fma_rn(-c, sn, cor);                                // - sn*c
  cor = fma_rn(s, cs, cor);                                 // + cs*s
  return copysign(sn + cor, xold);
}

MISO_HD double cos_fma(double x) {
  const uint32_t k = static_cast<uint32_t>(bits_of(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;                          // |x| < 2^-27
  if (k < 0x3feb6000u) return do_cos(x, 0.0);               // |x| < 0.855469
  if (k < 0x400368fdu) {                                    // |x| < 2.426265
    const double y = d_of(k_cos_hp0) - fabs(x);
    const double a = y + d_of(k_cos_hp1);
    const double da = (y - a) + d_of(k_cos_hp1);
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {                                    // |x| < 105414350: reduce_sincos
    const double toint = d_of(k_cos_toint);
    const double t = fma_rn(x, d_of(k_cos_hpinv), toint);
    const double xn = t - toint;
    const int n = static_cast<int>(static_cast<uint32_t>(bits_of(t)) & 3u);
    double y = fma_rn(-xn, d_of(k_cos_mp1), x);
    y = fma_rn(-xn, d_of(k_cos_mp2), y);
    const double t2 = fma_rn(-xn, d_of(k_cos_pp3), y);      // y - xn*pp3
    double db = y - t2;
    db = fma_rn(-xn, d_of(k_cos_pp3), db);
    const double b = fma_rn(-xn, d_of(k_cos_pp4), t2);
    const double tb = t2 - b;
    db = db + fma_rn(-xn, d_of(k_cos_pp4), tb);
    const int m = n + 1;                                    // do_sincos (a, da, n + 1)
    const double r = (m & 1) ? do_cos(b, db) : do_sin(b, db);
    return (m & 2) ? -r : r;
  }
  return ::cos(x);  // huge or non-finite: not reachable from normal01
}

#undef MISO_HD

}  // namespace glibc
}  // namespace miso_b200
