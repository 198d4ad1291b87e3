// glibc_math2.cuh -- bit-exact restatements of glibc 2.39's x86_64 FMA variants of exp(),
// pow() and log1p(), the libm calls of the reference's trace generator (generate_trace,
// workload.hpp:97-114: DetRng::exponential -> log1p, make_synthetic_profile -> pow,
// draw_duration's lognormal -> exp; common.hpp:96-112, profiles.hpp:443-465). On an FMA+AVX2
// host libm's ifunc selects __exp_fma / __pow_fma / __log1p_fma; their numbers come from
// glibc_math2_gen.cuh (tools/extract_glibc_math.py) and their operation order is restated here
// from the disassembly of those functions (libm.so.6 0x79b60, 0x7a1e0, 0x7aff0): every fma_rn
// is one vfmadd/vfmsub/vfnmadd there, every other product and sum a separately rounded op.
//   exp:   sysdeps/ieee754/dbl-64/e_exp.c (128-entry table, degree-5 polynomial)
//   pow:   sysdeps/ieee754/dbl-64/e_pow.c (log_inline with a 128-entry table + exp_inline)
//   log1p: sysdeps/ieee754/dbl-64/s_log1p.c (fdlibm)
// Paths the generator cannot reach (x <= 0, subnormal, inf or nan for pow; y tiny or huge)
// fall back to the platform functions.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "glibc_math.cuh"
#include "glibc_math2_gen.cuh"

namespace miso_b200 {
namespace glibc {

#if defined(__CUDA_ARCH__)
#define MISO_HD2 __device__ __forceinline__
__device__ __forceinline__ uint64_t tab_exp(int i) { return __ldg(reinterpret_cast<const unsigned long long*>(k_exp_tab) + i); }
__device__ __forceinline__ double tab_pow(int i) { return d_of(__ldg(reinterpret_cast<const unsigned long long*>(k_pow_tab) + i)); }
#else
#define MISO_HD2 inline
extern const uint64_t* host_exp_tab;
extern const uint64_t* host_pow_tab;
inline uint64_t tab_exp(int i) { return host_exp_tab[i]; }
inline double tab_pow(int i) { return d_of(host_pow_tab[i]); }
#endif

MISO_HD2 uint32_t top12(double x) { return static_cast<uint32_t>(bits_of(x) >> 52); }

// e_exp.c specialcase (|x| in [512, 1024) after the range check), as in __exp_fma.
MISO_HD2 double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {  // k > 0: the exponent of scale might have overflowed
    sbits -= 1009ull << 52;
    const double scale = d_of(sbits);
    const double y = fma_rn(scale, tmp, scale);
    return y * 0x1p1009;
  }
  sbits += 1022ull << 52;  // k < 0: avoid double rounding in the subnormal range
  const double scale = d_of(sbits);
  const double st = tmp * scale;
  double y = scale + st;
  if (y < 1.0) {
    const double hi = y + 1.0;
    double lo = scale - y;
    lo = lo + st;
    double t = 1.0 - hi;
    t = t + y;
    t = t + lo;
    t = t + hi;
    y = t - 1.0;
    if (y == 0.0) y = 0.0;  // avoid -0.0
  }
  return y * 0x1p-1022;
}

// exp_inline of e_exp.c / e_pow.c: exp(x + xtail) * 2^(sign_bias bits). with_tail: pow's form
// (r += xtail); otherwise __exp (no tail term).
MISO_HD2 double exp_core(double x, double xtail, bool with_tail, uint64_t sign_bias) {
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {  // top12(0x1p-54), top12(512) - top12(0x1p-54)
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) {  // tiny x (0 is common)
      const double one = 1.0 + x;
      return sign_bias ? -one : one;
    }
    if (abstop >= 0x409u) return ::exp(x);  // |x| >= 1024: overflow / underflow / inf / nan
    abstop = 0;                              // large x: specialcase below
  }
  double kd = fma_rn(x, d_of(k_exp_invln2N), d_of(k_exp_shift));
  const uint64_t ki = bits_of(kd);
  kd = kd - d_of(k_exp_shift);
  double r = fma_rn(kd, d_of(k_exp_negln2hiN), x);
  r = fma_rn(kd, d_of(k_exp_negln2loN), r);
  if (with_tail) r = xtail + r;
  const int idx = static_cast<int>(2 * (ki & 0x7f));
  const uint64_t top = (ki + sign_bias) << 45;
  const double tail = d_of(tab_exp(idx));
  const uint64_t sbits = tab_exp(idx + 1) + top;
  const double p23 = fma_rn(r, d_of(k_exp_C3), d_of(k_exp_C2));
  const double t = r + tail;
  const double r2 = r * r;
  const double p45 = fma_rn(r, d_of(k_exp_C5), d_of(k_exp_C4));
  const double q = fma_rn(p23, r2, t);
  const double r4 = r2 * r2;
  const double tmp = fma_rn(p45, r4, q);
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = d_of(sbits);
  return fma_rn(tmp, scale, scale);
}

// exp: __exp_fma.
MISO_HD2 double exp_fma(double x) { return exp_core(x, 0.0, false, 0); }

// log_inline of e_pow.c as compiled into __pow_fma: log(x) = hi + tail, ix a positive normal.
MISO_HD2 double pow_log_inline(uint64_t ix, double* tail) {
  const uint64_t tmp = ix - 0x3fe6955500000000ull;  // OFF
  const int i = static_cast<int>((tmp >> 45) & 0x7f);
  const int32_t k = static_cast<int32_t>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double z = d_of(iz);
  const double kd = static_cast<double>(k);
  const double invc = tab_pow(3 * i), logc = tab_pow(3 * i + 1), logctail = tab_pow(3 * i + 2);
  const double t1 = fma_rn(kd, d_of(k_pow_ln2hi), logc);
  const double lo1 = fma_rn(kd, d_of(k_pow_ln2lo), logctail);
  const double r = fma_rn(z, invc, -1.0);
  const double ar = r * d_of(k_pow_A0);
  const double a12 = fma_rn(r, d_of(k_pow_A2), d_of(k_pow_A1));
  const double a34 = fma_rn(r, d_of(k_pow_A4), d_of(k_pow_A3));
  const double t2 = r + t1;
  double lo2 = t1 - t2;
  lo2 = lo2 + r;
  const double ar2 = r * ar;
  const double ar3 = r * ar2;
  const double lo3 = fma_rn(ar, r, -ar2);
  const double hi = t2 + ar2;
  double a56 = fma_rn(r, d_of(k_pow_A6), d_of(k_pow_A5));
  double lo4 = t2 - hi;
  a56 = fma_rn(a56, ar2, a34);
  lo4 = lo4 + ar2;
  const double q = fma_rn(ar2, a56, a12);
  double lo = lo1 + lo2;
  lo = lo + lo3;
  lo = lo + lo4;
  lo = fma_rn(ar3, q, lo);
  const double y = hi + lo;
  double tl = hi - y;
  tl = tl + lo;
  *tail = tl;
  return y;
}

// pow: __pow_fma for x a positive normal and y with 0x3be <= top12(|y|) <= 0x43d (the range
// the main path handles; everything else goes to the platform pow).
MISO_HD2 double pow_fma(double x, double y) {
  const uint64_t ix = bits_of(x), iy = bits_of(y);
  const uint32_t topx = static_cast<uint32_t>(ix >> 52), topy = static_cast<uint32_t>(iy >> 52) & 0x7ff;
  if (topx - 0x001u >= 0x7feu || topy - 0x3beu > 0x7fu) return ::pow(x, y);
  double lo;
  const double hi = pow_log_inline(ix, &lo);
  const double ehi = y * hi;
  const double elo = fma_rn(y, lo, fma_rn(hi, y, -ehi));
  return exp_core(ehi, elo, true, 0);
}

// log1p: __log1p_fma (s_log1p.c).
MISO_HD2 double log1p_fma(double x) {
  const int32_t hx = static_cast<int32_t>(bits_of(x) >> 32);
  const double ln2_hi = d_of(k_log1p_ln2_hi), ln2_lo = d_of(k_log1p_ln2_lo);
  int k = 0;
  double f, c = 0.0, u;
  int32_t hu;
  bool kpath;
  if (hx <= 0x3fda8279) {                        // x < 0.41422
    const int32_t ax = hx & 0x7fffffff;
    if (ax > 0x3fefffff) return ::log1p(x);      // x <= -1
    if (ax <= 0x3e1fffff) {                      // |x| < 2^-29
      if (ax <= 0x3c8fffff) return x;            // |x| < 2^-54
      const double xx = x * x;
      return fma_rn(-xx, 0.5, x);
    }
    kpath = static_cast<uint32_t>(hx + 0x402d413c) <= 0x402d413cu;  // -1 < x <= -0.2929
  } else {
    if (hx > 0x7fefffff) return x + x;           // inf or nan
    kpath = true;
  }
  if (!kpath) {                                  // -0.2929 < x < 0.41422: f = x, k = 0
    f = x;
    hu = 1;
  } else {
    if (hx <= 0x433fffff) {
      u = 1.0 + x;
      hu = static_cast<int32_t>(bits_of(u) >> 32);
      k = (hu >> 20) - 1023;
      c = k > 0 ? 1.0 - (u - x) : x - (u - 1.0);  // correction term
      c = c / u;
    } else {
      u = x;
      hu = hx;
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const uint64_t lo32 = bits_of(u) & 0xffffffffull;
    if (hu <= 0x6a09d) {
      u = d_of((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3ff00000)) << 32) | lo32);
    } else {
      k += 1;
      u = d_of((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3fe00000)) << 32) | lo32);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hf = f * 0.5;
  const double hfsq = hf * f;
  if (hu == 0) {                                 // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = static_cast<double>(k);
      return fma_rn(kd, ln2_hi, fma_rn(kd, ln2_lo, c));
    }
    double R = fma_rn(-f, d_of(k_log1p_two_thirds), 1.0);
    R = R * hfsq;
    if (k == 0) return f - R;
    const double kd = static_cast<double>(k);
    double t = R - fma_rn(kd, ln2_lo, c);
    t = t - f;
    return fma_rn(kd, ln2_hi, -t);
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = fma_rn(z, d_of(k_log1p_Lp3), d_of(k_log1p_Lp2));
  const double R3 = fma_rn(z, d_of(k_log1p_Lp5), d_of(k_log1p_Lp4));
  const double R4 = fma_rn(z, d_of(k_log1p_Lp7), d_of(k_log1p_Lp6));
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = fma_rn(z, d_of(k_log1p_Lp1), z2 * R2);
  R = fma_rn(z4, R3, R);
  R = fma_rn(z6, R4, R);
  const double sr = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - sr);
  const double kd = static_cast<double>(k);
  double t = fma_rn(kd, ln2_lo, c) + sr;
  t = hfsq - t;
  t = t - f;
  return fma_rn(kd, ln2_hi, -t);
}

}  // namespace glibc
}  // namespace miso_b200

#undef MISO_HD2
