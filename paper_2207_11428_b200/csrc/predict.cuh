// predict.cuh -- device restatement of the MISO MPS->MIG predictor chain (kernel (a)).
//
//   mix_seed / splitmix64            common.hpp:70-83
//   DetRng(seed) first three draws   common.hpp:85-108 (std::mt19937_64, see below)
//   perturb_speed                    profiles.hpp:193-205
//   predict_mig_speeds (one column)  profiles.hpp:214-253
//   extrapolate_small_slices         profiles.hpp:259-273, 370-384
//   effective_speed                  profiles.hpp:60-65
//
// std::mt19937_64 draws 0..2 only depend on the seeded words x[0..3] and x[156..158]
// (the first twist rewrites mt[i] from mt[i], mt[i+1], mt[i+156]), so a perturbed entry costs
// 158 seeding steps instead of a 312-word seed plus a full 312-word twist.
//
// FP64 arithmetic is IEEE round-to-nearest without contraction (TU compiled --fmad=false), in
// the reference's expression order. log and cos are bit-exact restatements of the glibc 2.39
// FMA variants the reference runs (glibc_math.cuh), so predicted speeds are bit-identical.
#pragma once
#include <cstdint>

#include "glibc_math.cuh"

namespace miso_b200 {

constexpr double kSpeedFloor = 1e-9;  // profiles.hpp:33

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t tag) {
  return splitmix64(splitmix64(seed) ^ splitmix64(tag));
}

__device__ __forceinline__ uint64_t mt64_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// [rand.eng.mers] seeding step x' = f * (x ^ (x >> 62)) + i mod 2^64, f = 0x5851F42D4C957F2D,
// i < 2^32, in 32-bit halves: the xor only flips the low word's two low bits, so
//   lo' = lo ^ (hi >> 30);  t = lo' * f_hi + hi * f_lo  (hi * f_lo is off the critical path);
//   lo(x') = lo(lo' * f_lo) + i, carry;  hi(x') = hi(lo' * f_lo) + t + carry
// as a mad.lo.cc / madc.hi carry chain: 6 instructions per step. (The plain 64-bit expression
// compiles to a wide multiply plus a separate 64-bit add of i, 8.)
__device__ __forceinline__ uint64_t mt64_seed_step(uint64_t x, uint32_t i) {
  constexpr uint32_t kFLo = 0x4C957F2Du, kFHi = 0x5851F42Du;
  const uint32_t hi = static_cast<uint32_t>(x >> 32);
  const uint32_t lo = static_cast<uint32_t>(x) ^ (hi >> 30);
  const uint32_t t = lo * kFHi + hi * kFLo;
  uint32_t rlo, rhi;
  asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\t"
      "madc.hi.u32 %1, %2, %3, %5;"
      : "=r"(rlo), "=r"(rhi)
      : "r"(lo), "r"(kFLo), "r"(i), "r"(t));
  return (static_cast<uint64_t>(rhi) << 32) | rlo;
}

__device__ __forceinline__ uint64_t mt64_twist_draw(uint64_t xk, uint64_t xk1, uint64_t xk156) {
  constexpr uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  const uint64_t y = (xk & UM) | (xk1 & LM);
  return mt64_temper(xk156 ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull));
}

// First three outputs of std::mt19937_64(seed).
__device__ __forceinline__ void mt64_first3(uint64_t seed, uint64_t out[3]) {
  const uint64_t x0 = seed;
  const uint64_t x1 = mt64_seed_step(x0, 1);
  const uint64_t x2 = mt64_seed_step(x1, 2);
  const uint64_t x3 = mt64_seed_step(x2, 3);
  uint64_t x = x3;
#pragma unroll 8
  for (uint32_t i = 4; i <= 155; ++i) x = mt64_seed_step(x, i);
  const uint64_t x156 = mt64_seed_step(x, 156);
  const uint64_t x157 = mt64_seed_step(x156, 157);
  const uint64_t x158 = mt64_seed_step(x157, 158);
  out[0] = mt64_twist_draw(x0, x1, x156);
  out[1] = mt64_twist_draw(x1, x2, x157);
  out[2] = mt64_twist_draw(x2, x3, x158);
}

// Two independent streams at once: the 158-step seeding recurrences are serial chains of
// 64-bit multiplies, so interleaving the two perturbed entries of a column doubles the ILP.
__device__ __forceinline__ void mt64_first3_x2(uint64_t sa, uint64_t sb, uint64_t ra[3],
                                               uint64_t rb[3]) {
  const uint64_t a1 = mt64_seed_step(sa, 1), b1 = mt64_seed_step(sb, 1);
  const uint64_t a2 = mt64_seed_step(a1, 2), b2 = mt64_seed_step(b1, 2);
  const uint64_t a3 = mt64_seed_step(a2, 3), b3 = mt64_seed_step(b2, 3);
  uint64_t xa = a3, xb = b3;
#pragma unroll 8
  for (uint32_t i = 4; i <= 155; ++i) {
    xa = mt64_seed_step(xa, i);
    xb = mt64_seed_step(xb, i);
  }
  const uint64_t a156 = mt64_seed_step(xa, 156), b156 = mt64_seed_step(xb, 156);
  const uint64_t a157 = mt64_seed_step(a156, 157), b157 = mt64_seed_step(b156, 157);
  const uint64_t a158 = mt64_seed_step(a157, 158), b158 = mt64_seed_step(b157, 158);
  ra[0] = mt64_twist_draw(sa, a1, a156);
  ra[1] = mt64_twist_draw(a1, a2, a157);
  ra[2] = mt64_twist_draw(a2, a3, a158);
  rb[0] = mt64_twist_draw(sb, b1, b156);
  rb[1] = mt64_twist_draw(b1, b2, b157);
  rb[2] = mt64_twist_draw(b2, b3, b158);
}

__device__ __forceinline__ double uniform01_of(uint64_t raw) {  // common.hpp:90
  return static_cast<double>(raw >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {  // std::clamp
  return v < lo ? lo : (hi < v ? hi : v);
}

// profiles.hpp:193-205, given the entry's first three raw draws.
// perturb_speed's draws (profiles.hpp:197-201): the N(0,1) magnitude and the sign coin. They
// depend only on the entry's RNG stream, not on the speed or the target MAE.
struct NoiseDraw {
  double n01;
  bool coin;
};

__device__ __forceinline__ NoiseDraw noise_draw(const uint64_t r[3]) {
  double u1 = uniform01_of(r[0]);
  const double u2 = uniform01_of(r[1]);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  NoiseDraw d;
  d.n01 = sqrt(-2.0 * glibc::log_fma(u1)) *
          glibc::cos_fma(6.283185307179586476925287 * u2);  // common.hpp:103-108
  d.coin = uniform01_of(r[2]) < 0.5;
  return d;
}

__device__ __forceinline__ double perturb_apply(double truth, double target_mae, NoiseDraw d) {
  const double sigma = target_mae * sqrt(3.14159265358979323846 / 2.0);
  const double mag = fabs(d.n01) * sigma;
  const bool up_ok = truth + mag <= 1.0;
  const bool dn_ok = truth - mag >= kSpeedFloor;
  if (up_ok && dn_ok) return d.coin ? truth + mag : truth - mag;
  if (up_ok) return truth + mag;
  if (dn_ok) return truth - mag;
  return (1.0 - truth >= truth - kSpeedFloor) ? 1.0 : kSpeedFloor;
}

__device__ __forceinline__ double perturb_with(double truth, double target_mae, const uint64_t r[3]) {
  return perturb_apply(truth, target_mae, noise_draw(r));
}

// profiles.hpp:193-205
__device__ __forceinline__ double perturb_speed(double truth, double target_mae, uint64_t entry_seed) {
  if (target_mae <= 0.0) return truth;
  uint64_t r[3];
  mt64_first3(entry_seed, r);
  return perturb_with(truth, target_mae, r);
}

struct ModelW {
  double w2[4], w1[4];  // LinearMap weights over (f7, f4, f3, 1)
};

// One real (non-dummy) column: truth (f7, f4, f3) -> est speeds in kind order 1g..7g.
// predict_mig_speeds column c of call `nonce` (profiles.hpp:234-248) then
// extrapolate_small_slices (profiles.hpp:376-381).
__device__ __forceinline__ void predict_column(double f7, double f4, double f3, int col,
                                               uint64_t rng_seed, uint64_t nonce, bool noisy,
                                               double target_mae, const ModelW& w,
                                               double out5[5], bool anchor = true) {
  double v0 = f7, v1 = f4, v2 = f3;
  if (noisy && target_mae > 0.0) {  // (target_mae <= 0: perturb_speed returns the truth)
    const uint64_t base = mix_seed(rng_seed, nonce);
    uint64_t ra[3], rb[3];
    mt64_first3_x2(mix_seed(base, static_cast<uint64_t>(col) * 8 + 1),
                   mix_seed(base, static_cast<uint64_t>(col) * 8 + 2), ra, rb);
    v1 = perturb_with(f4, target_mae, ra);
    v2 = perturb_with(f3, target_mae, rb);
  }
  if (anchor) {  // (anchor = false: extrapolate_small_slices alone, on given mig rows)
    double mx = v0;  // std::max({a, b, c})
    if (mx < v1) mx = v1;
    if (mx < v2) mx = v2;
    v0 = clampd(v0 / mx, kSpeedFloor, 1.0);
    v1 = clampd(v1 / mx, kSpeedFloor, 1.0);
    v2 = clampd(v2 / mx, kSpeedFloor, 1.0);
  }
  const double p2 = w.w2[0] * v0 + w.w2[1] * v1 + w.w2[2] * v2 + w.w2[3];
  const double p1 = w.w1[0] * v0 + w.w1[1] * v1 + w.w1[2] * v2 + w.w1[3];
  const double f2 = clampd(p2, kSpeedFloor, v2);
  const double f1 = clampd(p1, kSpeedFloor, f2);
  out5[0] = f1;
  out5[1] = f2;
  out5[2] = v2;
  out5[3] = v1;
  out5[4] = v0;
}

// predict_column with the call's two noise draws given (4g entry d4, 3g entry d3): the
// perturbation, re-anchoring and extrapolation of predict_column in the same operations.
__device__ __forceinline__ void predict_column_drawn(double f7, double f4, double f3,
                                                     NoiseDraw d4, NoiseDraw d3, double target_mae,
                                                     const ModelW& w, double out5[5]) {
  double v0 = f7;
  double v1 = perturb_apply(f4, target_mae, d4);
  double v2 = perturb_apply(f3, target_mae, d3);
  double mx = v0;  // std::max({a, b, c})
  if (mx < v1) mx = v1;
  if (mx < v2) mx = v2;
  v0 = clampd(v0 / mx, kSpeedFloor, 1.0);
  v1 = clampd(v1 / mx, kSpeedFloor, 1.0);
  v2 = clampd(v2 / mx, kSpeedFloor, 1.0);
  const double p2 = w.w2[0] * v0 + w.w2[1] * v1 + w.w2[2] * v2 + w.w2[3];
  const double p1 = w.w1[0] * v0 + w.w1[1] * v1 + w.w1[2] * v2 + w.w1[3];
  const double f2 = clampd(p2, kSpeedFloor, v2);
  const double f1 = clampd(p1, kSpeedFloor, f2);
  out5[0] = f1;
  out5[1] = f2;
  out5[2] = v2;
  out5[3] = v1;
  out5[4] = v0;
}

// A NoiseDraw packed in one double: |n01| with the sign bit clear iff the coin is heads.
// perturb_apply reads only fabs(n01) and the coin, so the pair round-trips exactly.
__device__ __forceinline__ double pack_draw(NoiseDraw d) {
  const double a = fabs(d.n01);
  return d.coin ? a : -a;
}
__device__ __forceinline__ NoiseDraw unpack_draw(double x) {
  NoiseDraw d;
  d.n01 = fabs(x);
  d.coin = !signbit(x);
  return d;
}

// The draws of predictor call `nonce`, column c, entry e (0 = 4g, 1 = 3g) for rng_seed
// (profiles.hpp:234-244: entry seed mix_seed(mix_seed(rng_seed, nonce), 8c + 1 + e)).
__device__ __forceinline__ NoiseDraw column_draw(uint64_t rng_seed, uint64_t nonce, int c, int e) {
  uint64_t r[3];
  mt64_first3(mix_seed(mix_seed(rng_seed, nonce), static_cast<uint64_t>(c) * 8 + 1 + e), r);
  return noise_draw(r);
}

// profiles.hpp:60-65 with kind tables (topology.hpp:39-45). qos_kind < 0: no QoS floor.
__host__ __device__ __forceinline__ int kind_mem_gb(int kind) {
  return kind < 2 ? (kind == 0 ? 5 : 10) : (kind < 4 ? 20 : 40);
}
__host__ __device__ __forceinline__ int kind_gpc(int kind) { return kind < 4 ? kind + 1 : 7; }

__device__ __forceinline__ double effective_speed(double s, int kind, int mem_gb, int qos_kind) {
  if (kind_mem_gb(kind) < mem_gb) return 0.0;
  if (qos_kind >= 0 && kind_gpc(kind) < kind_gpc(qos_kind)) return 0.0;
  return s;
}

}  // namespace miso_b200
