// model_host.cu -- host-side one-time fit of the small-slice linear model (the LinearMap the
// predictor extrapolates 2g/1g speeds with). Restates, in this library's host code:
//   make_synthetic_profile  profiles.hpp:443-465
//   make_training_corpus    profiles.hpp:469-475
//   jacobi_eigen3 / solve_min_norm / fit_small_slice_model  profiles.hpp:279-361
// The shared default model is fit_small_slice_model(make_training_corpus(3000, 0x5eed))
// (sim.hpp:894-898). Eight weights; computed once per process and passed to the kernels.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <random>

#include "internal.h"
#include "predict.cuh"

namespace miso_b200 {
namespace {

struct HostRng {  // DetRng (common.hpp:85-119) draws used here
  std::mt19937_64 eng;
  explicit HostRng(uint64_t s) : eng(s) {}
  double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
};

void synthetic_speeds(HostRng& r, double v[5]) {
  static const double gpc[5] = {1, 2, 3, 4, 7};
  double alpha = r.uniform(0.1, 1.0);
  for (int k = 0; k < 5; ++k) {
    double base = std::pow(gpc[k] / 7.0, alpha);
    v[k] = base * (1.0 + r.uniform(-0.03, 0.03));
  }
  double anchor = v[4];
  for (int k = 0; k < 5; ++k) v[k] /= anchor;
  v[4] = 1.0;
  for (int i = 3; i >= 0; --i) v[i] = std::clamp(v[i], 1e-6, v[i + 1]);
  (void)r.uniform01();  // memory-class draw (profiles.hpp:457) keeps the stream aligned
}

using M3 = std::array<std::array<double, 3>, 3>;

void jacobi_eigen3(M3 a, std::array<double, 3>& vals, M3& vecs) {
  vecs = {{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = std::abs(a[0][1]) + std::abs(a[0][2]) + std::abs(a[1][2]);
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (std::abs(a[p][q]) < 1e-300) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        double sgn = theta >= 0 ? 1.0 : -1.0;
        double tgt = sgn / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(tgt * tgt + 1.0);
        double s = tgt * c;
        for (int k = 0; k < 3; ++k) {
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = vecs[k][p], vkq = vecs[k][q];
          vecs[k][p] = c * vkp - s * vkq;
          vecs[k][q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) vals[i] = a[i][i];
}

std::array<double, 3> solve_min_norm(const M3& ata, const std::array<double, 3>& aty) {
  std::array<double, 3> vals;
  M3 vecs;
  jacobi_eigen3(ata, vals, vecs);
  double lmax = std::max({std::abs(vals[0]), std::abs(vals[1]), std::abs(vals[2])});
  double tol = lmax * 1e-12;
  std::array<double, 3> w{};
  for (int e = 0; e < 3; ++e) {
    if (std::abs(vals[e]) <= tol) continue;
    double proj = 0;
    for (int k = 0; k < 3; ++k) proj += vecs[k][e] * aty[k];
    proj /= vals[e];
    for (int k = 0; k < 3; ++k) w[k] += vecs[k][e] * proj;
  }
  return w;
}

}  // namespace

void default_model(double w2o[4], double w1o[4]) {
  static double cache[8];
  static bool done = false;
  if (!done) {
    HostRng r(mix_seed(0x5eedull, 0x7261696eull));
    M3 ata{};
    std::array<double, 3> aty2{}, aty1{};
    for (int n = 0; n < 3000; ++n) {
      double v[5];
      synthetic_speeds(r, v);
      const std::array<double, 3> x = {v[3], v[2], 1.0};
      for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) ata[i][j] += x[i] * x[j];
        aty2[i] += x[i] * v[1];
        aty1[i] += x[i] * v[0];
      }
    }
    const auto w2 = solve_min_norm(ata, aty2);
    const auto w1 = solve_min_norm(ata, aty1);
    cache[0] = 0.0; cache[1] = w2[0]; cache[2] = w2[1]; cache[3] = w2[2];
    cache[4] = 0.0; cache[5] = w1[0]; cache[6] = w1[1]; cache[7] = w1[2];
    done = true;
  }
  for (int i = 0; i < 4; ++i) {
    w2o[i] = cache[i];
    w1o[i] = cache[4 + i];
  }
}

}  // namespace miso_b200
