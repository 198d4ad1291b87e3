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

// ---------------------------------------------------------------------------------------
// Host trace generator: generate_trace (workload.hpp:97-114) with draw_duration (:72-89) and
// make_synthetic_profile (profiles.hpp:443-465). Host libm (log1p/exp/log/cos/pow) so traces
// are bit-identical to the reference's on the same host. Output per job: arrival_s, duration,
// truth speeds (kind order 1g..7g), memory demand.
// ---------------------------------------------------------------------------------------
namespace miso_b200 {

void host_generate_trace(uint64_t seed, int job_count, double lambda_s, double max_duration_s,
                         int dist_kind, double sigma, double fixed_s, double lo_s, double hi_s,
                         double* arrival_s, double* duration_s, double* speeds5, int* mem_gb) {
  HostRng arr(mix_seed(seed, 0x41));  // 'A'
  HostRng prof(mix_seed(seed, 0x50));  // 'P'
  static const double gpc[5] = {1, 2, 3, 4, 7};
  double arrival = 0;
  for (int i = 0; i < job_count; ++i) {
    if (i > 0) {
      double u = arr.uniform01();  // DetRng::exponential(1.0), common.hpp:96-99
      arrival += lambda_s * (-1.0 * std::log1p(-u));
    }
    arrival_s[i] = arrival;
    double* v = speeds5 + 5 * i;
    double alpha = prof.uniform(0.1, 1.0);
    for (int k = 0; k < 5; ++k) {
      double base = std::pow(gpc[k] / 7.0, alpha);
      v[k] = base * (1.0 + prof.uniform(-0.03, 0.03));
    }
    double anchor = v[4];
    for (int k = 0; k < 5; ++k) v[k] /= anchor;
    v[4] = 1.0;
    for (int k = 3; k >= 0; --k) v[k] = std::clamp(v[k], 1e-6, v[k + 1]);
    double u = prof.uniform01();
    mem_gb[i] = u < 4.0 / 9.0 ? 5 : (u < 7.0 / 9.0 ? 10 : 20);
    double d = 0;
    if (dist_kind == 0) {  // lognormal
      double mu = std::log(max_duration_s) - 1.2815515655446004 * sigma;  // kZ90
      double u1 = prof.uniform01();
      double u2 = prof.uniform01();
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      double n01 = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
      d = std::exp(mu + sigma * n01);
    } else if (dist_kind == 1) {
      d = fixed_s;
    } else {
      d = prof.uniform(lo_s, hi_s);
    }
    duration_s[i] = std::clamp(d, 1.0, max_duration_s);
  }
}

// max_spare_slice_for (topology.hpp:227-252) over an arbitrary catalog (rows of 5 counts),
// tabulated by the pinned min-kind count vector (c0..c4, sum <= 6): index
// ((((c0*7+c1)*7+c2)*7+c3)*7+c4), value = kind or -1.
void host_spare_lut(const uint8_t* counts, int n_entries, int8_t* lut /* 16807 */) {
  for (int i = 0; i < 16807; ++i) lut[i] = -1;
  int c[5];
  for (c[0] = 0; c[0] <= 6; ++c[0])
    for (c[1] = 0; c[0] + c[1] <= 6; ++c[1])
      for (c[2] = 0; c[0] + c[1] + c[2] <= 6; ++c[2])
        for (c[3] = 0; c[0] + c[1] + c[2] + c[3] <= 6; ++c[3])
          for (c[4] = 0; c[0] + c[1] + c[2] + c[3] + c[4] <= 6; ++c[4]) {
            int mk[6], m = 0;
            for (int k = 4; k >= 0; --k)  // pinned kinds sorted descending
              for (int r = 0; r < c[k]; ++r) mk[m++] = k;
            int best = -1;
            for (int e = 0; e < n_entries; ++e) {
              const uint8_t* ec = counts + 5 * e;
              int sl[7], ns = 0;
              for (int k = 4; k >= 0; --k)
                for (int r = 0; r < ec[k]; ++r) sl[ns++] = k;
              if (ns != m + 1) continue;
              for (int spare = 0; spare < ns; ++spare) {
                if (spare > 0 && sl[spare] == sl[spare - 1]) continue;
                if (best >= 0 && sl[spare] <= best) continue;
                bool ok = true;
                for (int i = 0, j = 0; i < ns && ok; ++i) {
                  if (i == spare) continue;
                  if (sl[i] < mk[j]) ok = false;
                  ++j;
                }
                if (ok) best = sl[spare];
              }
            }
            lut[(((c[0] * 7 + c[1]) * 7 + c[2]) * 7 + c[3]) * 7 + c[4]] = static_cast<int8_t>(best);
          }
}

}  // namespace miso_b200
