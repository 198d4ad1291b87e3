// trace_kernel.cu -- device trace generation: generate_trace (workload.hpp:97-114) with
// make_synthetic_profile (profiles.hpp:443-465) and draw_duration (workload.hpp:72-89) for many
// seeds at once, bit-identical to the reference on an FMA+AVX2 host (its libm calls are the
// glibc_math2.cuh / glibc_math.cuh restatements of __exp_fma, __pow_fma, __log1p_fma, __log_fma
// and __cos_fma).
//
// One warp per trace. Each trace owns two std::mt19937_64 streams (DetRng, common.hpp:85-119):
// arrivals mix_seed(seed, 'A') and profiles mix_seed(seed, 'P'). A stream's 312-word state
// lives in shared memory: seeding is the standard's serial recurrence (one lane), and each
// twist is done by the warp in three dependency phases (words [0,156) read only old words,
// [156,311) read words of the first phase, 311 reads word 0). Every job draws a fixed number
// of values from the profile stream (alpha, 5 jitters, memory, then 2/0/1 for a lognormal /
// fixed / uniform duration), so after each twist the jobs whose draws are complete are decoded
// by the lanes in parallel from a two-block ring of tempered outputs. Arrivals are the
// reference's sequential FP64 running sum, evaluated in job order through warp shuffles.
#include <cuda_runtime.h>

#include <cstdint>

#include "glibc_math2.cuh"
#include "internal.h"
#include "predict.cuh"

namespace miso_b200 {

namespace {

constexpr int kMtN = 312;
constexpr uint64_t kMtUM = 0xFFFFFFFF80000000ull, kMtLM = 0x7FFFFFFFull;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;

__device__ __forceinline__ void mt_seed(uint64_t* mt, uint64_t seed) {  // [rand.eng.mers]
  if ((threadIdx.x & 31) == 0) {
    uint64_t x = seed;
    mt[0] = x;
    for (int i = 1; i < kMtN; ++i) {
      x = mt64_seed_step(x, static_cast<uint32_t>(i));
      mt[i] = x;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t xi, uint64_t xi1, uint64_t xm) {
  const uint64_t y = (xi & kMtUM) | (xi1 & kMtLM);
  return xm ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

// One full twist of the 312-word state, then the 312 tempered outputs into out[0..311].
__device__ __forceinline__ void mt_block(uint64_t* mt, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  for (int b = 0; b < 156; b += 32) {  // phase 1: i < 156 reads old words only
    const int i = b + lane;
    uint64_t v = 0;
    if (i < 156) v = mt_mix(mt[i], mt[i + 1], mt[i + 156]);
    __syncwarp();
    if (i < 156) mt[i] = v;
    __syncwarp();
  }
  for (int b = 156; b < kMtN - 1; b += 32) {  // phase 2: reads new mt[i - 156]
    const int i = b + lane;
    uint64_t v = 0;
    if (i < kMtN - 1) v = mt_mix(mt[i], mt[i + 1], mt[i - 156]);
    __syncwarp();
    if (i < kMtN - 1) mt[i] = v;
    __syncwarp();
  }
  if (lane == 0) mt[kMtN - 1] = mt_mix(mt[kMtN - 1], mt[0], mt[155]);
  __syncwarp();
  for (int i = lane; i < kMtN; i += 32) out[i] = mt64_temper(mt[i]);
  __syncwarp();
}

__device__ __forceinline__ double u01(uint64_t raw) { return static_cast<double>(raw >> 11) * 0x1.0p-53; }

}  // namespace

struct TraceGenParams {
  int job_count, dist;  // 0 lognormal, 1 fixed, 2 uniform
  double lambda_s, max_duration_s, sigma, fixed_s, lo_s, hi_s;
  double mu;            // log(max_duration_s) - kZ90 * sigma (host libm, as the reference)
};

__global__ void __launch_bounds__(32) generate_traces_kernel(const uint64_t* __restrict__ seeds,
                                                            int n, TraceGenParams p,
                                                            double* __restrict__ arrival_s,
                                                            double* __restrict__ duration_s,
                                                            double* __restrict__ speeds5,
                                                            int* __restrict__ mem_gb) {
  __shared__ uint64_t mt[kMtN];
  __shared__ uint64_t ring[2 * kMtN];
  const int t = blockIdx.x;
  if (t >= n) return;
  const int lane = threadIdx.x & 31;
  const int J = p.job_count;
  const size_t o = size_t(t) * size_t(J);
  const uint64_t seed = seeds[t];

  // ---- profiles stream 'P': make_synthetic_profile + draw_duration per job ----
  const int dpj = 7 + (p.dist == 0 ? 2 : (p.dist == 2 ? 1 : 0));
  const long total = long(J) * dpj;
  mt_seed(mt, mix_seed(seed, 0x50));
  int next_job = 0;
  for (long blk = 0; blk * kMtN < total; ++blk) {
    mt_block(mt, ring + (blk & 1) * kMtN);
    const long avail = (blk + 1) * kMtN;  // draws [0, avail) produced; the ring holds the last 624
    const int ready = static_cast<int>(avail / dpj < J ? avail / dpj : J);
    for (int i = next_job + lane; i < ready; i += 32) {
      const long d0 = long(i) * dpj;
      auto draw = [&](int q) { return ring[(d0 + q) % (2 * kMtN)]; };
      const double alpha = 0.1 + (1.0 - 0.1) * u01(draw(0));  // uniform(0.1, 1.0)
      double v[5];
      const double gpc[5] = {1, 2, 3, 4, 7};
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const double base = glibc::pow_fma(gpc[k] / 7.0, alpha);
        v[k] = base * (1.0 + (-0.03 + (0.03 - -0.03) * u01(draw(1 + k))));
      }
      const double anchor = v[4];
#pragma unroll
      for (int k = 0; k < 5; ++k) v[k] = v[k] / anchor;
      v[4] = 1.0;
#pragma unroll
      for (int k = 3; k >= 0; --k) v[k] = clampd(v[k], 1e-6, v[k + 1]);
      const double um = u01(draw(6));
      const int mem = um < 4.0 / 9.0 ? 5 : (um < 7.0 / 9.0 ? 10 : 20);
      double d;
      if (p.dist == 0) {  // lognormal(mu, sigma) = exp(mu + sigma * normal01())
        double u1 = u01(draw(7));
        const double u2 = u01(draw(8));
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        const double n01 = sqrt(-2.0 * glibc::log_fma(u1)) *
                           glibc::cos_fma(6.283185307179586476925287 * u2);
        d = glibc::exp_fma(p.mu + p.sigma * n01);
      } else if (p.dist == 1) {
        d = p.fixed_s;
      } else {
        d = p.lo_s + (p.hi_s - p.lo_s) * u01(draw(7));
      }
      duration_s[o + i] = clampd(d, 1.0, p.max_duration_s);
#pragma unroll
      for (int k = 0; k < 5; ++k) speeds5[(o + i) * 5 + k] = v[k];
      mem_gb[o + i] = mem;
    }
    next_job = ready;
    __syncwarp();
  }

  // ---- arrivals stream 'A': arrival += lambda_s * exponential(1.0), job order ----
  mt_seed(mt, mix_seed(seed, 0x41));
  double arrival = 0.0;
  if (lane == 0) arrival_s[o] = 0.0;
  for (long blk = 0; blk * kMtN < long(J) - 1; ++blk) {
    mt_block(mt, ring);
    const int j0 = static_cast<int>(blk * kMtN) + 1;  // job j uses draw j - 1
    const int cnt = (J - j0) < kMtN ? (J - j0) : kMtN;
    for (int b = 0; b < cnt; b += 32) {
      double term = 0.0;
      if (b + lane < cnt) term = p.lambda_s * (-1.0 * glibc::log1p_fma(-u01(ring[b + lane])));
      const int m = (cnt - b) < 32 ? (cnt - b) : 32;
      double mine = 0.0;
      for (int q = 0; q < m; ++q) {
        arrival = arrival + __shfl_sync(0xffffffffu, term, q);
        if (lane == q) mine = arrival;
      }
      if (lane < m) arrival_s[o + j0 + b + lane] = mine;
    }
    __syncwarp();
  }
}

cudaError_t launch_generate_traces(const uint64_t* seeds, int n, int job_count, double lambda_s,
                                   double max_duration_s, int dist, double sigma, double fixed_s,
                                   double lo_s, double hi_s, double mu, double* arrival_s,
                                   double* duration_s, double* speeds5, int* mem_gb,
                                   cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  TraceGenParams p;
  p.job_count = job_count;
  p.dist = dist;
  p.lambda_s = lambda_s;
  p.max_duration_s = max_duration_s;
  p.sigma = sigma;
  p.fixed_s = fixed_s;
  p.lo_s = lo_s;
  p.hi_s = hi_s;
  p.mu = mu;
  generate_traces_kernel<<<n, 32, 0, stream>>>(seeds, n, p, arrival_s, duration_s, speeds5, mem_gb);
  return cudaGetLastError();
}

}  // namespace miso_b200
