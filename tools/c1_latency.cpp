// c1_latency.cpp -- config-1 latency from C++, the drop-in binding's host language: K calls of
// miso_b200_decide (host pointers) on the 3-job roster of generate_trace(seed 7), noisy
// predictor (target MAE 0.017, rng_seed 7), call nonces 1..K -- the same chain and inputs the
// reference arm times (tests/oracle_lib.py c1_time). Built by paper_2207_11428_b200/build.py
// into _lib/c1_latency; bench.py --config c1 runs it. Prints one JSON object:
//   consecutive_us      median latency, nonces 1..K (the server's draw-ahead applies)
//   nonconsecutive_us   median latency, nonces 1000003*k + 17 (draw-ahead never matches)
//   launch_per_call_us  median latency with miso_b200_decide_server(ctx, 0)
//   obj_sum_hex         bit pattern of the sum of the K objectives (parity with the reference)
// With `c1_latency K MIXFILE OUTFILE` it also times the scalar optimize_partition drop-in
// (miso_b200_optimize, one instance per call, host pointers) over the mixes in MIXFILE
// (u64 n, u32 offsets[n+1], f64 speeds[5 * offsets[n]]) and writes each call's entry (i32)
// and objective (f64) to OUTFILE for the parity check against the reference:
//   optimize_us / optimize_p99_us   median / p99 latency per call
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "miso_b200.h"

namespace {

struct Roster {
  double truth3[9];
  uint8_t mem[3];
  int8_t qos[3] = {-1, -1, -1};
};

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

double pct(std::vector<double> v, double q) {
  std::sort(v.begin(), v.end());
  return v[std::min(v.size() - 1, static_cast<size_t>(q * v.size()))];
}

// K timed calls; nonce(k) for k = 1..K. Returns per-call microseconds; *acc = objective sum.
template <class NonceFn>
std::vector<double> run(miso_b200_ctx* ctx, const Roster& r, int K, NonceFn nonce, double* acc) {
  std::vector<double> us;
  us.reserve(K);
  int entry = -1;
  uint8_t place[7];
  double obj = 0.0;
  *acc = 0.0;
  for (int k = 1; k <= K; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = miso_b200_decide(ctx, r.truth3, r.mem, r.qos, 3, nonce(k), 7, 1, 0.017, &entry,
                                    place, &obj, nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (rc < 0) {
      std::fprintf(stderr, "miso_b200_decide failed: %s\n", miso_b200_last_error());
      std::exit(1);
    }
    if (rc == 1) *acc += obj;
    us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
  }
  return us;
}

}  // namespace

// Scalar optimize_partition calls over a mix file; returns per-call microseconds.
std::vector<double> run_optimize(miso_b200_ctx* ctx, const char* mixfile, const char* outfile) {
  FILE* f = std::fopen(mixfile, "rb");
  if (!f) {
    std::fprintf(stderr, "cannot open %s\n", mixfile);
    std::exit(1);
  }
  uint64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) std::exit(1);
  std::vector<uint32_t> offs(n + 1);
  if (std::fread(offs.data(), 4, n + 1, f) != n + 1) std::exit(1);
  std::vector<double> sp(size_t(offs[n]) * 5);
  if (std::fread(sp.data(), 8, sp.size(), f) != sp.size()) std::exit(1);
  std::fclose(f);
  std::vector<int32_t> ent(n);
  std::vector<double> obj(n), us;
  uint8_t place[7];
  for (int pass = 0; pass < 2; ++pass) {  // pass 0 warms the server and the caches
    us.clear();
    for (uint64_t i = 0; i < n; ++i) {
      const int m = int(offs[i + 1] - offs[i]);
      int e = -1;
      double o = 0.0;
      const auto t0 = std::chrono::steady_clock::now();
      const int rc = miso_b200_optimize(ctx, sp.data() + size_t(offs[i]) * 5, m, &e, place, &o);
      const auto t1 = std::chrono::steady_clock::now();
      if (rc < 0) {
        std::fprintf(stderr, "miso_b200_optimize failed: %s\n", miso_b200_last_error());
        std::exit(1);
      }
      ent[i] = rc == 1 ? e : -1;
      obj[i] = rc == 1 ? o : 0.0;
      us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
  }
  FILE* g = std::fopen(outfile, "wb");
  if (!g || std::fwrite(ent.data(), 4, n, g) != n || std::fwrite(obj.data(), 8, n, g) != n) std::exit(1);
  std::fclose(g);
  return us;
}

int main(int argc, char** argv) {
  const int K = argc > 1 ? std::atoi(argv[1]) : 1000;
  double arr[3], dur[3], sp[15];
  int mem[3];
  if (miso_b200_generate_trace(7, 3, 60.0, 7200.0, 0, 1.5, 600.0, 60.0, 7200.0, arr, dur, sp, mem)) {
    std::fprintf(stderr, "generate_trace failed\n");
    return 1;
  }
  Roster r;
  for (int c = 0; c < 3; ++c) {
    r.truth3[3 * c + 0] = sp[5 * c + 4];  // (f7, f4, f3)
    r.truth3[3 * c + 1] = sp[5 * c + 3];
    r.truth3[3 * c + 2] = sp[5 * c + 2];
    r.mem[c] = static_cast<uint8_t>(mem[c]);
  }
  miso_b200_ctx* ctx = nullptr;
  if (miso_b200_create(0, &ctx)) {
    std::fprintf(stderr, "create failed: %s\n", miso_b200_last_error());
    return 1;
  }
  double acc = 0.0, tmp = 0.0;
  run(ctx, r, 50, [](int k) { return uint64_t(900000 + k); }, &tmp);  // warm-up
  const std::vector<double> cons = run(ctx, r, K, [](int k) { return uint64_t(k); }, &acc);
  const std::vector<double> miss =
      run(ctx, r, K, [](int k) { return uint64_t(1000003) * uint64_t(k) + 17; }, &tmp);
  std::vector<double> opt;
  if (argc > 3) opt = run_optimize(ctx, argv[2], argv[3]);
  miso_b200_decide_server(ctx, 0);
  const std::vector<double> launch = run(ctx, r, K, [](int k) { return uint64_t(k); }, &tmp);
  miso_b200_destroy(ctx);
  uint64_t bits;
  static_assert(sizeof(bits) == sizeof(acc), "");
  __builtin_memcpy(&bits, &acc, sizeof(bits));
  std::printf("{\"consecutive_us\": %.4f, \"consecutive_p99_us\": %.4f, \"nonconsecutive_us\": %.4f, "
              "\"launch_per_call_us\": %.4f, \"calls\": %d, \"obj_sum_hex\": \"%016" PRIx64 "\"",
              median(cons), pct(cons, 0.99), median(miss), median(launch), K, bits);
  if (!opt.empty())
    std::printf(", \"optimize_us\": %.4f, \"optimize_p99_us\": %.4f, \"optimize_calls\": %zu",
                median(opt), pct(opt, 0.99), opt.size());
  std::printf("}\n");
  return 0;
}
