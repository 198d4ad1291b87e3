// c1_latency.cpp -- config-1 latency from C++, the drop-in binding's host language: K calls of
// miso_b200_decide (host pointers) on the 3-job roster of generate_trace(seed 7), noisy
// predictor (target MAE 0.017, rng_seed 7), call nonces 1..K -- the same chain and inputs the
// reference arm times (tests/oracle_lib.py c1_time). Built by paper_2207_11428_b200/build.py
// into _lib/c1_latency; bench.py --config c1 runs it. Prints one JSON object:
//   consecutive_us      median latency, nonces 1..K (the server's draw-ahead applies)
//   nonconsecutive_us   median latency, nonces 1000003*k + 17 (draw-ahead never matches)
//   launch_per_call_us  median latency with miso_b200_decide_server(ctx, 0)
//   obj_sum_hex         bit pattern of the sum of the K objectives (parity with the reference)
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
  miso_b200_decide_server(ctx, 0);
  const std::vector<double> launch = run(ctx, r, K, [](int k) { return uint64_t(k); }, &tmp);
  miso_b200_destroy(ctx);
  uint64_t bits;
  static_assert(sizeof(bits) == sizeof(acc), "");
  __builtin_memcpy(&bits, &acc, sizeof(bits));
  std::printf("{\"consecutive_us\": %.4f, \"consecutive_p99_us\": %.4f, \"nonconsecutive_us\": %.4f, "
              "\"launch_per_call_us\": %.4f, \"calls\": %d, \"obj_sum_hex\": \"%016" PRIx64 "\"}\n",
              median(cons), pct(cons, 0.99), median(miss), median(launch), K, bits);
  return 0;
}
