// decide_probe.cu -- latency breakdown of the resident decision server (decide_server_kernel):
// host post -> device sees the request -> roster fetched -> computed -> published -> host sees
// the completion number. Links the library's internal launch_decide_server.
//   nvcc -std=c++17 -O2 -Ipaper_2207_11428_b200/csrc tools/decide_probe.cu
//        -Lpaper_2207_11428_b200/_lib -lmiso_b200 -o gpurun_out/decide_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../include/miso_b200.h"
#include "candidates_gen.cuh"
#include "internal.h"

using namespace miso_b200;

int main(int argc, char** argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 2000;
  const uint32_t poll_ns = argc > 2 ? uint32_t(atoi(argv[2])) : 0u;
  double arr[3], dur[3], sp[15];
  int mem[3];
  miso_b200_generate_trace(7, 3, 10.0, 7200.0, 0, 1.5, 0, 0, 0, arr, dur, sp, mem);
  DecideMailbox* mb;
  DecideOneOut* out;
  uint64_t* st;
  cudaHostAlloc(&mb, sizeof(DecideMailbox), cudaHostAllocMapped);
  cudaHostAlloc(&out, sizeof(DecideOneOut), cudaHostAllocMapped);
  cudaHostAlloc(&st, 16 * sizeof(uint64_t), cudaHostAllocMapped);
  std::memset(mb, 0, sizeof(*mb));
  std::memset(out, 0, sizeof(*out));
  DecideOneArgs a;
  std::memset(&a, 0, sizeof(a));
  a.m = 3;
  for (int c = 0; c < 3; ++c) {
    a.truth[c][0] = sp[5 * c + 4];
    a.truth[c][1] = sp[5 * c + 3];
    a.truth[c][2] = sp[5 * c + 2];
    a.mem[c] = uint8_t(mem[c]);
    a.qos[c] = -1;
  }
  miso_b200_default_model(a.w2, a.w1);
  a.target_mae = 0.017;
  a.rng_seed = 7;
  a.noisy = 1;
  a.en0 = ~0ull;
  a.en1 = (1ull << (kNumCands - 64)) - 1;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  launch_decide_server(mb, out, 0, 2000000000ull, 4000000000ull, s, st, poll_ns);
  std::vector<double> host_us, fetch_ns, comp_ns, pub_ns, cyc[3], ph[3];
  std::vector<double> dev_total;
  for (int k = 1; k <= K + 100; ++k) {
    a.nonce = uint64_t(k);
    a.seq = uint64_t(k);
    st[3] = 0;
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t* aw = reinterpret_cast<const uint64_t*>(&a);
    uint64_t check = 0;
    for (int i = 0; i < kArgWords; ++i) check += mbx_mix(aw[i], uint64_t(i));
    volatile uint64_t* mw = reinterpret_cast<volatile uint64_t*>(mb);
    for (int i = 0; i < kArgWords; ++i) mw[i] = aw[i];
    mw[kArgWords] = check;
    const volatile uint64_t* hw = reinterpret_cast<const volatile uint64_t*>(out);
    for (;;) {
      if (hw[kOutSeq] != a.seq) continue;
      uint64_t sum = 0;
      for (int i = 0; i < kOutEst + 15; ++i)
        if (i != kOutCheck) sum += mbx_mix(hw[i], uint64_t(i));
      if (sum == hw[kOutCheck]) break;
    }
    const auto t1 = std::chrono::steady_clock::now();
    while (*reinterpret_cast<volatile uint64_t*>(&st[3]) == 0) {
    }
    if (k <= 100) continue;
    host_us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    fetch_ns.push_back(double(st[1] - st[0]));
    comp_ns.push_back(double(st[2] - st[1]));
    pub_ns.push_back(double(st[3] - st[2]));
    for (int q = 0; q < 3; ++q) cyc[q].push_back(double(st[4 + q]));
    for (int q = 0; q < 3; ++q) ph[q].push_back(double(st[8 + q]));
  }
  *reinterpret_cast<volatile uint64_t*>(&mb->stop) = 1;
  cudaStreamSynchronize(s);
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"poll_ns\": %u, \"host_roundtrip_us\": %.3f, \"fetch_ns\": %.0f, \"compute_ns\": %.0f, \"publish_ns\": %.0f, "
         "\"hit\": %.0f, \"compute_cyc\": %.0f, \"publish_cyc\": %.0f, \"clock_khz\": %d, \"obj\": %.17g, "
         "\"perturb_cyc\": %.0f, \"predict_cyc\": %.0f, \"search_cyc\": %.0f, \"err\": \"%s\"}\n",
         poll_ns, med(host_us), med(fetch_ns), med(comp_ns), med(pub_ns), med(cyc[0]), med(cyc[1]), med(cyc[2]),
         clk, out->obj, med(ph[0]), med(ph[1]), med(ph[2]), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
