// Timeline probe for the search pipeline (debug tool, GPU box only):
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 --fmad=false -I include \
//        -DMISO_B200_TRACE=1 tools/trace_search.cu -o /tmp/trace && /tmp/trace
// Prints per-tile (producer issue, TMA landed/sort start, sorted, first chunk, released)
// timestamps for CTA 0, relative to the first producer issue, in ns.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2207_11428_b200/csrc/search_kernel.cu"

int main() {
  const uint64_t n = 1000000;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> off(n + 1, 0);
  for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + 1 + rng() % 7;
  std::vector<double> sp(size_t(off[n]) * 5);
  for (auto& x : sp) x = (rng() >> 11) * 0x1p-53;
  double *ds, *dobj; uint32_t* doff; uint8_t* dc;
  cudaMalloc(&ds, sp.size() * 8); cudaMalloc(&doff, (n + 1) * 4); cudaMalloc(&dc, n); cudaMalloc(&dobj, n * 8);
  cudaMemcpy(ds, sp.data(), sp.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(doff, off.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  const uint64_t e0 = ~0ull, e1 = (1ull << 47) - 1;
  for (int it = 0; it < 5; ++it) miso_b200::launch_optimize(ds, doff, n, dc, dobj, e0, e1, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  miso_b200::launch_optimize(ds, doff, n, dc, dobj, e0, e1, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("kernel %.1f us  err=%s\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  static unsigned long long tr[148][4096];
  cudaMemcpyFromSymbol(tr, miso_b200::g_trace, sizeof(tr));
  // Per-CTA summary: kernel entry (slot 4095), first TMA issue, first consumer start, last
  // consumer done -- all relative to the earliest kernel entry.
  unsigned long long g0 = ~0ull;
  for (int c = 0; c < 148; ++c) if (tr[c][4095] && tr[c][4095] < g0) g0 = tr[c][4095];
  double s_entry = 0, s_issue = 0, s_first = 0, s_last = 0, mx_last = 0, mn_last = 1e18;
  for (int c = 0; c < 148; ++c) {
    unsigned long long last = 0;
    for (int k = 0; k < 255; ++k) if (tr[c][k * 16 + 7] > last) last = tr[c][k * 16 + 7];
    s_entry += tr[c][4095] - g0; s_issue += tr[c][3] - g0; s_first += tr[c][6] - g0;
    s_last += last - g0;
    if (last - g0 > mx_last) mx_last = last - g0;
    if (last - g0 < mn_last) mn_last = last - g0;
  }
  printf("mean over CTAs (ns from first entry): entry %.0f  first-issue %.0f  first-consume %.0f  last-done %.0f (min %.0f max %.0f)\n",
         s_entry / 148, s_issue / 148, s_first / 148, s_last / 148, mn_last, mx_last);
  for (int cta : {0, 77}) {
    unsigned long long t0 = tr[cta][4095];
    printf("CTA %d (ns rel. to first producer iteration):\n k  - - - p.issue - - c.start c.done | chunk done times\n", cta);
    for (int k = 0; k < 27; ++k) {
      printf("%2d", k);
      for (int e = 0; e < 16; ++e) {
        unsigned long long v = tr[cta][k * 16 + e];
        if (e == 8) printf(" |");
        printf(" %6lld", v ? (long long)(v - t0) : -1LL);
      }
      printf("\n");
    }
  }
  return 0;
}
