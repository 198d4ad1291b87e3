// internal.h -- launchers shared between the kernel TUs and the C ABI (capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace miso_b200 {

// One batch of independent instances for the search (device pointers).
struct SearchBatch {
  const double* speeds;
  const uint32_t* offsets;
  uint64_t n;
  uint8_t* cand;
  double* obj;
};
constexpr int kMaxPipeBatches = 32;  // batches per persistent-pipeline launch
// Several batches in one persistent launch (queued batches share the launch's fixed cost).
cudaError_t launch_optimize_batches(const SearchBatch* batches, int nb, uint64_t en0,
                                    uint64_t en1, cudaStream_t stream);
cudaError_t launch_optimize(const double* speeds, const uint32_t* offsets, uint64_t n,
                            uint8_t* cand, double* obj, uint64_t en0, uint64_t en1,
                            cudaStream_t stream);

cudaError_t launch_predict(const double* truth3, uint64_t ncols, int cpg, uint64_t first_nonce,
                           uint64_t rng_seed, int noisy, double target_mae, const double* w2,
                           const double* w1, double* out5, cudaStream_t stream);

cudaError_t launch_decide(const double* truth3, const uint8_t* mem_gb, const int8_t* qos_kind,
                          const uint32_t* offsets, const uint64_t* nonce, uint64_t n,
                          uint64_t rng_seed, int noisy, double target_mae, const double* w2,
                          const double* w1, uint64_t en0, uint64_t en1, uint8_t* cand,
                          double* obj, double* est_out, cudaStream_t stream);

// Single-roster decision (miso_b200_decide). Requests and results cross PCIe through mapped
// pinned memory with no fences: each side covers its words with a check word (the sum of
// mbx_mix over the words), and the reader accepts a record only when the check matches, so a
// record read while it is being written (torn) is simply read again.
// noisy == kSearchOnly: an optimize_partition request (miso_b200_optimize). The job speeds
// replace truth/w2/w1/target_mae: 4 per job (1g..4g) packed from truth[0][0], or 5 for m = 1.
constexpr int kSearchOnly = 2;
struct DecideOneArgs {
  double truth[7][3];  // (f7, f4, f3) per job
  double w2[4], w1[4];
  double target_mae;
  uint64_t nonce, rng_seed, en0, en1, seq;
  int m, noisy;
  uint8_t mem[7];
  int8_t qos[7];
};
struct DecideOneOut {
  uint64_t seq;    // the request this record answers
  uint64_t cand;
  double obj;
  uint64_t check;  // sum of mbx_mix over words 0..2 and the 5m est words
  double est[35];
};
// Resident decision server (decide_server_kernel): the request mailbox, read by the server
// in one PCIe round trip (20 lanes x 16 B).
struct DecideMailbox {
  DecideOneArgs args;  // args.seq = request number
  uint64_t check;      // sum of mbx_mix over the kArgWords words of args
  uint64_t stop;       // nonzero: the server exits
};
static_assert(__builtin_offsetof(DecideOneArgs, target_mae) == 29 * 8,
              "search-only requests pack up to 29 speeds over truth/w2/w1");
constexpr int kArgWords = static_cast<int>(sizeof(DecideOneArgs) / 8);
constexpr int kArgSeqWord = static_cast<int>(__builtin_offsetof(DecideOneArgs, seq) / 8);
constexpr int kOutWords = static_cast<int>(sizeof(DecideOneOut) / 8);
constexpr int kOutSeq = 0, kOutCand = 1, kOutObj = 2, kOutCheck = 3, kOutEst = 4;
static_assert(sizeof(DecideOneArgs) % 8 == 0, "mailbox records are 8-byte words");
static_assert(sizeof(DecideMailbox) == 16 * 20, "the server fetches the mailbox as 20 x 16 B");
static_assert(kOutWords == 39, "DecideOneOut layout");

#ifdef __CUDACC__
__host__ __device__
#endif
inline uint64_t mbx_mix(uint64_t w, uint64_t i) {  // splitmix64 finaliser of (word, index)
  uint64_t z = w + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

cudaError_t launch_decide_one(const DecideOneArgs& a, DecideOneOut* out, cudaStream_t stream);
// stamps (timing probe only, else nullptr): globaltimer at request seen / roster fetched /
// computed / published, written after each request.
// poll_ns: spacing of the server's two in-flight mailbox polls.
cudaError_t launch_decide_server(const DecideMailbox* mb, DecideOneOut* out, uint64_t last,
                                 uint64_t idle_ns, uint64_t life_ns, cudaStream_t stream,
                                 uint64_t* stamps = nullptr, uint32_t poll_ns = 0);

// Device: generate_trace for n seeds, one warp per trace (trace_kernel.cu). mu = the
// lognormal's log(max_duration_s) - kZ90 * sigma, computed on the host as the reference does.
cudaError_t launch_generate_traces(const uint64_t* seeds, int n, int job_count, double lambda_s,
                                   double max_duration_s, int dist, double sigma, double fixed_s,
                                   double lo_s, double hi_s, double mu, double* arrival_s,
                                   double* duration_s, double* speeds5, int* mem_gb,
                                   cudaStream_t stream);

// Host: generate_trace (workload.hpp:97-114); dist_kind 0 lognormal, 1 fixed, 2 uniform.
void host_generate_trace(uint64_t seed, int job_count, double lambda_s, double max_duration_s,
                         int dist_kind, double sigma, double fixed_s, double lo_s, double hi_s,
                         double* arrival_s, double* duration_s, double* speeds5, int* mem_gb);

// Host: max_spare_slice_for (topology.hpp:227-252) tabulated over min-kind count vectors.
void host_spare_lut(const uint8_t* counts, int n_entries, int8_t* lut);

// Host: fit_small_slice_model(make_training_corpus(3000, 0x5eed)) (sim.hpp:894-898).
void default_model(double w2[4], double w1[4]);

}  // namespace miso_b200
