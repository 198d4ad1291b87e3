// capi.cu -- the C ABI (include/miso_b200.h): contexts, catalogs, launch plumbing and the
// host-pointer pipelines. Host-side C++; the kernels live in *_kernel.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/miso_b200.h"
#include "candidates_gen.cuh"
#include "internal.h"
#include "sim_types.h"

using namespace miso_b200;

struct miso_b200_ctx {
  int device = 0;
  int n_entries = 0;
  uint8_t counts[kNumEntries][5] = {};
  int default_to_active[kNumEntries];  // default-catalog index -> active index (-1 absent)
  uint64_t en0 = 0, en1 = 0;           // enabled-candidate mask
  // host-path scratch
  cudaStream_t streams[2] = {nullptr, nullptr};
  double* d_speeds = nullptr;
  size_t cap_rows = 0;
  uint32_t* d_offsets = nullptr;
  uint8_t* d_cand = nullptr;
  double* d_obj = nullptr;
  size_t cap_inst = 0;
  void* h_stage = nullptr;  // single-decision staging (miso_b200_decide)
  void* d_stage = nullptr;
  uint64_t decide_seq = 0;
  // resident decision server (decide_server_kernel): mailbox, its stream and exit event
  DecideMailbox* h_mail = nullptr;
  DecideMailbox* d_mail = nullptr;
  cudaStream_t srv_stream = nullptr;
  cudaEvent_t srv_done = nullptr;
  bool srv_live = false;         // launched and not yet observed to have exited
  int64_t srv_idle_ns = -1;      // -1: not configured yet (MISO_B200_DECIDE_IDLE_US, default 2 ms)
  std::chrono::steady_clock::time_point srv_last_ok{};
  // simulator
  int8_t* d_spare_lut = nullptr;  // max_spare_slice_for LUT of the active catalog
  bool lut_valid = false;          // device copy of the LUT matches the catalog
  std::vector<int8_t> h_lut;       // host copy (built from the same catalog)
  bool h_lut_valid = false;
  unsigned char* d_sim_ws = nullptr;
  size_t sim_ws_bytes = 0;
  double* d_sim_draws = nullptr;  // the noisy predictor's precomputed draws (SimBatch::draws)
  size_t sim_draws_bytes = 0;
  // device staging arena of the synchronous *_host simulator / predictor / trace calls (grown
  // stream-ordered, reused across calls)
  unsigned char* d_arena = nullptr;
  size_t arena_bytes = 0;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(MISO_B200_E_UNEXPECTED, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                  \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

constexpr uint64_t kServerLifeNs = 500000000ull;  // a server warp lives at most 0.5 s per launch

// Stop the resident decision server (if any) and wait for it to exit: used before calls that
// synchronise the device implicitly (cudaFree) and on teardown. The server checks `stop`
// every poll, so this costs about one PCIe round trip.
int stop_server(miso_b200_ctx* ctx) {
  if (!ctx->srv_live) return MISO_B200_OK;
  *reinterpret_cast<volatile uint64_t*>(&ctx->h_mail->stop) = 1;
  ctx->srv_live = false;
  CUDA_TRY(cudaStreamSynchronize(ctx->srv_stream));
  return MISO_B200_OK;
}

int64_t server_idle_ns(miso_b200_ctx* ctx) {
  if (ctx->srv_idle_ns < 0) {
    long us = 2000;
    if (const char* e = getenv("MISO_B200_DECIDE_IDLE_US")) us = std::max(0l, atol(e));
    ctx->srv_idle_ns = int64_t(us) * 1000;
  }
  return ctx->srv_idle_ns;
}

int launch_server(miso_b200_ctx* ctx, uint64_t last) {
  if (!ctx->srv_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->srv_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->srv_done, cudaEventDisableTiming));
  }
  *reinterpret_cast<volatile uint64_t*>(&ctx->h_mail->stop) = 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  static const uint32_t poll_ns = [] {  // spacing of the server's two in-flight polls (about
    const char* e = getenv("MISO_B200_DECIDE_POLL_NS");  // half a PCIe read round trip)
    return e ? static_cast<uint32_t>(std::max(0, atoi(e))) : 400u;
  }();
  CUDA_TRY(launch_decide_server(ctx->d_mail, static_cast<DecideOneOut*>(ctx->d_stage), last,
                                uint64_t(ctx->srv_idle_ns), kServerLifeNs, ctx->srv_stream,
                                nullptr, poll_ns));
  CUDA_TRY(cudaEventRecord(ctx->srv_done, ctx->srv_stream));
  ctx->srv_live = true;
  return MISO_B200_OK;
}

// PartitionConfig::violation (topology.hpp:84-101)
bool feasible(const uint8_t* c) {
  static const int gpc[5] = {1, 2, 3, 4, 7}, units[5] = {1, 2, 4, 4, 8}, maxc[5] = {7, 3, 2, 1, 1};
  int total = 0, g = 0, u = 0;
  for (int k = 0; k < 5; ++k) {
    if (c[k] > maxc[k]) return false;
    total += c[k];
    g += c[k] * gpc[k];
    u += c[k] * units[k];
  }
  return total > 0 && g <= 7 && u <= 8 && !(c[3] > 0 && c[2] > 0);
}

int default_index(const uint8_t* c) {
  for (int e = 0; e < kNumEntries; ++e)
    if (std::memcmp(kEntryCounts[e], c, 5) == 0) return e;
  return -1;
}

void apply_catalog(miso_b200_ctx* ctx) {
  ctx->en0 = ctx->en1 = 0;
  for (int c = 0; c < kNumCands; ++c) {
    if (ctx->default_to_active[kCandEntry[c]] < 0) continue;
    if (c < 64) ctx->en0 |= 1ull << c;
    else ctx->en1 |= 1ull << (c - 64);
  }
}

// max_spare_slice_for over the active catalog for every roster of <= 6 min kinds (the table
// the simulator reads on the device; index = base-7 digits of the per-kind counts).
const std::vector<int8_t>& host_lut(miso_b200_ctx* ctx) {
  if (!ctx->h_lut_valid) {
    ctx->h_lut.assign(16807, -1);
    host_spare_lut(&ctx->counts[0][0], ctx->n_entries, ctx->h_lut.data());
    ctx->h_lut_valid = true;
  }
  return ctx->h_lut;
}

int ensure_host_scratch(miso_b200_ctx* ctx, size_t rows, size_t inst) {
  if (!ctx->streams[0]) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  }
  if (!ctx->streams[1]) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[1], cudaStreamNonBlocking));
  }
  if (rows > ctx->cap_rows || inst > ctx->cap_inst) {
    if (int rc = stop_server(ctx)) return rc;
  }
  if (rows > ctx->cap_rows) {
    cudaFree(ctx->d_speeds);
    ctx->d_speeds = nullptr;
    CUDA_TRY(cudaMalloc(&ctx->d_speeds, std::max<size_t>(rows, 1) * 5 * sizeof(double)));
    ctx->cap_rows = rows;
  }
  if (inst > ctx->cap_inst) {
    cudaFree(ctx->d_offsets);
    cudaFree(ctx->d_cand);
    cudaFree(ctx->d_obj);
    ctx->d_offsets = nullptr;
    ctx->d_cand = nullptr;
    ctx->d_obj = nullptr;
    CUDA_TRY(cudaMalloc(&ctx->d_offsets, (inst + 1) * sizeof(uint32_t)));
    CUDA_TRY(cudaMalloc(&ctx->d_cand, std::max<size_t>(inst, 1)));
    CUDA_TRY(cudaMalloc(&ctx->d_obj, std::max<size_t>(inst, 1) * sizeof(double)));
    ctx->cap_inst = inst;
  }
  return MISO_B200_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};


}  // namespace

extern "C" {

int miso_b200_version(void) { return 100; }

const char* miso_b200_last_error(void) { return g_last_error.c_str(); }

int miso_b200_create(int device, miso_b200_ctx** out) {
  if (!out) return fail(MISO_B200_E_INVALID, "null out pointer");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(MISO_B200_E_UNEXPECTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(MISO_B200_E_INVALID, "device out of range");
  DeviceGuard g(device);
  CUDA_TRY(cudaFree(nullptr));  // materialise the primary context
  auto* ctx = new miso_b200_ctx();
  ctx->device = device;
  ctx->n_entries = kNumEntries;
  std::memcpy(ctx->counts, kEntryCounts, sizeof(kEntryCounts));
  for (int i = 0; i < kNumEntries; ++i) ctx->default_to_active[i] = i;
  apply_catalog(ctx);
  *out = ctx;
  return MISO_B200_OK;
}

void miso_b200_destroy(miso_b200_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  stop_server(ctx);
  if (ctx->srv_done) cudaEventDestroy(ctx->srv_done);
  if (ctx->srv_stream) cudaStreamDestroy(ctx->srv_stream);
  if (ctx->h_mail) cudaFreeHost(ctx->h_mail);
  cudaFree(ctx->d_speeds);
  cudaFree(ctx->d_offsets);
  cudaFree(ctx->d_cand);
  cudaFree(ctx->d_obj);
  cudaFree(ctx->d_spare_lut);
  cudaFree(ctx->d_sim_ws);
  cudaFree(ctx->d_sim_draws);
  cudaFree(ctx->d_arena);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  for (auto& s : ctx->streams)
    if (s) cudaStreamDestroy(s);
  delete ctx;
}

int miso_b200_set_catalog(miso_b200_ctx* ctx, const uint8_t* counts, int n) {
  if (!ctx || (!counts && n > 0)) return fail(MISO_B200_E_INVALID, "null argument");
  if (n < 1 || n > kNumEntries) return fail(MISO_B200_E_INVALID, "catalog must have 1..36 entries");
  int map[kNumEntries];
  for (int i = 0; i < kNumEntries; ++i) map[i] = -1;
  for (int i = 0; i < n; ++i) {
    const uint8_t* c = counts + 5 * i;
    if (!feasible(c)) return fail(MISO_B200_E_INVALID, "catalog entry " + std::to_string(i) + " is not a feasible partition");
    int d = default_index(c);
    if (d < 0 || map[d] >= 0) return fail(MISO_B200_E_INVALID, "duplicate catalog entry " + std::to_string(i));
    map[d] = i;
  }
  ctx->n_entries = n;
  std::memcpy(ctx->counts, counts, size_t(n) * 5);
  std::memcpy(ctx->default_to_active, map, sizeof(map));
  apply_catalog(ctx);
  ctx->lut_valid = false;
  ctx->h_lut_valid = false;
  return MISO_B200_OK;
}

int miso_b200_get_catalog(const miso_b200_ctx* ctx, uint8_t* counts) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (counts) std::memcpy(counts, ctx->counts, size_t(ctx->n_entries) * 5);
  return ctx->n_entries;
}

int miso_b200_candidate(const miso_b200_ctx* ctx, int cand, int* entry, int* m, uint8_t place[7]) {
  if (cand < 0 || cand >= kNumCands) return fail(MISO_B200_E_INVALID, "candidate id out of range");
  int mm = 0;
  while (mm < 8 && !(kCandBase[mm] <= cand && cand < kCandBase[mm + 1])) ++mm;
  if (entry) *entry = ctx ? ctx->default_to_active[kCandEntry[cand]] : kCandEntry[cand];
  if (m) *m = mm;
  if (place) std::memcpy(place, kCandPlace[cand], 7);
  return MISO_B200_OK;
}

int miso_b200_optimize_batch(miso_b200_ctx* ctx, const double* speeds, const uint32_t* offsets,
                             uint64_t n, uint8_t* cand, double* obj, void* stream) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (n == 0) return MISO_B200_OK;
  if (!speeds || !offsets || !cand || !obj) return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  CUDA_TRY(launch_optimize(speeds, offsets, n, cand, obj, ctx->en0, ctx->en1,
                           static_cast<cudaStream_t>(stream)));
  return MISO_B200_OK;
}

static_assert(sizeof(miso_b200_batch) == sizeof(SearchBatch) &&
                  offsetof(miso_b200_batch, obj) == offsetof(SearchBatch, obj),
              "miso_b200_batch mirrors SearchBatch");

int miso_b200_optimize_batches(miso_b200_ctx* ctx, const miso_b200_batch* batches,
                               int n_batches, void* stream) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (n_batches < 0 || (n_batches > 0 && !batches)) return fail(MISO_B200_E_INVALID, "bad batch list");
  for (int i = 0; i < n_batches; ++i) {
    const miso_b200_batch& b = batches[i];
    if (b.n && (!b.speeds || !b.offsets || !b.cand || !b.obj))
      return fail(MISO_B200_E_INVALID, "null buffer in batch " + std::to_string(i));
  }
  if (n_batches == 0) return MISO_B200_OK;
  DeviceGuard g(ctx->device);
  CUDA_TRY(launch_optimize_batches(reinterpret_cast<const SearchBatch*>(batches), n_batches,
                                   ctx->en0, ctx->en1, static_cast<cudaStream_t>(stream)));
  return MISO_B200_OK;
}

int miso_b200_optimize_batch_host(miso_b200_ctx* ctx, const double* speeds,
                                  const uint32_t* offsets, uint64_t n, uint8_t* cand,
                                  double* obj) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (n == 0) return MISO_B200_OK;
  if (!speeds || !offsets || !cand || !obj) return fail(MISO_B200_E_INVALID, "null buffer");
  if (offsets[n] < offsets[0]) return fail(MISO_B200_E_MALFORMED, "offsets must be non-decreasing");
  DeviceGuard g(ctx->device);
  const size_t rows = offsets[n];
  int rc = ensure_host_scratch(ctx, rows, n);
  if (rc) return rc;
  // Two-stream pipeline: chunk k's H2D overlaps chunk k-1's search and D2H.
  static uint64_t kChunk = 0;
  if (!kChunk) {  // MISO_B200_E2E_CHUNK: instances per pipeline chunk (tuning)
    const char* e = getenv("MISO_B200_E2E_CHUNK");
    kChunk = e ? std::max<uint64_t>(1024, strtoull(e, nullptr, 10)) : (1u << 17);
  }
  int k = 0;
  for (uint64_t i0 = 0; i0 < n; i0 += kChunk, ++k) {
    const uint64_t i1 = std::min(n, i0 + kChunk);
    cudaStream_t s = ctx->streams[k & 1];
    // each chunk's offsets are checked just before its copies are queued, so the host check
    // of chunk k+1 overlaps the transfers of chunk k (a malformed chunk stops the pipeline:
    // earlier chunks' results may have been written)
    for (uint64_t i = i0; i < i1; ++i)
      if (offsets[i + 1] < offsets[i] || offsets[i + 1] > rows) {  // (rows = offsets[n])
        cudaStreamSynchronize(ctx->streams[0]);
        cudaStreamSynchronize(ctx->streams[1]);
        return fail(MISO_B200_E_MALFORMED, "offsets must be non-decreasing");
      }
    const uint32_t r0 = offsets[i0], r1 = offsets[i1];
    CUDA_TRY(cudaMemcpyAsync(ctx->d_offsets + i0, offsets + i0, (i1 - i0 + 1) * sizeof(uint32_t),
                             cudaMemcpyHostToDevice, s));
    if (r1 > r0)
      CUDA_TRY(cudaMemcpyAsync(ctx->d_speeds + size_t(r0) * 5, speeds + size_t(r0) * 5,
                               size_t(r1 - r0) * 5 * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(launch_optimize(ctx->d_speeds, ctx->d_offsets + i0, i1 - i0, ctx->d_cand + i0,
                             ctx->d_obj + i0, ctx->en0, ctx->en1, s));
    CUDA_TRY(cudaMemcpyAsync(cand + i0, ctx->d_cand + i0, i1 - i0, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(obj + i0, ctx->d_obj + i0, (i1 - i0) * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->streams[0]));
  CUDA_TRY(cudaStreamSynchronize(ctx->streams[1]));
  return MISO_B200_OK;
}

static int run_decide_request(miso_b200_ctx* ctx, const DecideOneArgs& a, int pub_m);

int miso_b200_optimize(miso_b200_ctx* ctx, const double* speeds, int m, int* entry,
                       uint8_t* place, double* obj) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (m < 1 || m > 7)
    return fail(MISO_B200_E_INVALID, "optimize_partition needs 1..7 jobs, got " + std::to_string(m));
  if (!speeds) return fail(MISO_B200_E_INVALID, "null speeds");
  DeviceGuard g(ctx->device);
  // One instance is a latency problem: it goes to the resident decision server as a
  // search-only request (one PCIe round trip), not through the batch pipeline.
  DecideOneArgs a;
  std::memset(&a, 0, sizeof(a));
  double* sp = &a.truth[0][0];
  const int stride = m == 1 ? 5 : 4;  // only the m = 1 entry "7g" reads a 7g speed
  for (int j = 0; j < m; ++j)
    for (int k = 0; k < stride; ++k) sp[j * stride + k] = speeds[5 * j + k];
  a.en0 = ctx->en0;
  a.en1 = ctx->en1;
  a.seq = ++ctx->decide_seq;
  a.m = m;
  a.noisy = kSearchOnly;
  if (int rc = run_decide_request(ctx, a, 0)) return rc;
  const DecideOneOut* h = static_cast<const DecideOneOut*>(ctx->h_stage);
  const uint8_t c = static_cast<uint8_t>(h->cand);
  const double o = h->obj;
  if (c == MISO_B200_CAND_INFEASIBLE) return 0;
  int e = -1, mm = 0;
  uint8_t p[7];
  miso_b200_candidate(ctx, c, &e, &mm, p);
  if (entry) *entry = e;
  if (place) std::memcpy(place, p, size_t(m));
  if (obj) *obj = o;
  return 1;
}

int miso_b200_default_model(double* w2, double* w1) {
  if (!w2 || !w1) return fail(MISO_B200_E_INVALID, "null weights");
  default_model(w2, w1);
  return MISO_B200_OK;
}

static int check_predictor(int mode, double target_mae) {
  if (mode != 0 && mode != 1) return fail(MISO_B200_E_INVALID, "mode must be 0 (oracle) or 1 (noisy)");
  if (!(target_mae >= 0.0 && target_mae <= 0.5))  // validate_predictor_spec, profiles.hpp:180-183
    return fail(MISO_B200_E_INVALID, "target_mae must be in [0, 0.5]");
  return MISO_B200_OK;
}

int miso_b200_predict_batch(miso_b200_ctx* ctx, const double* truth3, uint64_t ncols,
                            int cols_per_group, uint64_t first_nonce, uint64_t rng_seed, int mode,
                            double target_mae, const double* w2, const double* w1, double* out5,
                            void* stream) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (mode != 2)
    if (int rc = check_predictor(mode, target_mae)) return rc;
  if (cols_per_group < 1 || cols_per_group > 7)
    return fail(MISO_B200_E_INVALID, "cols_per_group must be 1..7 (pad_to_seven)");
  if (ncols == 0) return MISO_B200_OK;
  if (!truth3 || !out5) return fail(MISO_B200_E_INVALID, "null buffer");
  double dw2[4], dw1[4];
  if (!w2 || !w1) default_model(dw2, dw1);
  DeviceGuard g(ctx->device);
  CUDA_TRY(launch_predict(truth3, ncols, cols_per_group, first_nonce, rng_seed, mode, target_mae,
                          w2 ? w2 : dw2, w1 ? w1 : dw1, out5, static_cast<cudaStream_t>(stream)));
  return MISO_B200_OK;
}

int miso_b200_decide_batch(miso_b200_ctx* ctx, const double* truth3, const uint8_t* mem_gb,
                           const int8_t* qos_kind, const uint32_t* offsets, const uint64_t* nonce,
                           uint64_t n, uint64_t rng_seed, int mode, double target_mae,
                           const double* w2, const double* w1, uint8_t* cand, double* obj,
                           double* est5, void* stream) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (int rc = check_predictor(mode, target_mae)) return rc;
  if (n == 0) return MISO_B200_OK;
  if (!truth3 || !mem_gb || !qos_kind || !offsets || !nonce || !cand || !obj)
    return fail(MISO_B200_E_INVALID, "null buffer");
  double dw2[4], dw1[4];
  if (!w2 || !w1) default_model(dw2, dw1);
  DeviceGuard g(ctx->device);
  CUDA_TRY(launch_decide(truth3, mem_gb, qos_kind, offsets, nonce, n, rng_seed, mode, target_mae,
                         w2 ? w2 : dw2, w1 ? w1 : dw1, ctx->en0, ctx->en1, cand, obj, est5,
                         static_cast<cudaStream_t>(stream)));
  return MISO_B200_OK;
}

// One single-roster request (args filled in, a.seq assigned) through the resident server or
// one decide_one_kernel launch; returns once the result record in ctx->h_stage answers it.
// pub_m: the est rows the device publishes with the header (0 for search-only requests).
static int run_decide_request(miso_b200_ctx* ctx, const DecideOneArgs& a, int pub_m) {
  if (!ctx->h_stage) {
    CUDA_TRY(cudaHostAlloc(&ctx->h_stage, sizeof(DecideOneOut), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer(&ctx->d_stage, ctx->h_stage, 0));
    std::memset(ctx->h_stage, 0, sizeof(DecideOneOut));
  }
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  DecideOneOut* h = static_cast<DecideOneOut*>(ctx->h_stage);
  // The result record is accepted once it names this request and its check word matches
  // (decide_publish: the device stores it without a fence).
  const volatile uint64_t* hw = reinterpret_cast<const volatile uint64_t*>(h);
  auto answered = [&]() {
    if (hw[kOutSeq] != a.seq) return false;
    uint64_t sum = 0;
    for (int i = 0; i < kOutEst + 5 * pub_m; ++i)
      if (i != kOutCheck) sum += mbx_mix(hw[i], uint64_t(i));
    return sum == hw[kOutCheck];
  };
  if (server_idle_ns(ctx) > 0) {
    // Resident server: post the request (args, then their check word), make sure a server
    // warp is running, spin on the answer. A server that idled out between the liveness check
    // and the post is caught by the periodic event query and relaunched; it serves the pending
    // request because it starts from last = seq - 1.
    if (!ctx->h_mail) {
      CUDA_TRY(cudaHostAlloc(&ctx->h_mail, sizeof(DecideMailbox), cudaHostAllocMapped));
      CUDA_TRY(cudaHostGetDevicePointer(&ctx->d_mail, ctx->h_mail, 0));
      std::memset(ctx->h_mail, 0, sizeof(DecideMailbox));
    }
    const uint64_t* aw = reinterpret_cast<const uint64_t*>(&a);
    uint64_t check = 0;
    for (int i = 0; i < kArgWords; ++i) check += mbx_mix(aw[i], uint64_t(i));
    volatile uint64_t* mw = reinterpret_cast<volatile uint64_t*>(ctx->h_mail);
    for (int i = 0; i < kArgWords; ++i) mw[i] = aw[i];
    mw[kArgWords] = check;
    const auto now = std::chrono::steady_clock::now();
    const bool surely_live =
        ctx->srv_live && now - ctx->srv_last_ok < std::chrono::nanoseconds(ctx->srv_idle_ns / 2);
    if (!surely_live) {
      cudaError_t q = ctx->srv_live ? cudaEventQuery(ctx->srv_done) : cudaSuccess;
      if (q != cudaSuccess && q != cudaErrorNotReady) return cuda_fail(q, "decide server");
      if (q == cudaSuccess)
        if (int rc = launch_server(ctx, a.seq - 1)) return rc;
    }
    int relaunches = 0;
    for (long spin = 1; !answered(); ++spin) {
      if ((spin & 0xfff) != 0) continue;
      const cudaError_t q = cudaEventQuery(ctx->srv_done);
      if (q == cudaErrorNotReady) continue;
      if (q != cudaSuccess) {
        ctx->srv_live = false;
        return cuda_fail(q, "decide server");
      }
      if (answered()) break;
      if (++relaunches > 3) return fail(MISO_B200_E_UNEXPECTED, "decide server did not answer");
      if (int rc = launch_server(ctx, a.seq - 1)) return rc;
    }
    ctx->srv_last_ok = std::chrono::steady_clock::now();
  } else {
    cudaStream_t s = ctx->streams[0];
    CUDA_TRY(launch_decide_one(a, static_cast<DecideOneOut*>(ctx->d_stage), s));
    // Spin on the answer; after ~50 ms of spinning fall back to a stream sync, which also
    // surfaces any launch/execution error.
    for (long spin = 0; !answered(); ++spin) {
      if (spin > (1l << 20)) {
        CUDA_TRY(cudaStreamSynchronize(s));
        if (!answered()) return fail(MISO_B200_E_UNEXPECTED, "decide kernel did not complete");
        break;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return MISO_B200_OK;
}

int miso_b200_decide(miso_b200_ctx* ctx, const double* truth3, const uint8_t* mem_gb,
                     const int8_t* qos_kind, int m, uint64_t nonce, uint64_t rng_seed, int mode,
                     double target_mae, int* entry, uint8_t* place, double* obj, double* est5) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (m < 1 || m > 7)
    return fail(MISO_B200_E_INVALID, "optimize_partition needs 1..7 jobs, got " + std::to_string(m));
  if (int rc = check_predictor(mode, target_mae)) return rc;
  DeviceGuard g(ctx->device);
  // Latency path: the roster goes by value in the launch, results come back through mapped
  // pinned memory, completion is a sequence number the kernel stores last (decide_one_kernel).
  DecideOneArgs a;
  std::memset(&a, 0, sizeof(a));
  for (int c = 0; c < m; ++c) {
    for (int k = 0; k < 3; ++k) a.truth[c][k] = truth3[3 * c + k];
    a.mem[c] = mem_gb[c];
    a.qos[c] = qos_kind[c];
  }
  default_model(a.w2, a.w1);
  a.target_mae = target_mae;
  a.nonce = nonce;
  a.rng_seed = rng_seed;
  a.en0 = ctx->en0;
  a.en1 = ctx->en1;
  a.seq = ++ctx->decide_seq;
  a.m = m;
  a.noisy = mode;
  if (int rc = run_decide_request(ctx, a, m)) return rc;
  const DecideOneOut* h = static_cast<const DecideOneOut*>(ctx->h_stage);
  if (est5) std::memcpy(est5, h->est, sizeof(double) * 5 * m);
  if (h->cand == MISO_B200_CAND_INFEASIBLE) return 0;
  int e = -1, mm = 0;
  uint8_t p[7];
  miso_b200_candidate(ctx, static_cast<int>(h->cand), &e, &mm, p);
  if (entry) *entry = e;
  if (place) std::memcpy(place, p, size_t(m));
  if (obj) *obj = h->obj;
  return 1;
}

int miso_b200_decide_server(miso_b200_ctx* ctx, int idle_us) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (idle_us < 0) return fail(MISO_B200_E_INVALID, "idle_us must be >= 0");
  DeviceGuard g(ctx->device);
  if (int rc = stop_server(ctx)) return rc;
  ctx->srv_idle_ns = int64_t(idle_us) * 1000;
  return MISO_B200_OK;
}

int miso_b200_generate_trace(uint64_t seed, int job_count, double lambda_s,
                             double max_duration_s, int dist, double sigma, double fixed_s,
                             double lo_s, double hi_s, double* arrival_s, double* duration_s,
                             double* speeds5, int* mem_gb) {
  // validate_trace_spec (workload.hpp:37-46)
  if (job_count < 1) return fail(MISO_B200_E_INVALID, "job_count must be >= 1");
  if (!(lambda_s > 0)) return fail(MISO_B200_E_INVALID, "lambda_s must be positive");
  if (!(max_duration_s > 0)) return fail(MISO_B200_E_INVALID, "max_duration_s must be positive");
  if (dist < 0 || dist > 2) return fail(MISO_B200_E_INVALID, "unknown duration distribution");
  if (dist == 0 && !(sigma > 0)) return fail(MISO_B200_E_INVALID, "lognormal sigma must be positive");
  if (dist == 2 && !(lo_s > 0 && lo_s <= hi_s))
    return fail(MISO_B200_E_INVALID, "uniform bounds must satisfy 0 < lo_s <= hi_s");
  if (!arrival_s || !duration_s || !speeds5 || !mem_gb) return fail(MISO_B200_E_INVALID, "null buffer");
  host_generate_trace(seed, job_count, lambda_s, max_duration_s, dist, sigma, fixed_s, lo_s, hi_s,
                      arrival_s, duration_s, speeds5, mem_gb);
  return MISO_B200_OK;
}

int miso_b200_generate_traces(const uint64_t* seeds, int n_traces, int job_count, double lambda_s,
                              double max_duration_s, int dist, double sigma, double fixed_s,
                              double lo_s, double hi_s, int threads, double* arrival_s,
                              double* duration_s, double* speeds5, int* mem_gb) {
  if (n_traces < 0) return fail(MISO_B200_E_INVALID, "n_traces < 0");
  if (n_traces == 0) return MISO_B200_OK;
  if (!seeds) return fail(MISO_B200_E_INVALID, "null buffer");
  // validate once with the first trace (same spec for all)
  int rc = miso_b200_generate_trace(seeds[0], job_count, lambda_s, max_duration_s, dist, sigma,
                                    fixed_s, lo_s, hi_s, arrival_s, duration_s, speeds5, mem_gb);
  if (rc) return rc;
  int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, n_traces - 1));
  std::atomic<int> next{1};
  auto work = [&]() {
    for (int r = next.fetch_add(1); r < n_traces; r = next.fetch_add(1)) {
      const size_t o = size_t(r) * size_t(job_count);
      host_generate_trace(seeds[r], job_count, lambda_s, max_duration_s, dist, sigma, fixed_s,
                          lo_s, hi_s, arrival_s + o, duration_s + o, speeds5 + 5 * o, mem_gb + o);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  return MISO_B200_OK;
}

int miso_b200_generate_traces_device(miso_b200_ctx* ctx, const uint64_t* seeds, int n_traces,
                                     int job_count, double lambda_s, double max_duration_s,
                                     int dist, double sigma, double fixed_s, double lo_s,
                                     double hi_s, double* arrival_s, double* duration_s,
                                     double* speeds5, int* mem_gb, void* stream) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (n_traces < 0) return fail(MISO_B200_E_INVALID, "n_traces < 0");
  // validate_trace_spec (workload.hpp:37-46), as miso_b200_generate_trace
  if (job_count < 1) return fail(MISO_B200_E_INVALID, "job_count must be >= 1");
  if (!(lambda_s > 0)) return fail(MISO_B200_E_INVALID, "lambda_s must be positive");
  if (!(max_duration_s > 0)) return fail(MISO_B200_E_INVALID, "max_duration_s must be positive");
  if (dist < 0 || dist > 2) return fail(MISO_B200_E_INVALID, "unknown duration distribution");
  if (dist == 0 && !(sigma > 0)) return fail(MISO_B200_E_INVALID, "lognormal sigma must be positive");
  if (dist == 2 && !(lo_s > 0 && lo_s <= hi_s))
    return fail(MISO_B200_E_INVALID, "uniform bounds must satisfy 0 < lo_s <= hi_s");
  if (n_traces == 0) return MISO_B200_OK;
  if (!seeds || !arrival_s || !duration_s || !speeds5 || !mem_gb) return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  const double mu = std::log(max_duration_s) - 1.2815515655446004 * sigma;  // kZ90, workload.hpp:75
  CUDA_TRY(launch_generate_traces(seeds, n_traces, job_count, lambda_s, max_duration_s, dist, sigma,
                                  fixed_s, lo_s, hi_s, mu, arrival_s, duration_s, speeds5, mem_gb,
                                  static_cast<cudaStream_t>(stream)));
  return MISO_B200_OK;
}

static int64_t us_from_s_host(double s) { return static_cast<int64_t>(std::llround(s * 1e6)); }

int miso_b200_simulate_batch(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                             int n_traces, int max_jobs, const int32_t* task_trace,
                             const uint8_t* static_counts, const int32_t* job_offsets,
                             const double* arrival_s, const double* base_s, const double* speeds5,
                             const uint8_t* mem_gb, const int8_t* qos_kind,
                             const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                             int64_t* job_jct_us, miso_b200_log_record* log, int64_t log_cap,
                             double* stp_series, int64_t stp_cap, void* stream) {
  return miso_b200_simulate_batch_ex(ctx, opt, n_seeds, n_traces, max_jobs, task_trace,
                                     static_counts, job_offsets, arrival_s, base_s, speeds5,
                                     mem_gb, qos_kind, nullptr, rng_seed, metrics, job_jct_us,
                                     nullptr, log, log_cap, stp_series, stp_cap, 0u, stream);
}

namespace {
// Stream-ordered: every check below is on host-side arguments; per-task input errors (the
// reference's invalid_argument cases) are found by the kernel and reported per task.
int simulate_impl(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds, int n_traces,
                  int max_jobs, const int32_t* task_trace, const uint8_t* static_counts,
                  const int32_t* job_offsets, const double* arrival_s, const double* base_s,
                  const double* speeds5, const uint8_t* mem_gb, const int8_t* qos_kind,
                  const uint8_t* instances, const uint64_t* rng_seed,
                  miso_b200_sim_metrics* metrics, int64_t* job_jct_us, int64_t* job_out,
                  miso_b200_log_record* log, int64_t log_cap, double* stp_series,
                  int64_t stp_cap, unsigned flags, int64_t* prune_bound, void* stream) {
  if (!ctx || !opt) return fail(MISO_B200_E_INVALID, "null argument");
  if (flags & ~MISO_B200_SIM_JCT_ONLY) return fail(MISO_B200_E_INVALID, "unknown flags");
  if ((flags & MISO_B200_SIM_JCT_ONLY) && stp_series)
    return fail(MISO_B200_E_INVALID, "JCT_ONLY runs keep no STP series");
  if (n_seeds < 0) return fail(MISO_B200_E_INVALID, "n_seeds < 0");
  if (n_seeds == 0) return MISO_B200_OK;
  if (n_traces < 1) return fail(MISO_B200_E_INVALID, "n_traces must be >= 1");
  if (!task_trace && n_traces < n_seeds) return fail(MISO_B200_E_INVALID, "fewer traces than tasks");
  if (max_jobs < 1) return fail(MISO_B200_E_INVALID, "max_jobs must be >= 1");
  if (opt->policy != MISO_B200_POLICY_NOPART && opt->policy != MISO_B200_POLICY_ORACLE &&
      opt->policy != MISO_B200_POLICY_MISO && opt->policy != MISO_B200_POLICY_OPTSTA)
    return fail(MISO_B200_E_INVALID, "unknown policy");
  if (opt->policy == MISO_B200_POLICY_OPTSTA && !static_counts)  // sim.hpp:208-209
    return fail(MISO_B200_E_INVALID, "optsta requires a static partition");
  if (opt->cluster_size < 1 || opt->cluster_size > 32767)
    return fail(MISO_B200_E_INVALID, "cluster_size must be >= 1");
  // validate_overheads (sim.hpp:69-74), validate_predictor_spec (profiles.hpp:180-183)
  if (opt->mig_reconfig_s < 0 || opt->checkpoint_restart_s < 0 || opt->mps_window_s < 0)
    return fail(MISO_B200_E_INVALID, "overhead durations must be >= 0");
  if (!(opt->interference > 0.0 && opt->interference <= 1.0))
    return fail(MISO_B200_E_INVALID, "interference must be in (0, 1]");
  if (int rc = check_predictor(opt->predictor_noisy ? 1 : 0, opt->target_mae)) return rc;
  if (job_jct_us && task_trace)
    return fail(MISO_B200_E_INVALID, "job_jct_us is indexed by trace job: not with task_trace (use job_out)");
  if (!job_offsets || !arrival_s || !base_s || !speeds5 || !mem_gb || !qos_kind || !rng_seed ||
      !metrics)
    return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!ctx->lut_valid) {  // (host_lut persists in the context: the async copy may lag)
    const std::vector<int8_t>& lut = host_lut(ctx);
    if (!ctx->d_spare_lut) CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ctx->d_spare_lut), lut.size(), s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_spare_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice, s));
    ctx->lut_valid = true;
  }
  const size_t stride = sim_workspace_stride(max_jobs, opt->cluster_size);
  const size_t need = stride * size_t(n_seeds);
  if (need > ctx->sim_ws_bytes) {  // grown in stream order (no device-wide synchronisation)
    if (ctx->d_sim_ws) CUDA_TRY(cudaFreeAsync(ctx->d_sim_ws, s));
    ctx->d_sim_ws = nullptr;
    ctx->sim_ws_bytes = 0;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ctx->d_sim_ws), need, s));
    ctx->sim_ws_bytes = need;
  }
  SimParams p{};
  p.policy = opt->policy;
  p.cluster_size = opt->cluster_size;
  p.noisy = opt->predictor_noisy ? 1 : 0;
  p.check_invariants = opt->check_invariants ? 1 : 0;
  p.window_us = us_from_s_host(opt->mps_window_s);
  p.reconfig_us = us_from_s_host(opt->mig_reconfig_s);
  p.ckpt_us = us_from_s_host(opt->checkpoint_restart_s);
  p.interference = opt->interference;
  p.target_mae = opt->target_mae;
  p.drift_threshold = opt->reprofile_drift_threshold;
  p.max_events = opt->max_events;
  p.track_stp = (flags & MISO_B200_SIM_JCT_ONLY) ? 0 : 1;
  p.en0 = ctx->en0;
  p.en1 = ctx->en1;
  SimBatch b{};
  b.n_seeds = n_seeds;
  b.n_traces = n_traces;
  b.max_jobs = max_jobs;
  b.job_offsets = job_offsets;
  b.task_trace = task_trace;
  b.static_counts = opt->policy == MISO_B200_POLICY_OPTSTA ? static_counts : nullptr;
  b.arrival_s = arrival_s;
  b.base_s = base_s;
  b.speeds5 = speeds5;
  b.mem_gb = mem_gb;
  b.instances = instances;
  b.qos_kind = qos_kind;
  b.rng_seed = rng_seed;
  b.spare_lut = ctx->d_spare_lut;
  b.workspace = ctx->d_sim_ws;
  b.ws_stride = stride;
  b.metrics = metrics;
  b.job_jct_us = job_jct_us;
  b.job_out = job_out;
  b.log = log;
  b.log_cap = log ? log_cap : 0;
  b.stp_series = stp_series;
  b.stp_cap = stp_series ? stp_cap : 0;
  b.prune_bound = prune_bound;
  double w2[4], w1[4];
  if (opt->small_slice_model_fitted) {  // SimOptions::small_slice_model (sim.hpp:88, 894-896)
    std::memcpy(w2, opt->small_slice_w2, sizeof(w2));
    std::memcpy(w1, opt->small_slice_w1, sizeof(w1));
  } else {
    default_model(w2, w1);
  }
  // miso with the noisy predictor: every task's draws for call nonces 1..max_jobs computed
  // ahead by a throughput kernel (a session caches estimates for at least one job, so without
  // re-profiling there are at most max_jobs calls; later nonces are drawn in the event loop)
  static const bool draws_on = [] {
    const char* e = getenv("MISO_B200_SIM_DRAWS");  // (tuning: 0 = draw inside the event loop)
    return !(e && atoi(e) == 0);
  }();
  if (draws_on && opt->policy == MISO_B200_POLICY_MISO && p.noisy && p.target_mae > 0.0) {
    const size_t need_d = size_t(n_seeds) * size_t(max_jobs) * 14 * sizeof(double);
    if (need_d > ctx->sim_draws_bytes) {
      if (ctx->d_sim_draws) CUDA_TRY(cudaFreeAsync(ctx->d_sim_draws, s));
      ctx->d_sim_draws = nullptr;
      ctx->sim_draws_bytes = 0;
      CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ctx->d_sim_draws), need_d, s));
      ctx->sim_draws_bytes = need_d;
    }
    CUDA_TRY(launch_sim_draws(rng_seed, n_seeds, max_jobs, ctx->d_sim_draws, s));
    b.draws = ctx->d_sim_draws;
    b.draws_k = max_jobs;
  }
  CUDA_TRY(launch_simulate(b, p, w2, w1, s));
  return MISO_B200_OK;
}
}  // namespace

int miso_b200_simulate_batch_ex(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                                int n_traces, int max_jobs, const int32_t* task_trace,
                                const uint8_t* static_counts, const int32_t* job_offsets,
                                const double* arrival_s, const double* base_s,
                                const double* speeds5, const uint8_t* mem_gb,
                                const int8_t* qos_kind, const uint8_t* instances,
                                const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                                int64_t* job_jct_us, int64_t* job_out, miso_b200_log_record* log,
                                int64_t log_cap, double* stp_series, int64_t stp_cap,
                                unsigned flags, void* stream) {
  return simulate_impl(ctx, opt, n_seeds, n_traces, max_jobs, task_trace, static_counts,
                       job_offsets, arrival_s, base_s, speeds5, mem_gb, qos_kind, instances,
                       rng_seed, metrics, job_jct_us, job_out, log, log_cap, stp_series, stp_cap,
                       flags, nullptr, stream);
}

int miso_b200_simulate_batch_pruned(miso_b200_ctx* ctx, const miso_b200_sim_options* opt,
                                    int n_tasks, int n_traces, int max_jobs,
                                    const int32_t* task_trace, const uint8_t* static_counts,
                                    const int32_t* job_offsets, const double* arrival_s,
                                    const double* base_s, const double* speeds5,
                                    const uint8_t* mem_gb, const int8_t* qos_kind,
                                    const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                                    int64_t* bound, unsigned flags, void* stream) {
  if (!opt || opt->policy != MISO_B200_POLICY_OPTSTA)
    return fail(MISO_B200_E_INVALID, "pruned runs are optsta candidate searches");
  if (!task_trace || !bound) return fail(MISO_B200_E_INVALID, "task_trace and bound are required");
  return simulate_impl(ctx, opt, n_tasks, n_traces, max_jobs, task_trace, static_counts,
                       job_offsets, arrival_s, base_s, speeds5, mem_gb, qos_kind, nullptr,
                       rng_seed, metrics, nullptr, nullptr, nullptr, 0, nullptr, 0, flags, bound,
                       stream);
}

extern "C++" {
namespace {
// The synchronous host-pointer calls stage their device copies in one per-context arena,
// carved with 256-byte alignment and grown in stream order (no per-call cudaMalloc/cudaFree).
struct Arena {
  size_t used = 0;
  std::vector<std::pair<void**, size_t>> parts;
  template <class T>
  void add(T** p, size_t n) {
    parts.emplace_back(reinterpret_cast<void**>(p), n * sizeof(T));
    *p = nullptr;
  }
  int commit(miso_b200_ctx* ctx, cudaStream_t s) {
    size_t total = 0;
    for (auto& pr : parts) total += (pr.second + 255) & ~size_t(255);
    if (total > ctx->arena_bytes) {
      if (ctx->d_arena) CUDA_TRY(cudaFreeAsync(ctx->d_arena, s));
      ctx->d_arena = nullptr;
      ctx->arena_bytes = 0;
      CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ctx->d_arena), total, s));
      ctx->arena_bytes = total;
    }
    size_t off = 0;
    for (auto& pr : parts) {
      *pr.first = pr.second ? ctx->d_arena + off : nullptr;
      off += (pr.second + 255) & ~size_t(255);
    }
    return MISO_B200_OK;
  }
};
template <class T>
int upload(T* d, const T* src, size_t n, cudaStream_t s) {
  if (!src || n == 0) return MISO_B200_OK;
  CUDA_TRY(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return MISO_B200_OK;
}
int ensure_stream0(miso_b200_ctx* ctx) {
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  return MISO_B200_OK;
}
}  // namespace
}  // extern "C++"

int miso_b200_simulate_batch_host(miso_b200_ctx* ctx, const miso_b200_sim_options* opt,
                                  int n_tasks, int n_traces, const int32_t* task_trace,
                                  const uint8_t* static_counts, const int32_t* job_offsets,
                                  const double* arrival_s, const double* base_s,
                                  const double* speeds5, const uint8_t* mem_gb,
                                  const int8_t* qos_kind, const uint8_t* instances,
                                  const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                                  int64_t* job_out, miso_b200_log_record* log, int64_t log_cap,
                                  double* stp_series, int64_t stp_cap, unsigned flags) {
  if (!ctx || !opt) return fail(MISO_B200_E_INVALID, "null argument");
  if (n_tasks < 0 || n_traces < 0) return fail(MISO_B200_E_INVALID, "negative count");
  if (n_tasks == 0) return MISO_B200_OK;
  if (!job_offsets || !arrival_s || !base_s || !speeds5 || !mem_gb || !qos_kind || !rng_seed ||
      !metrics)
    return fail(MISO_B200_E_INVALID, "null buffer");
  if (n_traces < 1) return fail(MISO_B200_E_INVALID, "n_traces must be >= 1");
  if (!task_trace && n_traces < n_tasks) return fail(MISO_B200_E_INVALID, "fewer traces than tasks");
  const bool prune = (flags & MISO_B200_SIM_PRUNE) != 0;
  flags &= ~MISO_B200_SIM_PRUNE;
  if (prune) {  // miso_b200_simulate_batch_pruned's contract
    if (opt->policy != MISO_B200_POLICY_OPTSTA || !task_trace)
      return fail(MISO_B200_E_INVALID, "pruned runs are optsta candidate searches with task_trace");
    if (job_out || log || stp_series)
      return fail(MISO_B200_E_INVALID, "pruned runs return metrics only");
    for (int q = 0; instances && q < job_offsets[n_traces]; ++q)
      if (instances[q] != 1) return fail(MISO_B200_E_INVALID, "pruned runs take single-instance traces");
  }
  for (int i = 0; i < n_traces; ++i)
    if (job_offsets[i + 1] < job_offsets[i]) return fail(MISO_B200_E_INVALID, "job_offsets must be non-decreasing");
  if (task_trace)
    for (int t = 0; t < n_tasks; ++t)
      if (task_trace[t] < 0 || task_trace[t] >= n_traces) return fail(MISO_B200_E_INVALID, "task_trace out of range");
  int max_jobs = 1;
  for (int i = 0; i < n_traces; ++i) {
    int Jt = job_offsets[i + 1] - job_offsets[i];
    for (int q = job_offsets[i]; instances && q < job_offsets[i + 1]; ++q)
      Jt += instances[q] > 1 ? instances[q] - 1 : 0;  // (< 1: the kernel reports the task)
    max_jobs = std::max(max_jobs, Jt);
  }
  const size_t J = size_t(job_offsets[n_traces]);
  DeviceGuard g(ctx->device);
  if (int rc = ensure_stream0(ctx)) return rc;
  cudaStream_t s = ctx->streams[0];
  int32_t *d_tt, *d_off;
  uint8_t *d_sc, *d_mem, *d_inst;
  double *d_arr, *d_base, *d_sp, *d_stp;
  int8_t* d_qos;
  uint64_t* d_seed;
  miso_b200_sim_metrics* d_met;
  int64_t *d_jo, *d_bound;
  miso_b200_log_record* d_log;
  const size_t jo_n = job_out ? size_t(n_tasks) * size_t(max_jobs) * MISO_B200_JOB_OUT_FIELDS : 0;
  const size_t log_n = log ? size_t(n_tasks) * size_t(std::max<int64_t>(log_cap, 0)) : 0;
  const size_t stp_n = stp_series ? size_t(n_tasks) * 2 * size_t(std::max<int64_t>(stp_cap, 0)) : 0;
  Arena ar;
  ar.add(&d_tt, task_trace ? size_t(n_tasks) : 0);
  ar.add(&d_sc, static_counts ? size_t(n_tasks) * 5 : 0);
  ar.add(&d_off, size_t(n_traces) + 1);
  ar.add(&d_arr, J);
  ar.add(&d_base, J);
  ar.add(&d_sp, J * 5);
  ar.add(&d_mem, J);
  ar.add(&d_qos, J);
  ar.add(&d_inst, instances ? J : 0);
  ar.add(&d_seed, size_t(n_tasks));
  ar.add(&d_met, size_t(n_tasks));
  ar.add(&d_jo, jo_n);
  ar.add(&d_log, log_n);
  ar.add(&d_stp, stp_n);
  ar.add(&d_bound, prune ? size_t(n_traces) : 0);
  int rc;
  if ((rc = ar.commit(ctx, s))) return rc;
  std::vector<int64_t> b0(prune ? size_t(n_traces) : 0, INT64_MAX);  // no completed candidate yet
  if ((rc = upload(d_tt, task_trace, task_trace ? size_t(n_tasks) : 0, s))) return rc;
  if ((rc = upload(d_sc, static_counts, static_counts ? size_t(n_tasks) * 5 : 0, s))) return rc;
  if ((rc = upload(d_off, job_offsets, size_t(n_traces) + 1, s))) return rc;
  if ((rc = upload(d_arr, arrival_s, J, s))) return rc;
  if ((rc = upload(d_base, base_s, J, s))) return rc;
  if ((rc = upload(d_sp, speeds5, J * 5, s))) return rc;
  if ((rc = upload(d_mem, mem_gb, J, s))) return rc;
  if ((rc = upload(d_qos, qos_kind, J, s))) return rc;
  if ((rc = upload(d_inst, instances, instances ? J : 0, s))) return rc;
  if ((rc = upload(d_seed, rng_seed, size_t(n_tasks), s))) return rc;
  if ((rc = upload(d_bound, b0.data(), b0.size(), s))) return rc;
  rc = simulate_impl(ctx, opt, n_tasks, n_traces, max_jobs, d_tt, d_sc, d_off, d_arr, d_base,
                     d_sp, d_mem, d_qos, prune ? nullptr : d_inst, d_seed, d_met, nullptr, d_jo,
                     d_log, log ? log_cap : 0, d_stp, stp_series ? stp_cap : 0, flags,
                     prune ? d_bound : nullptr, s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(metrics, d_met, sizeof(miso_b200_sim_metrics) * size_t(n_tasks),
                           cudaMemcpyDeviceToHost, s));
  if (jo_n) CUDA_TRY(cudaMemcpyAsync(job_out, d_jo, jo_n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (log_n) CUDA_TRY(cudaMemcpyAsync(log, d_log, log_n * sizeof(miso_b200_log_record), cudaMemcpyDeviceToHost, s));
  if (stp_n) CUDA_TRY(cudaMemcpyAsync(stp_series, d_stp, stp_n * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MISO_B200_OK;
}

int miso_b200_predict_host(miso_b200_ctx* ctx, const double* truth3, uint64_t ncols,
                           int cols_per_group, uint64_t first_nonce, uint64_t rng_seed, int mode,
                           double target_mae, const double* w2, const double* w1, double* out5) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (ncols == 0) return MISO_B200_OK;
  if (!truth3 || !out5) return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  if (int rc = ensure_stream0(ctx)) return rc;
  cudaStream_t s = ctx->streams[0];
  double *d_in, *d_out;
  Arena ar;
  ar.add(&d_in, size_t(ncols) * 3);
  ar.add(&d_out, size_t(ncols) * 5);
  int rc;
  if ((rc = ar.commit(ctx, s))) return rc;
  if ((rc = upload(d_in, truth3, size_t(ncols) * 3, s))) return rc;
  rc = miso_b200_predict_batch(ctx, d_in, ncols, cols_per_group, first_nonce, rng_seed, mode,
                               target_mae, w2, w1, d_out, s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out5, d_out, size_t(ncols) * 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MISO_B200_OK;
}

int miso_b200_generate_traces_device_host(miso_b200_ctx* ctx, const uint64_t* seeds,
                                          int n_traces, int job_count, double lambda_s,
                                          double max_duration_s, int dist, double sigma,
                                          double fixed_s, double lo_s, double hi_s,
                                          double* arrival_s, double* duration_s, double* speeds5,
                                          int* mem_gb) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (n_traces < 0) return fail(MISO_B200_E_INVALID, "n_traces < 0");
  if (n_traces == 0 || job_count < 1)  // (the spec checks and their messages: the device call)
    return miso_b200_generate_traces_device(ctx, seeds, n_traces, job_count, lambda_s,
                                            max_duration_s, dist, sigma, fixed_s, lo_s, hi_s,
                                            arrival_s, duration_s, speeds5, mem_gb, nullptr);
  if (!seeds || !arrival_s || !duration_s || !speeds5 || !mem_gb) return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  if (int rc = ensure_stream0(ctx)) return rc;
  cudaStream_t s = ctx->streams[0];
  const size_t J = size_t(n_traces) * size_t(job_count);
  uint64_t* d_seed;
  double *d_a, *d_d, *d_sp;
  int* d_m;
  Arena ar;
  ar.add(&d_seed, size_t(n_traces));
  ar.add(&d_a, J);
  ar.add(&d_d, J);
  ar.add(&d_sp, J * 5);
  ar.add(&d_m, J);
  int rc;
  if ((rc = ar.commit(ctx, s))) return rc;
  if ((rc = upload(d_seed, seeds, size_t(n_traces), s))) return rc;
  rc = miso_b200_generate_traces_device(ctx, d_seed, n_traces, job_count, lambda_s, max_duration_s,
                                        dist, sigma, fixed_s, lo_s, hi_s, d_a, d_d, d_sp, d_m, s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(arrival_s, d_a, J * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(duration_s, d_d, J * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(speeds5, d_sp, J * 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(mem_gb, d_m, J * sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MISO_B200_OK;
}

int miso_b200_max_spare_slice(miso_b200_ctx* ctx, const uint8_t* min_kinds, int n, int* kind) {
  if (!ctx || !kind || (n > 0 && !min_kinds)) return fail(MISO_B200_E_INVALID, "null argument");
  if (n < 0) return fail(MISO_B200_E_INVALID, "negative count");
  *kind = -1;
  if (n >= 7) return MISO_B200_OK;  // no entry has n + 1 > 7 slices (topology.hpp:229)
  int cnt[5] = {0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    if (min_kinds[i] > 4) return fail(MISO_B200_E_INVALID, "slice kind must be 0..4");
    ++cnt[min_kinds[i]];
  }
  *kind = host_lut(ctx)[size_t((((cnt[0] * 7 + cnt[1]) * 7 + cnt[2]) * 7 + cnt[3]) * 7 + cnt[4])];
  return MISO_B200_OK;
}

int miso_b200_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

}  // extern "C"

namespace {
// One host thread per context (a context serves one host thread at a time); the first failing
// shard's status and message are reported on the caller's thread.
int run_shards(int n_ctx, const std::function<int(int)>& f) {
  std::vector<int> rc(static_cast<size_t>(n_ctx), 0);
  std::vector<std::string> errs(static_cast<size_t>(n_ctx), std::string());
  auto one = [&rc, &errs, &f](int k) {
    const int r = f(k);
    rc[size_t(k)] = r;
    if (r) errs[size_t(k)].assign(miso_b200_last_error());
  };
  std::vector<std::thread> th;
  for (int k = 1; k < n_ctx; ++k) th.emplace_back(one, k);
  one(0);
  for (auto& t : th) t.join();
  for (int k = 0; k < n_ctx; ++k)
    if (rc[size_t(k)]) return fail(rc[size_t(k)], "shard " + std::to_string(k) + ": " + errs[size_t(k)]);
  return MISO_B200_OK;
}
}  // namespace

extern "C" {

int miso_b200_optimize_batch_sharded(miso_b200_ctx* const* ctxs, int n_ctx, const double* speeds,
                                     const uint32_t* offsets, uint64_t n, uint8_t* cand,
                                     double* obj) {
  if (!ctxs || n_ctx < 1) return fail(MISO_B200_E_INVALID, "need at least one context");
  for (int k = 0; k < n_ctx; ++k)
    if (!ctxs[k]) return fail(MISO_B200_E_INVALID, "null context");
  if (n == 0) return MISO_B200_OK;
  if (!speeds || !offsets || !cand || !obj) return fail(MISO_B200_E_INVALID, "null buffer");
  if (offsets[n] < offsets[0]) return fail(MISO_B200_E_MALFORMED, "offsets must be non-decreasing");
  if (n_ctx == 1) return miso_b200_optimize_batch_host(ctxs[0], speeds, offsets, n, cand, obj);
  return run_shards(n_ctx, [&](int k) -> int {
    const uint64_t lo = n * uint64_t(k) / uint64_t(n_ctx), hi = n * uint64_t(k + 1) / uint64_t(n_ctx);
    if (hi == lo) return MISO_B200_OK;
    const uint32_t base = offsets[lo];
    std::vector<uint32_t> off(hi - lo + 1);  // the shard's offsets, rebased to its first row
    for (uint64_t i = 0; i <= hi - lo; ++i) {
      if (offsets[lo + i] < base) return fail(MISO_B200_E_MALFORMED, "offsets must be non-decreasing");
      off[i] = offsets[lo + i] - base;
    }
    return miso_b200_optimize_batch_host(ctxs[k], speeds + size_t(base) * 5, off.data(), hi - lo,
                                         cand + lo, obj + lo);
  });
}

int miso_b200_simulate_batch_sharded(miso_b200_ctx* const* ctxs, int n_ctx,
                                     const miso_b200_sim_options* opt, int n_tasks, int n_traces,
                                     const int32_t* task_trace, const uint8_t* static_counts,
                                     const int32_t* job_offsets, const double* arrival_s,
                                     const double* base_s, const double* speeds5,
                                     const uint8_t* mem_gb, const int8_t* qos_kind,
                                     const uint8_t* instances, const uint64_t* rng_seed,
                                     miso_b200_sim_metrics* metrics, int64_t* job_out,
                                     miso_b200_log_record* log, int64_t log_cap,
                                     double* stp_series, int64_t stp_cap, unsigned flags) {
  if (!ctxs || n_ctx < 1) return fail(MISO_B200_E_INVALID, "need at least one context");
  for (int k = 0; k < n_ctx; ++k)
    if (!ctxs[k]) return fail(MISO_B200_E_INVALID, "null context");
  if (n_ctx == 1 || n_tasks <= 1)
    return miso_b200_simulate_batch_host(ctxs[0], opt, n_tasks, n_traces, task_trace, static_counts,
                                         job_offsets, arrival_s, base_s, speeds5, mem_gb, qos_kind,
                                         instances, rng_seed, metrics, job_out, log, log_cap,
                                         stp_series, stp_cap, flags);
  if (!opt) return fail(MISO_B200_E_INVALID, "null argument");
  if (n_tasks < 0 || n_traces < 1) return fail(MISO_B200_E_INVALID, "negative count");
  if (!job_offsets || !metrics || !rng_seed) return fail(MISO_B200_E_INVALID, "null buffer");
  if (!task_trace && n_traces < n_tasks) return fail(MISO_B200_E_INVALID, "fewer traces than tasks");
  for (int t = 0; task_trace && t < n_tasks; ++t)
    if (task_trace[t] < 0 || task_trace[t] >= n_traces) return fail(MISO_B200_E_INVALID, "task_trace out of range");
  for (int i = 0; i < n_traces; ++i)
    if (job_offsets[i + 1] < job_offsets[i]) return fail(MISO_B200_E_INVALID, "job_offsets must be non-decreasing");
  // the single-call layout: job_out stride = the largest instance total of all traces
  int max_jobs = 1;
  for (int i = 0; i < n_traces; ++i) {
    int Jt = job_offsets[i + 1] - job_offsets[i];
    for (int q = job_offsets[i]; instances && q < job_offsets[i + 1]; ++q)
      Jt += instances[q] > 1 ? instances[q] - 1 : 0;
    max_jobs = std::max(max_jobs, Jt);
  }
  // tasks per trace -> contiguous trace ranges of about n_tasks / n_ctx tasks each
  const int used = task_trace ? n_traces : n_tasks;
  std::vector<int64_t> cum(static_cast<size_t>(used) + 1, 0);
  for (int t = 0; t < n_tasks; ++t) ++cum[size_t(task_trace ? task_trace[t] : t) + 1];
  for (int i = 0; i < used; ++i) cum[size_t(i) + 1] += cum[size_t(i)];
  std::vector<int> cut(static_cast<size_t>(n_ctx) + 1, used);
  cut[0] = 0;
  for (int k = 1; k < n_ctx; ++k) {
    const int64_t goal = int64_t(n_tasks) * k / n_ctx;
    cut[size_t(k)] = int(std::lower_bound(cum.begin(), cum.end(), goal) - cum.begin());
    cut[size_t(k)] = std::max(cut[size_t(k) - 1], std::min(cut[size_t(k)], used));
  }
  return run_shards(n_ctx, [&](int k) -> int {
    const int t0 = cut[size_t(k)], t1 = cut[size_t(k) + 1];  // this shard's traces
    std::vector<int> idx;  // its tasks, in task order
    for (int t = 0; t < n_tasks; ++t) {
      const int tr = task_trace ? task_trace[t] : t;
      if (tr >= t0 && tr < t1) idx.push_back(t);
    }
    if (idx.empty()) return MISO_B200_OK;
    const int nt = int(idx.size()), ntr = t1 - t0;
    const int32_t j0 = job_offsets[t0];
    std::vector<int32_t> off(static_cast<size_t>(ntr) + 1), tt(static_cast<size_t>(nt));
    for (int i = 0; i <= ntr; ++i) off[size_t(i)] = job_offsets[t0 + i] - j0;
    std::vector<uint8_t> sc(static_counts ? size_t(nt) * 5 : 0);
    std::vector<uint64_t> seeds(static_cast<size_t>(nt));
    for (int i = 0; i < nt; ++i) {
      const int t = idx[size_t(i)];
      tt[size_t(i)] = (task_trace ? task_trace[t] : t) - t0;
      seeds[size_t(i)] = rng_seed[t];
      if (static_counts) std::memcpy(&sc[size_t(i) * 5], static_counts + size_t(t) * 5, 5);
    }
    int mj = 1;  // this shard's job_out stride
    for (int i = 0; i < ntr; ++i) {
      int Jt = off[size_t(i) + 1] - off[size_t(i)];
      for (int q = j0 + off[size_t(i)]; instances && q < j0 + off[size_t(i) + 1]; ++q)
        Jt += instances[q] > 1 ? instances[q] - 1 : 0;
      mj = std::max(mj, Jt);
    }
    const size_t F = MISO_B200_JOB_OUT_FIELDS;
    std::vector<miso_b200_sim_metrics> met(static_cast<size_t>(nt));
    std::vector<int64_t> jo(job_out ? size_t(nt) * size_t(mj) * F : 0);
    std::vector<miso_b200_log_record> lg(log ? size_t(nt) * size_t(std::max<int64_t>(log_cap, 0)) : 0);
    std::vector<double> stp(stp_series ? size_t(nt) * 2 * size_t(std::max<int64_t>(stp_cap, 0)) : 0);
    const size_t J0 = size_t(j0);
    const int rc = miso_b200_simulate_batch_host(
        ctxs[k], opt, nt, ntr, tt.data(), static_counts ? sc.data() : nullptr, off.data(),
        arrival_s ? arrival_s + J0 : nullptr, base_s ? base_s + J0 : nullptr,
        speeds5 ? speeds5 + 5 * J0 : nullptr, mem_gb ? mem_gb + J0 : nullptr,
        qos_kind ? qos_kind + J0 : nullptr, instances ? instances + J0 : nullptr, seeds.data(),
        met.data(), job_out ? jo.data() : nullptr, log ? lg.data() : nullptr, log_cap,
        stp_series ? stp.data() : nullptr, stp_cap, flags);
    if (rc) return rc;
    for (int i = 0; i < nt; ++i) {  // scatter to the tasks' indices, single-call layout
      const size_t t = size_t(idx[size_t(i)]);
      metrics[t] = met[size_t(i)];
      if (job_out) {
        int64_t* dst = job_out + t * size_t(max_jobs) * F;
        std::memcpy(dst, &jo[size_t(i) * size_t(mj) * F], size_t(mj) * F * sizeof(int64_t));
      }
      if (log)
        std::memcpy(log + t * size_t(log_cap), &lg[size_t(i) * size_t(log_cap)],
                    size_t(log_cap) * sizeof(miso_b200_log_record));
      if (stp_series)
        std::memcpy(stp_series + t * 2 * size_t(stp_cap), &stp[size_t(i) * 2 * size_t(stp_cap)],
                    2 * size_t(stp_cap) * sizeof(double));
    }
    return MISO_B200_OK;
  });
}

int miso_b200_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(MISO_B200_E_INVALID, "null out pointer");
  CUDA_TRY(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
  return MISO_B200_OK;
}

void miso_b200_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
