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
#include <cstring>
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

int miso_b200_optimize(miso_b200_ctx* ctx, const double* speeds, int m, int* entry,
                       uint8_t* place, double* obj) {
  if (!ctx) return fail(MISO_B200_E_INVALID, "null context");
  if (m < 1 || m > 7)
    return fail(MISO_B200_E_INVALID, "optimize_partition needs 1..7 jobs, got " + std::to_string(m));
  if (!speeds) return fail(MISO_B200_E_INVALID, "null speeds");
  uint32_t offs[2] = {0, static_cast<uint32_t>(m)};
  uint8_t c = 0;
  double o = 0;
  int rc = miso_b200_optimize_batch_host(ctx, speeds, offs, 1, &c, &o);
  if (rc) return rc;
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
  if (!ctx->h_stage) {
    CUDA_TRY(cudaHostAlloc(&ctx->h_stage, sizeof(DecideOneOut), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer(&ctx->d_stage, ctx->h_stage, 0));
    std::memset(ctx->h_stage, 0, sizeof(DecideOneOut));
  }
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
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
  DecideOneOut* h = static_cast<DecideOneOut*>(ctx->h_stage);
  // The result record is accepted once it names this request and its check word matches
  // (decide_publish: the device stores it without a fence).
  const volatile uint64_t* hw = reinterpret_cast<const volatile uint64_t*>(h);
  auto answered = [&]() {
    if (hw[kOutSeq] != a.seq) return false;
    uint64_t sum = 0;
    for (int i = 0; i < kOutEst + 5 * m; ++i)
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
                             const int32_t* task_trace, const uint8_t* static_counts,
                             const int32_t* job_offsets, const double* arrival_s,
                             const double* base_s, const double* speeds5, const uint8_t* mem_gb,
                             const int8_t* qos_kind, const uint64_t* rng_seed,
                             miso_b200_sim_metrics* metrics, int64_t* job_jct_us,
                             miso_b200_log_record* log, int64_t log_cap, double* stp_series,
                             int64_t stp_cap, void* stream) {
  return miso_b200_simulate_batch_ex(ctx, opt, n_seeds, task_trace, static_counts, job_offsets,
                                     arrival_s, base_s, speeds5, mem_gb, qos_kind, nullptr,
                                     rng_seed, metrics, job_jct_us, nullptr, log, log_cap,
                                     stp_series, stp_cap, 0u, stream);
}

namespace {
int simulate_impl(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                  const int32_t* task_trace, const uint8_t* static_counts,
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
  if (!job_offsets || !arrival_s || !base_s || !speeds5 || !mem_gb || !qos_kind || !rng_seed ||
      !metrics)
    return fail(MISO_B200_E_INVALID, "null buffer");
  DeviceGuard g(ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // max jobs per task (device arrays: read the index arrays back once)
  int n_traces = n_seeds;
  std::vector<int32_t> tt;
  if (task_trace) {
    tt.resize(size_t(n_seeds));
    CUDA_TRY(cudaMemcpyAsync(tt.data(), task_trace, tt.size() * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    n_traces = 0;
    for (int v : tt) {
      if (v < 0) return fail(MISO_B200_E_INVALID, "negative task_trace entry");
      n_traces = std::max(n_traces, v + 1);
    }
  }
  std::vector<int32_t> offs(size_t(n_traces) + 1);
  CUDA_TRY(cudaMemcpyAsync(offs.data(), job_offsets, offs.size() * 4, cudaMemcpyDeviceToHost, s));
  if (static_counts && opt->policy == MISO_B200_POLICY_OPTSTA) {
    std::vector<uint8_t> sc(size_t(n_seeds) * 5);
    CUDA_TRY(cudaMemcpyAsync(sc.data(), static_counts, sc.size(), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < n_seeds; ++i)
      if (!feasible(&sc[size_t(i) * 5]))
        return fail(MISO_B200_E_INVALID, "static partition of task " + std::to_string(i) + " is not feasible");
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<uint8_t> inst;
  if (instances && offs[size_t(n_traces)] > offs[0]) {  // capacity includes every clone
    inst.resize(size_t(offs[size_t(n_traces)]));
    CUDA_TRY(cudaMemcpyAsync(inst.data(), instances, inst.size(), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  int max_jobs = 0;
  for (int i = 0; i < n_traces; ++i) {
    int J = offs[i + 1] - offs[i];
    if (J < 1) return fail(MISO_B200_E_INVALID, "trace has no jobs");  // sim.hpp:210
    for (int q = offs[i]; !inst.empty() && q < offs[i + 1]; ++q) {
      if (inst[size_t(q)] < 1) return fail(MISO_B200_E_INVALID, "instance count must be >= 1");
      J += inst[size_t(q)] - 1;
    }
    max_jobs = std::max(max_jobs, J);
  }
  if (!ctx->lut_valid) {
    const std::vector<int8_t>& lut = host_lut(ctx);
    if (!ctx->d_spare_lut) CUDA_TRY(cudaMalloc(&ctx->d_spare_lut, lut.size()));
    CUDA_TRY(cudaMemcpy(ctx->d_spare_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice));
    ctx->lut_valid = true;
  }
  const size_t stride = sim_workspace_stride(max_jobs, opt->cluster_size);
  const size_t need = stride * size_t(n_seeds);
  if (need > ctx->sim_ws_bytes) {
    if (int rc = stop_server(ctx)) return rc;
    cudaFree(ctx->d_sim_ws);
    ctx->d_sim_ws = nullptr;
    CUDA_TRY(cudaMalloc(&ctx->d_sim_ws, need));
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
  p.max_events = opt->max_events ? opt->max_events : 100000000ull;
  p.track_stp = (flags & MISO_B200_SIM_JCT_ONLY) ? 0 : 1;
  p.en0 = ctx->en0;
  p.en1 = ctx->en1;
  SimBatch b{};
  b.n_seeds = n_seeds;
  b.max_jobs = max_jobs;
  b.job_offsets = job_offsets;
  b.task_trace = task_trace;
  b.static_counts = static_counts;
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
  default_model(w2, w1);
  CUDA_TRY(launch_simulate(b, p, w2, w1, s));
  return MISO_B200_OK;
}
}  // namespace

int miso_b200_simulate_batch_ex(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                                const int32_t* task_trace, const uint8_t* static_counts,
                                const int32_t* job_offsets, const double* arrival_s,
                                const double* base_s, const double* speeds5,
                                const uint8_t* mem_gb, const int8_t* qos_kind,
                                const uint8_t* instances, const uint64_t* rng_seed,
                                miso_b200_sim_metrics* metrics, int64_t* job_jct_us,
                                int64_t* job_out, miso_b200_log_record* log, int64_t log_cap,
                                double* stp_series, int64_t stp_cap, unsigned flags,
                                void* stream) {
  return simulate_impl(ctx, opt, n_seeds, task_trace, static_counts, job_offsets, arrival_s,
                       base_s, speeds5, mem_gb, qos_kind, instances, rng_seed, metrics,
                       job_jct_us, job_out, log, log_cap, stp_series, stp_cap, flags, nullptr,
                       stream);
}

int miso_b200_simulate_batch_pruned(miso_b200_ctx* ctx, const miso_b200_sim_options* opt,
                                    int n_tasks, const int32_t* task_trace,
                                    const uint8_t* static_counts, const int32_t* job_offsets,
                                    const double* arrival_s, const double* base_s,
                                    const double* speeds5, const uint8_t* mem_gb,
                                    const int8_t* qos_kind, const uint64_t* rng_seed,
                                    miso_b200_sim_metrics* metrics, int64_t* bound,
                                    unsigned flags, void* stream) {
  if (!opt || opt->policy != MISO_B200_POLICY_OPTSTA)
    return fail(MISO_B200_E_INVALID, "pruned runs are optsta candidate searches");
  if (!task_trace || !bound) return fail(MISO_B200_E_INVALID, "task_trace and bound are required");
  return simulate_impl(ctx, opt, n_tasks, task_trace, static_counts, job_offsets, arrival_s,
                       base_s, speeds5, mem_gb, qos_kind, nullptr, rng_seed, metrics, nullptr,
                       nullptr, nullptr, 0, nullptr, 0, flags, bound, stream);
}

extern "C++" {
namespace {
struct DevBuf {  // owning device allocation for the synchronous host-pointer calls
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
};
template <class T>
int upload(DevBuf& d, const T* src, size_t n, cudaStream_t s) {
  if (!src || n == 0) return MISO_B200_OK;
  CUDA_TRY(cudaMalloc(&d.p, n * sizeof(T)));
  CUDA_TRY(cudaMemcpyAsync(d.p, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return MISO_B200_OK;
}
int alloc_out(DevBuf& d, size_t bytes) {
  if (bytes == 0) return MISO_B200_OK;
  CUDA_TRY(cudaMalloc(&d.p, bytes));
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
  {
    DeviceGuard g(ctx->device);
    if (int rc = stop_server(ctx)) return rc;  // the staging buffers below are cudaFree'd
  }
  if (!job_offsets || !arrival_s || !base_s || !speeds5 || !mem_gb || !qos_kind || !rng_seed ||
      !metrics)
    return fail(MISO_B200_E_INVALID, "null buffer");
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
  int max_jobs = 0;
  for (int i = 0; i < n_traces; ++i) {
    int Jt = job_offsets[i + 1] - job_offsets[i];
    for (int q = job_offsets[i]; instances && q < job_offsets[i + 1]; ++q) {
      if (instances[q] < 1) return fail(MISO_B200_E_INVALID, "instance count must be >= 1");
      Jt += instances[q] - 1;
    }
    max_jobs = std::max(max_jobs, Jt);
  }
  const size_t J = size_t(job_offsets[n_traces]);
  DeviceGuard g(ctx->device);
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  cudaStream_t s = ctx->streams[0];
  DevBuf d_tt, d_sc, d_off, d_arr, d_base, d_sp, d_mem, d_qos, d_inst, d_seed, d_met, d_jo, d_log,
      d_stp;
  int rc;
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
  if ((rc = alloc_out(d_met, sizeof(miso_b200_sim_metrics) * size_t(n_tasks)))) return rc;
  const size_t jo_n = job_out ? size_t(n_tasks) * size_t(max_jobs) * MISO_B200_JOB_OUT_FIELDS : 0;
  if ((rc = alloc_out(d_jo, jo_n * sizeof(int64_t)))) return rc;
  const size_t log_n = log ? size_t(n_tasks) * size_t(std::max<int64_t>(log_cap, 0)) : 0;
  if ((rc = alloc_out(d_log, log_n * sizeof(miso_b200_log_record)))) return rc;
  const size_t stp_n = stp_series ? size_t(n_tasks) * 2 * size_t(std::max<int64_t>(stp_cap, 0)) : 0;
  if ((rc = alloc_out(d_stp, stp_n * sizeof(double)))) return rc;
  DevBuf d_bound;
  std::vector<int64_t> b0(prune ? size_t(n_traces) : 0, INT64_MAX);  // no completed candidate yet
  if ((rc = upload(d_bound, b0.data(), b0.size(), s))) return rc;
  rc = simulate_impl(
      ctx, opt, n_tasks, static_cast<const int32_t*>(d_tt.p), static_cast<const uint8_t*>(d_sc.p),
      static_cast<const int32_t*>(d_off.p), static_cast<const double*>(d_arr.p),
      static_cast<const double*>(d_base.p), static_cast<const double*>(d_sp.p),
      static_cast<const uint8_t*>(d_mem.p), static_cast<const int8_t*>(d_qos.p),
      prune ? nullptr : static_cast<const uint8_t*>(d_inst.p), static_cast<const uint64_t*>(d_seed.p),
      static_cast<miso_b200_sim_metrics*>(d_met.p),
      nullptr, static_cast<int64_t*>(d_jo.p), static_cast<miso_b200_log_record*>(d_log.p),
      log ? log_cap : 0, static_cast<double*>(d_stp.p), stp_series ? stp_cap : 0, flags,
      prune ? static_cast<int64_t*>(d_bound.p) : nullptr, s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(metrics, d_met.p, sizeof(miso_b200_sim_metrics) * size_t(n_tasks),
                           cudaMemcpyDeviceToHost, s));
  if (jo_n) CUDA_TRY(cudaMemcpyAsync(job_out, d_jo.p, jo_n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (log_n) CUDA_TRY(cudaMemcpyAsync(log, d_log.p, log_n * sizeof(miso_b200_log_record), cudaMemcpyDeviceToHost, s));
  if (stp_n) CUDA_TRY(cudaMemcpyAsync(stp_series, d_stp.p, stp_n * sizeof(double), cudaMemcpyDeviceToHost, s));
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
  if (int rc = stop_server(ctx)) return rc;  // the staging buffers below are cudaFree'd
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  cudaStream_t s = ctx->streams[0];
  DevBuf d_in, d_out;
  int rc;
  if ((rc = upload(d_in, truth3, size_t(ncols) * 3, s))) return rc;
  if ((rc = alloc_out(d_out, size_t(ncols) * 5 * sizeof(double)))) return rc;
  rc = miso_b200_predict_batch(ctx, static_cast<const double*>(d_in.p), ncols, cols_per_group,
                               first_nonce, rng_seed, mode, target_mae, w2, w1,
                               static_cast<double*>(d_out.p), s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out5, d_out.p, size_t(ncols) * 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
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
  if (int rc = stop_server(ctx)) return rc;  // the staging buffers below are cudaFree'd
  if (!ctx->streams[0]) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
  cudaStream_t s = ctx->streams[0];
  const size_t J = size_t(n_traces) * size_t(job_count);
  DevBuf d_seed, d_a, d_d, d_sp, d_m;
  int rc;
  if ((rc = upload(d_seed, seeds, size_t(n_traces), s))) return rc;
  if ((rc = alloc_out(d_a, J * sizeof(double)))) return rc;
  if ((rc = alloc_out(d_d, J * sizeof(double)))) return rc;
  if ((rc = alloc_out(d_sp, J * 5 * sizeof(double)))) return rc;
  if ((rc = alloc_out(d_m, J * sizeof(int)))) return rc;
  rc = miso_b200_generate_traces_device(
      ctx, static_cast<const uint64_t*>(d_seed.p), n_traces, job_count, lambda_s, max_duration_s,
      dist, sigma, fixed_s, lo_s, hi_s, static_cast<double*>(d_a.p), static_cast<double*>(d_d.p),
      static_cast<double*>(d_sp.p), static_cast<int*>(d_m.p), s);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(arrival_s, d_a.p, J * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(duration_s, d_d.p, J * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(speeds5, d_sp.p, J * 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(mem_gb, d_m.p, J * sizeof(int), cudaMemcpyDeviceToHost, s));
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

int miso_b200_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(MISO_B200_E_INVALID, "null out pointer");
  CUDA_TRY(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
  return MISO_B200_OK;
}

void miso_b200_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
