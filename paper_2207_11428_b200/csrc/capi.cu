// capi.cu -- the C ABI (include/miso_b200.h): contexts, catalogs, launch plumbing and the
// host-pointer pipelines. Host-side C++; the kernels live in *_kernel.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/miso_b200.h"
#include "candidates_gen.cuh"
#include "internal.h"

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

int ensure_host_scratch(miso_b200_ctx* ctx, size_t rows, size_t inst) {
  if (!ctx->streams[0]) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[0], cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->streams[1], cudaStreamNonBlocking));
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
  cudaFree(ctx->d_speeds);
  cudaFree(ctx->d_offsets);
  cudaFree(ctx->d_cand);
  cudaFree(ctx->d_obj);
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
  for (uint64_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i]) return fail(MISO_B200_E_MALFORMED, "offsets must be non-decreasing");
  DeviceGuard g(ctx->device);
  const size_t rows = offsets[n];
  int rc = ensure_host_scratch(ctx, rows, n);
  if (rc) return rc;
  // Two-stream pipeline: chunk k's H2D overlaps chunk k-1's search and D2H.
  const uint64_t kChunk = 1u << 17;
  int k = 0;
  for (uint64_t i0 = 0; i0 < n; i0 += kChunk, ++k) {
    const uint64_t i1 = std::min(n, i0 + kChunk);
    cudaStream_t s = ctx->streams[k & 1];
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

int miso_b200_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(MISO_B200_E_INVALID, "null out pointer");
  CUDA_TRY(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
  return MISO_B200_OK;
}

void miso_b200_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
