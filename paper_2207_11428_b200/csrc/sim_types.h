// sim_types.h -- shared host/device types of the batched simulator (kernel (c)).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/miso_b200.h"

namespace miso_b200 {

typedef miso_b200_sim_metrics SimMetrics;
typedef miso_b200_log_record LogRec;

enum LogKind : uint8_t {
  kLogArrival = MISO_B200_LOG_ARRIVAL, kLogAdmit = MISO_B200_LOG_ADMIT,
  kLogStart = MISO_B200_LOG_START, kLogCkptStart = MISO_B200_LOG_CKPT_START,
  kLogMpsStart = MISO_B200_LOG_MPS_START, kLogMpsWindow = MISO_B200_LOG_MPS_WINDOW,
  kLogMpsEnd = MISO_B200_LOG_MPS_END, kLogReconfigStart = MISO_B200_LOG_RECONFIG_START,
  kLogPartition = MISO_B200_LOG_PARTITION, kLogAssign = MISO_B200_LOG_ASSIGN,
  kLogComplete = MISO_B200_LOG_COMPLETE, kLogShrink = MISO_B200_LOG_SHRINK,
  kLogAdmitSlot = MISO_B200_LOG_ADMIT_SLOT, kLogMigrate = MISO_B200_LOG_MIGRATE,
  kLogSpawn = MISO_B200_LOG_SPAWN,
};

// job_out record per job: completion_us, acc_us[5], parent (-1), clone ordinal k
constexpr int kJobOutFields = 8;

struct SimParams {
  int policy, cluster_size, noisy, check_invariants;
  int track_stp;  // 0: JCT-only run, refresh_stp skipped (MISO_B200_SIM_JCT_ONLY)
  int64_t window_us, reconfig_us, ckpt_us;
  double interference, target_mae, drift_threshold;
  uint64_t max_events;
  uint64_t en0, en1;  // enabled-candidate mask of the context's catalog
};

struct SimBatch {
  int n_seeds, n_traces, max_jobs;
  const int32_t* job_offsets;   // per trace
  const int32_t* task_trace;    // per task (nullable: task i = trace i)
  const uint8_t* static_counts; // per task, optsta static partition
  const double* arrival_s;
  const double* base_s;
  const double* speeds5;
  const uint8_t* mem_gb;
  const uint8_t* instances;     // per trace job, JobProfile::instance_count (nullable: all 1)
  const int8_t* qos_kind;
  const uint64_t* rng_seed;
  const int8_t* spare_lut;
  unsigned char* workspace;
  size_t ws_stride;
  SimMetrics* metrics;
  int64_t* job_jct_us;
  int64_t* job_out;  // per task: max_jobs x {completion_us (-1 unfinished), acc_us[5]}
  LogRec* log;
  int64_t log_cap;
  double* stp_series;
  int64_t stp_cap;
  int64_t* prune_bound;  // per trace (nullable): chosen-only best-static search, see capi
  // the noisy predictor's draws, precomputed per task for call nonces 1..draws_k (nullable):
  // [task][nonce - 1][column 0..6][entry 4g, 3g], pack_draw encoded (predict.cuh)
  const double* draws;
  int draws_k;
};

// Per-seed workspace layout: [jobs][gpus][slots][queue][progress mask][rate scratch]
constexpr size_t kSimJobBytes = 216;
constexpr size_t kSimGpuBytes = 256;
__host__ __device__ inline size_t sim_al(size_t x) { return (x + 127) & ~size_t(127); }
__host__ __device__ inline size_t sim_ws_gpus_off(int J) { return sim_al(size_t(J) * kSimJobBytes); }
__host__ __device__ inline size_t sim_ws_slots_off(int J, int G) {
  return sim_ws_gpus_off(J) + sim_al(size_t(G) * kSimGpuBytes);
}
__host__ __device__ inline size_t sim_ws_queue_off(int J, int G) {
  return sim_ws_slots_off(J, G) + sim_al(size_t(J + G) * 16);
}
__host__ __device__ inline size_t sim_ws_mask_off(int J, int G) {
  return sim_ws_queue_off(J, G) + sim_al(size_t(J + 1) * 4);
}
__host__ __device__ inline size_t sim_ws_scratch_off(int J, int G) {
  return sim_ws_mask_off(J, G) + sim_al(size_t((J + 31) / 32 + 32) * 4);
}
__host__ __device__ inline size_t sim_ws_prefix_off(int J, int G) {
  return sim_ws_scratch_off(J, G) + sim_al(size_t(J + 32) * 8);
}
__host__ __device__ inline size_t sim_ws_jst_off(int J, int G) {
  return sim_ws_prefix_off(J, G) + sim_al(size_t(J + 32) * 8);
}
__host__ __device__ inline size_t sim_ws_freemask_off(int J, int G) {
  return sim_ws_jst_off(J, G) + sim_al(size_t(J + 32));
}
// dense per-kind effective true speeds (5 x J doubles, kind-major) and arrival times (J int64)
__host__ __device__ inline size_t sim_ws_efftruth_off(int J, int G) {
  return sim_ws_freemask_off(J, G) + sim_al(size_t(5) * ((G + 31) / 32) * 4);
}
__host__ __device__ inline size_t sim_ws_arrival_off(int J, int G) {
  return sim_ws_efftruth_off(J, G) + sim_al(size_t(5) * J * 8);
}
// miso/oracle placement view: one byte per GPU
__host__ __device__ inline size_t sim_ws_gplace_off(int J, int G) {
  return sim_ws_arrival_off(J, G) + sim_al(size_t(J) * 8);
}
__host__ __device__ inline size_t sim_ws_total(int J, int G) {
  return sim_ws_gplace_off(J, G) + sim_al(size_t(G));
}

struct ModelW;  // predict.cuh

size_t sim_workspace_stride(int max_jobs, int cluster_size);
// one kernel per policy (sim_pol_*.cu); PRUNE = the chosen-only best-static search's runs
template <int POL, bool PRUNE>
cudaError_t launch_sim(const SimBatch& b, const SimParams& p, const ModelW& w, cudaStream_t s);
size_t sim_sizeof_job();
size_t sim_sizeof_gpu();
cudaError_t launch_simulate(const SimBatch& b, const SimParams& p, const double* w2,
                            const double* w1, cudaStream_t stream);
// The noisy predictor's draws of every task for call nonces 1..k (SimBatch::draws), one thread
// per draw: the throughput-bound half of finish_profiling, taken out of the event loop.
cudaError_t launch_sim_draws(const uint64_t* rng_seed, int n_tasks, int k, double* out,
                             cudaStream_t stream);

}  // namespace miso_b200
