/*
 * miso_b200.h -- C ABI of the B200-native MISO decision core.
 *
 * Plain pointers and sizes, no C++ or torch types. Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj/include/miso/). Status
 * codes mirror the reference CLI's exit codes (tools/miso_cli.cpp:4-5) as negatives:
 *   0 ok, -1 unexpected/CUDA error, -2 invalid argument, -3 malformed input, -4 infeasible.
 * Per-item outcomes of batch calls are reported in-band (see MISO_B200_CAND_*), never by
 * aborting the batch: the reference throws per call, a batch reports per instance.
 *
 * Threading: one context per device; a context may be used from one host thread at a time.
 * Device-pointer calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy default
 * stream) and do not synchronize. Host-pointer calls (`*_host`) are synchronous and overlap
 * H2D, compute and D2H internally; pass pinned memory (miso_b200_host_alloc) for full speed.
 */
#ifndef MISO_B200_H
#define MISO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MISO_B200_OK 0
#define MISO_B200_E_UNEXPECTED (-1)
#define MISO_B200_E_INVALID (-2)
#define MISO_B200_E_MALFORMED (-3)
#define MISO_B200_E_INFEASIBLE (-4)

/* Per-instance decision byte written by the optimize calls:
 *   0..110  winning candidate id (decode with miso_b200_candidate)
 *   0xFF    no valid assignment       == optimize_partition returning std::nullopt
 *                                        (optimizer.hpp:102)
 *   0xFE    job count m outside 1..7  == optimize_partition throwing invalid_argument
 *                                        (optimizer.hpp:65-66)                          */
#define MISO_B200_CAND_INFEASIBLE 0xFF
#define MISO_B200_CAND_BAD_M 0xFE
#define MISO_B200_NUM_CANDIDATES 111
#define MISO_B200_NUM_KINDS 5 /* slice kinds 1g,2g,3g,4g,7g = 0..4 (topology.hpp:27-45) */

typedef struct miso_b200_ctx miso_b200_ctx;

/* Library version (major*10000 + minor*100 + patch). */
int miso_b200_version(void);
/* Message of the last failing call on this host thread ("" if none). */
const char* miso_b200_last_error(void);

/* Create/destroy a context on a CUDA device. Owns the candidate table for its catalog and
 * scratch buffers for the host-pointer paths. */
int miso_b200_create(int device, miso_b200_ctx** out);
void miso_b200_destroy(miso_b200_ctx* ctx);

/* Replaces PartitionCatalog (topology.hpp:184-208, load_catalog :276-326): `counts` holds
 * n_entries rows of per-kind counts [1g,2g,3g,4g,7g] in the catalog's own order (the order
 * entry indices refer to). Rows must be feasible partitions (PartitionConfig::violation,
 * topology.hpp:84-101) and distinct; else -2. A new context uses default_catalog()
 * (topology.hpp:205-208). */
int miso_b200_set_catalog(miso_b200_ctx* ctx, const uint8_t* counts, int n_entries);
/* Copies the active catalog (<= 36 rows of 5 counts) into `counts`; returns n_entries. */
int miso_b200_get_catalog(const miso_b200_ctx* ctx, uint8_t* counts);

/* Decodes a candidate id: its index in the ACTIVE catalog (-1 if the entry is not in it),
 * its job count m and the slice kind of each job (place[0..m-1]). */
int miso_b200_candidate(const miso_b200_ctx* ctx, int cand, int* entry, int* m, uint8_t place[7]);

/* Batched optimize_partition (optimizer.hpp:62-115) over independent job mixes, DEVICE
 * pointers. speeds: packed rows of 5 FP64 effective speeds (kind order 1g..7g, already zeroed
 * by effective_speed, profiles.hpp:60-65) for sum(m) jobs; offsets: n+1 job offsets (instance
 * i owns rows offsets[i]..offsets[i+1]-1). Writes cand[i] (see MISO_B200_CAND_*) and obj[i]
 * (the FP64 objective, bit-exact with the reference; 0 when no decision). */
int miso_b200_optimize_batch(miso_b200_ctx* ctx, const double* speeds, const uint32_t* offsets,
                             uint64_t n, uint8_t* cand, double* obj, void* stream);

/* One batch for miso_b200_optimize_batches: the arguments of miso_b200_optimize_batch. */
typedef struct miso_b200_batch {
  const double* speeds;
  const uint32_t* offsets;
  uint64_t n;
  uint8_t* cand;
  double* obj;
} miso_b200_batch;

/* miso_b200_optimize_batch over n_batches independent batches (DEVICE pointers, each with the
 * contract above) in one stream-ordered call: up to 32 batches share one persistent-kernel
 * launch, so a queue of batches pays the launch's fixed cost (grid start, first-tile latency,
 * CTA tail) once instead of per batch. Outputs are the same bytes as one call per batch. The
 * descriptor array is read during the call (host memory; it may be reused on return). */
int miso_b200_optimize_batches(miso_b200_ctx* ctx, const miso_b200_batch* batches,
                               int n_batches, void* stream);

/* Same contract with HOST pointers: chunked H2D -> search -> D2H pipeline over two streams.
 * Synchronous. Offsets are validated chunk by chunk as the pipeline advances: on
 * MISO_B200_E_MALFORMED, results of instances before the offending chunk may have been written. */
int miso_b200_optimize_batch_host(miso_b200_ctx* ctx, const double* speeds,
                                  const uint32_t* offsets, uint64_t n, uint8_t* cand,
                                  double* obj);

/* One-instance drop-in for optimize_partition (optimizer.hpp:62-63), host pointers.
 * Returns 1 (decision written: entry index in the active catalog, place[m], *obj),
 * 0 (std::nullopt) or -2 (m outside 1..7, invalid_argument). */
int miso_b200_optimize(miso_b200_ctx* ctx, const double* speeds, int m, int* entry,
                       uint8_t* place, double* obj);

/* ---- predictor (kernel (a)) ------------------------------------------------------------ */

/* The shared default small-slice model: fit_small_slice_model(make_training_corpus(3000,
 * 0x5eed)) (sim.hpp:894-898, profiles.hpp:340-361, 469-475); weights over (f7, f4, f3, 1).
 * Computed once on the host. */
int miso_b200_default_model(double w2[4], double w1[4]);

/* Batched predict_mig_speeds + extrapolate_small_slices (profiles.hpp:214-253, 370-384),
 * DEVICE pointers. Column j is column j % cols_per_group of MPS group j / cols_per_group,
 * whose call nonce is first_nonce + j / cols_per_group (real jobs occupy columns
 * 0..cols_per_group-1, pad_to_seven profiles.hpp:106-113). truth3: (f7, f4, f3) per column;
 * out5: the estimated speed table per column, kind order 1g..7g. mode 0 = oracle, 1 = noisy
 * (PredictorSpec::Mode, profiles.hpp:173-178); target_mae in [0, 0.5] else -2. w2/w1 NULL =
 * the default model. mode 2 = extrapolate_small_slices alone (profiles.hpp:370-384): truth3
 * holds a mig matrix's (7g, 4g, 3g) rows, taken as given (no re-anchoring), and out5 gets
 * them back with the extrapolated 2g/1g. */
int miso_b200_predict_batch(miso_b200_ctx* ctx, const double* truth3, uint64_t ncols,
                            int cols_per_group, uint64_t first_nonce, uint64_t rng_seed, int mode,
                            double target_mae, const double* w2, const double* w1, double* out5,
                            void* stream);

/* The same with HOST pointers (synchronous). */
int miso_b200_predict_host(miso_b200_ctx* ctx, const double* truth3, uint64_t ncols,
                           int cols_per_group, uint64_t first_nonce, uint64_t rng_seed, int mode,
                           double target_mae, const double* w2, const double* w1, double* out5);

/* Fused per-GPU decision for n rosters, DEVICE pointers: for each instance i (jobs
 * offsets[i]..offsets[i+1]-1 in columns 0..m-1, call nonce nonce[i]) predict every job's
 * speeds, zero them by memory demand (mem_gb) and QoS floor (qos_kind: slice kind 0..4, -1 =
 * none) as effective_speed does (profiles.hpp:60-65), then optimize_partition -- the
 * finish_profiling -> reopt_and_apply step of the simulator (sim.hpp:691-733). Writes
 * cand/obj as miso_b200_optimize_batch, and the zeroed speed tables to est5 (sum(m) x 5) when
 * est5 != NULL. */
int miso_b200_decide_batch(miso_b200_ctx* ctx, const double* truth3, const uint8_t* mem_gb,
                           const int8_t* qos_kind, const uint32_t* offsets, const uint64_t* nonce,
                           uint64_t n, uint64_t rng_seed, int mode, double target_mae,
                           const double* w2, const double* w1, uint8_t* cand, double* obj,
                           double* est5, void* stream);

/* One roster, HOST pointers (config 1: the reference CPU example's chain, latency path).
 * Returns 1 (entry, place[m], *obj written), 0 (no valid partition) or a negative status.
 * est5 (optional, m x 5) receives the zeroed estimated speed tables. Default model. */
int miso_b200_decide(miso_b200_ctx* ctx, const double* truth3, const uint8_t* mem_gb,
                     const int8_t* qos_kind, int m, uint64_t nonce, uint64_t rng_seed, int mode,
                     double target_mae, int* entry, uint8_t* place, double* obj, double* est5);

/* miso_b200_decide's execution mode. idle_us > 0 (the default: 2000, or the environment's
 * MISO_B200_DECIDE_IDLE_US): a one-warp server kernel stays resident between calls, polling a
 * request mailbox in mapped pinned memory, and exits after idle_us without a request (it is
 * relaunched on the next call). While it runs, device-wide synchronisation
 * (cudaDeviceSynchronize, cudaFree) waits for it, i.e. at most idle_us after the last call.
 * idle_us = 0: one kernel launch per call. Stops a running server. A context serves one host
 * thread at a time. */
int miso_b200_decide_server(miso_b200_ctx* ctx, int idle_us);

/* max_spare_slice_for (topology.hpp:227-252) over the context's catalog: the largest slice
 * kind a partition could spare beside jobs pinned to at least min_kinds[0..n) (kind 0..4 =
 * 1g..7g), -1 if none (std::nullopt). This reads the table the simulator uses on the device
 * (the spare-slice LUT of placement, sim.hpp:581-607). */
int miso_b200_max_spare_slice(miso_b200_ctx* ctx, const uint8_t* min_kinds, int n, int* kind);

/* ---- cluster simulator (kernel (c)) ------------------------------------------------------ */

/* Policies (sim.hpp:42). */
#define MISO_B200_POLICY_NOPART 0
#define MISO_B200_POLICY_OPTSTA 1
#define MISO_B200_POLICY_ORACLE 2
#define MISO_B200_POLICY_MISO 3

/* Per-seed status (SimInvariantError and friends become per-seed codes; 0 = ok). */
#define MISO_B200_SIM_INVARIANT 1         /* work conservation / accounting / plan mismatch */
#define MISO_B200_SIM_NO_PARTITION 2      /* "no feasible partition for admitted roster" */
#define MISO_B200_SIM_INFEASIBLE_SLICE 3  /* "placed on infeasible slice" */
#define MISO_B200_SIM_EVENT_BUDGET 4      /* "event budget exhausted" (sim.hpp:224): the events
                                             pushed (= popped by the reference, stale ones
                                             included) exceed max_events */
#define MISO_B200_SIM_PRUNED 5            /* stopped by miso_b200_simulate_batch_pruned's bound */
#define MISO_B200_SIM_BAD_INPUT 6         /* the reference's std::invalid_argument for this
                                             task's trace or options; metrics.detail says which:
                                             MISO_B200_BAD_* | (job index << 8) */

/* metrics.detail codes of MISO_B200_SIM_BAD_INPUT. Per trace job, in the reference's order
 * (validate_profile, profiles.hpp:67-87; init_jobs, sim.hpp:246-254): */
#define MISO_B200_BAD_BASE 1              /* "base duration must be positive" */
#define MISO_B200_BAD_MEM 2               /* "memory demand must be in (0, 40] GB" */
#define MISO_B200_BAD_SPEED_RANGE 3       /* + kind 0..4: "speed on <kind> outside (0,1]" */
#define MISO_B200_BAD_SPEED_7G 8          /* "speed on 7g must be exactly 1" */
#define MISO_B200_BAD_MONOTONE 9          /* "speed table not monotone in gpc count" */
#define MISO_B200_BAD_INSTANCES 10        /* "instance count must be >= 1" */
#define MISO_B200_BAD_FIRST_ARRIVAL 11    /* "first arrival must be at t=0" */
#define MISO_B200_BAD_ARRIVAL_ORDER 12    /* "arrival times must be non-decreasing" */
/* per task: */
#define MISO_B200_BAD_NO_JOBS 13          /* "trace has no jobs" (sim.hpp:210) */
#define MISO_B200_BAD_TASK_TRACE 14       /* task_trace entry outside [0, n_traces) */
#define MISO_B200_BAD_STATIC 15           /* static partition is not a feasible partition */
#define MISO_B200_BAD_CAPACITY 16         /* trace jobs + clones exceed the call's max_jobs */

/* SimOptions (sim.hpp:81-96) + OverheadSpec (:62-67) + PredictorSpec (profiles.hpp:173-178).
 * Durations in seconds are converted with us_from_s = llround(s * 1e6) (sim.hpp:136). */
typedef struct {
  int policy;                      /* MISO_B200_POLICY_* */
  int cluster_size;                /* GPUs, >= 1 */
  double mig_reconfig_s;           /* default 4 */
  double checkpoint_restart_s;     /* default 30 */
  double mps_window_s;             /* default 10 */
  double interference;             /* default 0.8, in (0, 1] */
  int predictor_noisy;             /* 0 oracle predictor, 1 noisy */
  double target_mae;               /* default 0.017, [0, 0.5] */
  int check_invariants;            /* default 1 */
  double reprofile_drift_threshold;/* default 0 (off) */
  uint64_t max_events;             /* default 100000000 */
  /* SimOptions::small_slice_model (sim.hpp:88, 894-896): fitted != 0 uses w2/w1 (weights over
   * (f7, f4, f3, 1), LinearMap profiles.hpp:259-273); 0 uses the shared default model. */
  int small_slice_model_fitted;
  double small_slice_w2[4], small_slice_w1[4];
} miso_b200_sim_options;

/* MetricsReport (sim.hpp:106-122) scalars, per seed. */
typedef struct {
  int status, completed, job_count, completed_count, repartitions, migrations, mps_sessions;
  int detail;  /* MISO_B200_SIM_BAD_INPUT: MISO_B200_BAD_* | (job index << 8); else 0 */
  double avg_jct_s, makespan_s, stp_time_avg, jct_sum_s;
  double queue_frac, mps_frac, checkpoint_frac, run_frac, idle_frac;
  int64_t events, log_records, stp_points;
} miso_b200_sim_metrics;

/* Compact event-log record; render with the reference's text format (sim.hpp:365-367). */
typedef struct {
  int64_t t;       /* now_, integer microseconds */
  uint8_t kind;    /* MISO_B200_LOG_* */
  uint8_t x;       /* slice kind / roster size */
  uint16_t gpu;    /* 0xFFFF = none */
  int32_t job;     /* job index in the trace, -1 = none */
  uint32_t a, b;   /* payload (counts, levels, packed partition, 64-bit durations as a|b<<32) */
  double v;        /* rate for "start" */
} miso_b200_log_record;

#define MISO_B200_LOG_ARRIVAL 0
#define MISO_B200_LOG_ADMIT 1
#define MISO_B200_LOG_START 2
#define MISO_B200_LOG_CKPT_START 3
#define MISO_B200_LOG_MPS_START 4
#define MISO_B200_LOG_MPS_WINDOW 5
#define MISO_B200_LOG_MPS_END 6
#define MISO_B200_LOG_RECONFIG_START 7
#define MISO_B200_LOG_PARTITION 8  /* x = roster size, a = packed counts (4 bits per kind) */
#define MISO_B200_LOG_ASSIGN 9     /* follows PARTITION: job, x = slice kind */
#define MISO_B200_LOG_COMPLETE 10
#define MISO_B200_LOG_SHRINK 11
#define MISO_B200_LOG_ADMIT_SLOT 12 /* optsta admit: x = slot */
#define MISO_B200_LOG_MIGRATE 13    /* optsta migration: x = slice kind, a = slot */
#define MISO_B200_LOG_SPAWN 14      /* multi-instance clone: job = clone, a = parent job */

/* generate_trace (workload.hpp:97-114) on the host: dist 0 lognormal(sigma), 1 fixed(fixed_s),
 * 2 uniform(lo_s, hi_s). Arrays of job_count; speeds5 kind order 1g..7g. */
int miso_b200_generate_trace(uint64_t seed, int job_count, double lambda_s,
                             double max_duration_s, int dist, double sigma, double fixed_s,
                             double lo_s, double hi_s, double* arrival_s, double* duration_s,
                             double* speeds5, int* mem_gb);

/* generate_trace for n_traces seeds at once on `threads` host threads (<= 0: all hardware
 * threads), same spec for every trace; trace r writes job_count entries at offset r*job_count of
 * each output array (speeds5: 5 per job). Bit-identical to n calls of miso_b200_generate_trace. */
int miso_b200_generate_traces(const uint64_t* seeds, int n_traces, int job_count, double lambda_s,
                              double max_duration_s, int dist, double sigma, double fixed_s,
                              double lo_s, double hi_s, int threads, double* arrival_s,
                              double* duration_s, double* speeds5, int* mem_gb);

/* generate_trace for n_traces seeds ON THE DEVICE (one warp per trace; DEVICE pointers,
 * stream-ordered): the same outputs as miso_b200_generate_traces, bit for bit (the reference's
 * libm calls -- exp, pow, log1p, log, cos -- are restated from glibc 2.39's FMA variants,
 * csrc/glibc_math*.cuh). Same validation and layout (trace r at offset r*job_count). */
int miso_b200_generate_traces_device(miso_b200_ctx* ctx, const uint64_t* seeds, int n_traces,
                                     int job_count, double lambda_s, double max_duration_s,
                                     int dist, double sigma, double fixed_s, double lo_s,
                                     double hi_s, double* arrival_s, double* duration_s,
                                     double* speeds5, int* mem_gb, void* stream);

/* The same generation on the device with HOST pointers (synchronous): seeds in, the arrays out
 * (n_traces x job_count, trace-major). */
int miso_b200_generate_traces_device_host(miso_b200_ctx* ctx, const uint64_t* seeds,
                                          int n_traces, int job_count, double lambda_s,
                                          double max_duration_s, int dist, double sigma,
                                          double fixed_s, double lo_s, double hi_s,
                                          double* arrival_s, double* duration_s, double* speeds5,
                                          int* mem_gb);

/* run_simulation (sim.hpp:976-979) for n_seeds independent tasks at once, one warp per task,
 * DEVICE pointers, stream-ordered (no host synchronisation; the library reads no device array
 * back). Task s simulates trace task_trace[s] (task_trace NULL: trace s); trace r (< n_traces)
 * owns jobs job_offsets[r]..job_offsets[r+1]-1 (arrival_s as in TraceJob, converted with
 * us_from_s on the device; must be non-decreasing with the first at 0, sim.hpp:251-254; base
 * duration s; truth speeds; memory GB; QoS kind or -1). max_jobs: an upper bound on any task's
 * job count including multi-instance clones (it sizes the per-task workspace). rng_seed[s]
 * seeds the noisy predictor (experiment.hpp:305 sets it to the trace seed). Policy optsta needs
 * static_counts (5 per task: the static partition's per-kind counts, a feasible partition;
 * SimOptions::static_partition, sim.hpp:86) -- one launch can evaluate every candidate of
 * best_static_partition (sim.hpp:1031-1066) for many traces. Invalid inputs (the reference's
 * std::invalid_argument: validate_profile, init_jobs) are reported per task as
 * MISO_B200_SIM_BAD_INPUT with metrics.detail.
 * Outputs: metrics[s]; optional job_jct_us (completion - arrival, -1 if unfinished; indexed by
 * trace job, so only with task_trace == NULL, else -2), event log (log_cap records per task)
 * and STP series (stp_cap (t, stp) pairs per task).
 * Tasks on one context share its workspace: calls on different streams must use different
 * contexts (or be ordered). */
int miso_b200_simulate_batch(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                             int n_traces, int max_jobs, const int32_t* task_trace,
                             const uint8_t* static_counts, const int32_t* job_offsets,
                             const double* arrival_s, const double* base_s, const double* speeds5,
                             const uint8_t* mem_gb, const int8_t* qos_kind,
                             const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                             int64_t* job_jct_us, miso_b200_log_record* log, int64_t log_cap,
                             double* stp_series, int64_t stp_cap, void* stream);

/* miso_b200_simulate_batch with multi-instance jobs, flags and per-job outputs.
 * instances (optional, per trace job): JobProfile::instance_count (>= 1; NULL = all 1). A job
 * with k > 1 spawns k - 1 clones "id#1".."id#(k-1)" at its first admission (nopart, optsta) or
 * estimate caching (miso, oracle), exactly as SimEngine::spawn_instances (sim.hpp:432-455);
 * the metrics then count them (job_count = trace jobs + clones spawned).
 * MISO_B200_SIM_JCT_ONLY: the tasks' consumer needs only the job-completion metrics (avg_jct_s,
 * jct_sum_s, makespan, the time fractions, counters): the STP series (refresh_stp,
 * sim.hpp:353-361) is not maintained, stp_time_avg/stp_points read 0 and stp_series must be
 * NULL. Every other field, the event order and the event log are unchanged (STP never feeds
 * back into decisions). best_static_partition (sim.hpp:1031-1066) reads only avg_jct_s of its
 * candidate runs.
 * job_out (optional, any task_trace): per task max_jobs x MISO_B200_JOB_OUT_FIELDS int64 --
 * the job's completion time in us (-1 if it never finished), its per-phase accumulated us
 * (queued, mps, checkpoint, running, idle), its parent job index (-1 for trace jobs) and clone
 * ordinal k: the inputs of MetricsReport::per_job (sim.hpp:916-929). Jobs are in SimEngine
 * order (trace jobs, then clones in spawn order). */
#define MISO_B200_SIM_JCT_ONLY 1u
#define MISO_B200_JOB_OUT_FIELDS 8
int miso_b200_simulate_batch_ex(miso_b200_ctx* ctx, const miso_b200_sim_options* opt, int n_seeds,
                                int n_traces, int max_jobs, const int32_t* task_trace,
                                const uint8_t* static_counts, const int32_t* job_offsets,
                                const double* arrival_s, const double* base_s,
                                const double* speeds5, const uint8_t* mem_gb,
                                const int8_t* qos_kind, const uint8_t* instances,
                                const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                                int64_t* job_jct_us, int64_t* job_out, miso_b200_log_record* log,
                                int64_t log_cap, double* stp_series, int64_t stp_cap,
                                unsigned flags, void* stream);

/* Chosen-only best-static search (run_trial_unit reads only best_static_partition(...).chosen,
 * experiment.hpp:337): optsta candidate runs as miso_b200_simulate_batch_ex (task_trace
 * required, single-instance traces), plus bound[n_traces] (device int64, in/out; start it at
 * INT64_MAX or at a completed candidate's exact JCT sum). Every task that completes lowers
 * bound[its trace] (atomic min) to its exact JCT sum in us. A running task keeps a lower bound
 * on its own sum (finished JCTs, now - arrival of arrived unfinished jobs, a run-time floor for
 * jobs not started) and stops once it exceeds bound * (1 + 1e-9) + 2 * jobs. Its metrics then
 * carry status MISO_B200_SIM_PRUNED and avg_jct_s = +inf. Its true avg_jct_s is strictly
 * greater than that completed candidate's, so the first minimum over the catalog (sim.hpp:1058)
 * is unchanged. Launch likely winners first (or in an earlier call with the same bound) so
 * the rest stop early. A stopped candidate is not run to its end: an invariant failure or an
 * event-budget exhaustion it would meet later (where the reference's best_static_partition
 * throws) goes unseen, so the chosen entry equals the reference's whenever the reference's
 * search completes without throwing. */
int miso_b200_simulate_batch_pruned(miso_b200_ctx* ctx, const miso_b200_sim_options* opt,
                                    int n_tasks, int n_traces, int max_jobs,
                                    const int32_t* task_trace,
                                    const uint8_t* static_counts, const int32_t* job_offsets,
                                    const double* arrival_s, const double* base_s,
                                    const double* speeds5, const uint8_t* mem_gb,
                                    const int8_t* qos_kind, const uint64_t* rng_seed,
                                    miso_b200_sim_metrics* metrics, int64_t* bound,
                                    unsigned flags, void* stream);

/* The same with HOST pointers (synchronous): inputs are copied to the device, results back.
 * n_traces = entries of job_offsets minus one. The C++ binding include/miso_b200_sim.hpp builds
 * run_simulation / best_static_partition / run_experiment_in_memory on this call.
 * MISO_B200_SIM_PRUNE: the tasks are a chosen-only best-static search, run as
 * miso_b200_simulate_batch_pruned with one bound per trace starting at INT64_MAX (optsta,
 * task_trace, single-instance traces, metrics only). */
#define MISO_B200_SIM_PRUNE 2u
int miso_b200_simulate_batch_host(miso_b200_ctx* ctx, const miso_b200_sim_options* opt,
                                  int n_tasks, int n_traces, const int32_t* task_trace,
                                  const uint8_t* static_counts, const int32_t* job_offsets,
                                  const double* arrival_s, const double* base_s,
                                  const double* speeds5, const uint8_t* mem_gb,
                                  const int8_t* qos_kind, const uint8_t* instances,
                                  const uint64_t* rng_seed, miso_b200_sim_metrics* metrics,
                                  int64_t* job_out, miso_b200_log_record* log, int64_t log_cap,
                                  double* stp_series, int64_t stp_cap, unsigned flags);

/* ---- several devices (one context each) ------------------------------------------------ */

/* Number of visible CUDA devices (0 if none). */
int miso_b200_device_count(void);

/* miso_b200_optimize_batch_host over n_ctx contexts (normally one per device): instances are
 * split into n_ctx contiguous ranges, each context runs its range's H2D -> search -> D2H
 * pipeline on its own host thread, and every decision lands at its instance's index in
 * cand/obj -- the same bytes as one context's call (instances are
 * independent). HOST pointers, synchronous. */
int miso_b200_optimize_batch_sharded(miso_b200_ctx* const* ctxs, int n_ctx, const double* speeds,
                                     const uint32_t* offsets, uint64_t n, uint8_t* cand,
                                     double* obj);

/* miso_b200_simulate_batch_host over n_ctx contexts: traces are split into n_ctx contiguous
 * ranges of about equal task counts; each context uploads only its traces and runs their tasks
 * (a trace's tasks stay on one device, so a pruned best-static search keeps its per-trace
 * bound) on its own host thread; outputs land at each task's index with the layout of one
 * miso_b200_simulate_batch_host call (job_out stride = the largest instance total of ALL
 * traces). The results equal one context's call byte for byte. Same arguments and flags. */
int miso_b200_simulate_batch_sharded(miso_b200_ctx* const* ctxs, int n_ctx,
                                     const miso_b200_sim_options* opt, int n_tasks, int n_traces,
                                     const int32_t* task_trace, const uint8_t* static_counts,
                                     const int32_t* job_offsets, const double* arrival_s,
                                     const double* base_s, const double* speeds5,
                                     const uint8_t* mem_gb, const int8_t* qos_kind,
                                     const uint8_t* instances, const uint64_t* rng_seed,
                                     miso_b200_sim_metrics* metrics, int64_t* job_out,
                                     miso_b200_log_record* log, int64_t log_cap,
                                     double* stp_series, int64_t stp_cap, unsigned flags);

/* Pinned host memory for the *_host paths. */
int miso_b200_host_alloc(size_t bytes, void** out);
void miso_b200_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* MISO_B200_H */
