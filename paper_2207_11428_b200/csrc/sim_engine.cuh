// sim_engine.cuh -- kernel (c): batched event-step cluster simulator, one warp per trace seed.
//
// Restates SimEngine (sim.hpp:202-972) for the nopart, optsta, oracle and miso policies. Every
// event of one seed is processed by one warp (one 32-thread block) in lockstep: all 32 lanes
// execute the (sequential) event logic redundantly -- uniform loads are broadcasts, uniform
// stores idempotent -- and split only for the data-parallel parts:
//   * next event: per-lane minima over owned event slots, one warp argmin per event (below);
//   * placement (place_dynamic, sim.hpp:581-607): warp argmin over GPUs, with
//     max_spare_slice_for (topology.hpp:227-252) replaced by a LUT over the roster's min-kind
//     counts, cached per GPU;
//   * predictor (finish_profiling, sim.hpp:691-714): one lane per roster column (mt19937_64
//     seeding + glibc-exact log/cos, predict.cuh), results exchanged by shuffles;
//   * STP refresh (sim.hpp:353-361): a dense per-job effective-rate array summed sequentially
//     over the window of arrived, unfinished jobs (bit-exact STP series).
// The partition search of reopt_and_apply (sim.hpp:716-733) is search.cuh's straight-line
// search, executed redundantly by all lanes.
//
// Engine state: the warp-uniform scalars (clock, queue bounds, counters, options, workspace
// pointers) live in ONE shared-memory record per block (g_sim_ctx), not in per-lane local
// memory: every access is a shared-memory broadcast at a fixed address, and the 32 redundant
// per-lane copies no longer occupy L1 beside the job records. Uniform updates are executed by
// all lanes of the converged warp (same value to the same address); per-lane state (each
// lane's event-slot minimum) is indexed by lane.
//
// The engine is a template over the policy (and the pruned best-static search's bookkeeping),
// instantiated once per policy in its own TU (sim_<policy>.cu): a kernel carries only its
// policy's code, which keeps the instruction footprint of the event loop small.
//
// Event queue: the reference keeps a binary heap with lazy deletion (stale events are popped
// and skipped, sim.hpp:284-299). Each job has at most one live job-scoped event and each GPU
// at most one live GPU-scoped event (every push is preceded by an epoch bump), so this engine
// keeps one slot per job and per GPU holding that live event's (t, prio, seq) key, with `seq`
// the same global push counter (sim.hpp:280-282); the next event is the minimum live key --
// the same total order the heap pops. A slot is cleared whenever its epoch is bumped.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/miso_b200.h"
#include "internal.h"
#include "predict.cuh"
#include "search.cuh"
#include "sim_types.h"

namespace miso_b200 {
namespace simk {

enum Phase : uint8_t { kQueued = 0, kMps = 1, kCkpt = 2, kRunning = 3, kIdle = 4 };
enum Mode : uint8_t { kGpuIdle = 0, kGpuMig = 1, kGpuMps = 2, kGpuReconfig = 3 };
enum EvKind : uint32_t { kEvArrival = 0, kEvMpsEnd = 1, kEvReconfigDone = 2, kEvCkptDone = 3,
                         kEvCompletion = 4 };
enum JobFlag : uint8_t { kRunState = 1, kDone = 2, kHasEst = 4, kSpawned = 8 };

constexpr int64_t kNoEvent = INT64_MAX;

struct DJob {
  double remaining, consumed, rate, base;
  double truth[5];
  double est[5];
  int64_t arrival_us, last_update_us, first_progress_us, completion_us;
  int64_t acc[5];
  uint32_t epoch;
  int16_t gpu;
  uint8_t phase, slice, mem, min_kind, flags;
  int8_t qos;
  int8_t slot;      // optsta slot index on its GPU
  uint8_t inst;     // JobProfile::instance_count (clones: 1)
  int16_t clone_k;  // clones: k of "parent#k"; trace jobs: 0
  int32_t parent;   // clones: parent job index; trace jobs: -1
  double lbp;       // pruned search: this job's term of Ctx::lb_p while started and unfinished
};

struct DGpu {
  double objective, plan_obj;
  double plan_speed[7];
  int32_t roster[7];
  int32_t plan_job[7];
  uint32_t epoch;
  uint8_t mode, mps_level, nroster, plan_n, plan_valid;
  uint8_t part[5], plan_part[5], kind_cnt[5];
  int8_t spare;
  uint8_t plan_slice[7];
  uint8_t nslots;           // optsta: fixed slots of the static partition (sim.hpp:167-170)
  uint8_t slot_kind[7];
  int32_t slot_job[7];
  uint8_t fcnt[5];          // optsta: free slots per kind
};

static_assert(sizeof(DJob) <= kSimJobBytes, "workspace job stride");
static_assert(sizeof(DGpu) <= kSimGpuBytes, "workspace gpu stride");

struct Slot {
  int64_t t;
  uint64_t pk;  // prio << 62 | seq << 3 | kind
};

struct Ctx {  // warp-uniform engine state: one record per block, in shared memory
  DJob* jobs;
  DGpu* gpus;
  Slot* slots;          // [J job slots][G gpu slots]
  int32_t* queue;       // FCFS order (arrival_us, idx), qhead..qtail
  double* rate_eff;     // [J] rate if progressing and not done, else 0.0 (refresh_stp)
  double* stp_prefix;   // [J] cached sequential partial sums of rate_eff over the window
  int stp_cmin;         // smallest job index whose rate_eff changed since the last refresh
  int stp_lo, n_arrived; // jobs < stp_lo are done; jobs >= n_arrived have not arrived
  int stp_hi;            // rate_eff is 0.0 at every index >= stp_hi (<= n_arrived; never shrinks)
  int chunk;            // event slots per lane: lane l owns [l*chunk, (l+1)*chunk)
  uint8_t* jst;         // [J] SoA job state for warp scans: phase | slice << 3 | done << 6
  uint32_t* freemask;   // optsta: [5][W] bit g set iff GPU g has a free slot of that kind
  double* efftruth;     // [5][J]: effective_speed(truth[k], k, mem, qos) per job (static)
  int64_t* arr_us;      // [J]: arrival_us per job (dense copy for coalesced scans)
  int W;                // words per freemask row
  int part_min_gpc;     // optsta: the GPC count of the static partition's smallest slice kind
  uint8_t* gplace;      // miso/oracle: [G] placement view of each GPU (sync_place)
  LogRec* log;
  int64_t log_cap, log_n;
  int J, G;             // J: job capacity (trace jobs + every possible clone)
  int J_used;           // trace jobs + clones spawned so far (jobs_.size() in the reference)
  // admission memo (optsta / nopart): capacity only grows when a slot / GPU is freed, so a
  // failed admission of the queue head stays failed until cap_gen moves
  uint32_t cap_gen, fail_gen;
  int fail_job;
  int qhead, qtail;
  int64_t now;
  uint64_t seq;
  uint64_t nonce;
  double stp_cur, stp_integral;
  int64_t stp_last;
  int64_t stp_points;
  double* stp_series;  // optional (t_s, stp) pairs
  int64_t stp_cap;
  bool stp_dirty;
  int repartitions, migrations, mps_sessions, done_count;
  int64_t first_progress, last_completion;
  int status, detail;
  uint64_t processed;
  // chosen-only best-static search (SimBatch::prune_bound): a lower bound on this run's exact
  // JCT sum (us) = finished JCTs + (now - arrival) of arrived unfinished jobs + a runtime floor
  // for every job that has not started (see runtime_floor_us)
  bool prune;
  int64_t lb_fin, lb_narr, lb_arrsum, lb_unstarted;
  // started, unfinished jobs: sum of remaining_work / prune_mx in seconds, kept as
  // lb_p - lb_v * now_s with per-job terms (remaining + rate * t_update) / mx and rate / mx
  double lb_p, lb_v;
  // options
  SimParams prm;
  const int8_t* spare_lut;
  uint64_t rng_seed;
  ModelW w;
  const double* draws;  // this task's precomputed predictor draws (nonces 1..draws_k) or null
  int draws_k;
  // per lane: the minimum of the event slots this lane owns, lazily rescanned
  int64_t lmin_t[32];
  uint64_t lmin_pk[32];
  int lmin_idx[32];
  bool lmin_valid[32];
};

// The engine state of the block's simulation (one warp per block).
__shared__ Ctx g_sim_ctx;
// reopt_and_apply's m x 5 effective estimated speeds (the search's rows)
__shared__ double g_sim_rows[35];

// Asynchronous STP (the ASYNC kernels): the engine warp posts every change of a job's STP term
// and the end of every processed event into this ring; a second warp of the block replays
// them in order and computes the sequential STP sums, the series and the integral off the
// engine's critical path. Single producer (engine lane 0), single consumer (helper).
struct StpMsg {
  unsigned long long head;  // job index (term change) | kind << 32
  unsigned long long bits;  // the new term's bits (change) or the event time in us (event)
};
enum : int32_t { kStpChange = 0, kStpEvent = 1, kStpEnd = 2 };

// The ring is a single-producer / single-consumer queue published by a block fence and volatile
// index stores -- an ordering compute-sanitizer racecheck does not follow (it reports the
// cross-warp accesses as hazards). MISO_SIM_STP_ATOMIC_RING=1 builds the same protocol with
// every ring access a shared-memory atomic (racecheck-clean, slower).
#ifndef MISO_SIM_STP_ATOMIC_RING
#define MISO_SIM_STP_ATOMIC_RING 0
#endif
__device__ __forceinline__ uint32_t ring_ld(uint32_t* p) {
  if constexpr (MISO_SIM_STP_ATOMIC_RING) return atomicAdd(p, 0u);
  else return *reinterpret_cast<volatile uint32_t*>(p);
}
__device__ __forceinline__ void ring_st(uint32_t* p, uint32_t v) {
  if constexpr (MISO_SIM_STP_ATOMIC_RING) atomicExch(p, v);
  else *reinterpret_cast<volatile uint32_t*>(p) = v;
}
__device__ __forceinline__ unsigned long long ring_ld(unsigned long long* p) {
  if constexpr (MISO_SIM_STP_ATOMIC_RING) return atomicAdd(p, 0ull);
  else return *p;
}
__device__ __forceinline__ void ring_st(unsigned long long* p, unsigned long long v) {
  if constexpr (MISO_SIM_STP_ATOMIC_RING) atomicExch(p, v);
  else *p = v;
}
constexpr int kStpRing = 128;
struct StpRing {
  uint32_t tail;  // messages posted (the engine warp writes it)
  uint32_t head;  // messages consumed (helper lane 0 writes)
  int quit;       // 1: the task was rejected before its event loop; 2: producer watchdog fired
  StpMsg msg[kStpRing];
};
__shared__ StpRing g_stp_ring;

// the engine and helper warps meet here twice: after the engine's init, and at the end. The two
// warps reach it from different code, so it is the non-aligned barrier (barrier.sync without
// .aligned: participating threads may execute different barrier instructions); each warp
// reconverges first.
__device__ __forceinline__ void stp_pair_barrier() {
  __syncwarp();
  asm volatile("barrier.sync 1, 64;" ::: "memory");
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Single-writer update of a warp-uniform Ctx field (shared memory): every lane evaluates the
// new value from the same state, the warp barrier orders all of those reads before lane 0's
// store, and the second barrier orders the store before any later read. Plain stores of a
// value that does not depend on the field itself stay all-lane (identical values).
#define CTX_SET(field, value)             \
  do {                                    \
    const auto ctx_v_ = (value);          \
    __syncwarp();                         \
    if (lane_id() == 0) (field) = ctx_v_; \
    __syncwarp();                         \
  } while (0)

// The pruned search's bound terms (Ctx::lb_*) are lane 0's alone: only lane 0 updates them and
// only lane 0 evaluates the stop test (broadcast by a shuffle), so their updates need no warp
// barriers.
#define LB_SET(field, value)                    \
  do {                                          \
    if (lane_id() == 0) (field) = (value);      \
  } while (0)

__device__ __forceinline__ double s_from_us(int64_t us) { return static_cast<double>(us) * 1e-6; }
__device__ __forceinline__ int64_t us_from_s(double s) {  // llround: half away from zero
  return static_cast<int64_t>(llround(s * 1e6));
}

__device__ __forceinline__ bool progressing(uint8_t ph) { return ph == kMps || ph == kRunning; }

__device__ __forceinline__ uint32_t pack_part(const uint8_t* p) {
  return p[0] | (p[1] << 4) | (p[2] << 8) | (p[3] << 12) | (p[4] << 16);
}

// Pruned best-static search (SimBatch::prune_bound). Under optsta a job only ever runs in a slot
// of the static partition, at that slot kind's effective true speed (start_running), so it can
// never run faster than prune_mx = the largest effective true speed over the partition's kinds
// (set once at init, kept in the job's est[0]: the estimates are unused under optsta, and pruned
// runs have no clones). From any moment it therefore needs at least remaining / prune_mx more
// seconds (migrations only add checkpoint pauses), and a job that has not started needs at least
// base / prune_mx (completions are scheduled llround(remaining / rate * 1e6) us ahead: rounded
// down with margin). A job no kind of the partition can run never completes (the run ends
// incomplete); its floor uses 1.0, which is still a valid bound.
__device__ __forceinline__ double prune_mx(const DJob& j) { return j.est[0]; }
__device__ __forceinline__ int64_t runtime_floor_us(const DJob& j) {
  const double us = j.base / prune_mx(j) * 1e6 * (1.0 - 1e-12) - 2.0;
  return us > 0.0 ? static_cast<int64_t>(us) : 0;
}

__device__ __forceinline__ double true_rate(const DJob& j, int k) {
  return effective_speed(j.truth[k], k, j.mem, j.qos);
}
__device__ __forceinline__ double est_rate(const DJob& j, int k) {
  return effective_speed(j.est[k], k, j.mem, j.qos);
}

// The lane holding the warp's minimum of a key given as N 32-bit words, most significant first
// (among equal keys the lowest lane): one 32-bit warp min-reduction per word, each stage only
// among the lanes still tied, stopping as soon as one lane is left -- a few redux.sync steps
// instead of a five-round shuffle tree over the whole key.
template <int N>
__device__ __forceinline__ int warp_argmin_words(const uint32_t (&w)[N]) {
  const unsigned full = 0xffffffffu;
  bool in = true;
  unsigned c = full;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t m = __reduce_min_sync(full, in ? w[k] : 0xffffffffu);
    in = in && w[k] == m;
    c = __ballot_sync(full, in);
    if (!(c & (c - 1))) break;  // warp-uniform
  }
  return __ffs(c) - 1;
}

// event keys: (t >= 0, pk) -- live events' keys are distinct, and event times rarely tie, so
// this is usually two stages
__device__ __forceinline__ int warp_argmin_key(int64_t t, uint64_t pk) {
  const uint32_t w[4] = {static_cast<uint32_t>(static_cast<uint64_t>(t) >> 32),
                         static_cast<uint32_t>(t), static_cast<uint32_t>(pk >> 32),
                         static_cast<uint32_t>(pk)};
  return warp_argmin_words(w);
}

__device__ __forceinline__ int lut_index(const uint8_t* k) {
  return (((k[0] * 7 + k[1]) * 7 + k[2]) * 7 + k[3]) * 7 + k[4];
}

// LOG: the event-log writer is compiled in (the parity runs that request a log); measured runs
// use the LOG = false instantiation, which carries no log calls at all. STP: the STP series and
// integral are tracked (SimParams::track_stp; the best-static search's JCT-only candidate runs
// use STP = false, which carries no STP bookkeeping).
template <int POL, bool PRUNE, bool LOG, bool STP, bool ASYNC = false>
struct Engine {

  static __device__ __forceinline__ void sync_jst(int ji, const DJob& j) {
    Ctx& c = g_sim_ctx;
    c.jst[ji] = static_cast<uint8_t>(j.phase | (j.slice << 3) | ((j.flags & 2) ? 64 : 0));
  }

  static __device__ __forceinline__ void fail(int code) {
    Ctx& c = g_sim_ctx;
    CTX_SET(c.status, c.status == 0 ? code : c.status);
  }

  // ---- event log (optional) -------------------------------------------------------------
  // (the record writer is one out-of-line copy: inlined at every call site it would multiply
  // the kernel's instruction footprint for a path that is off in measured runs)
  static __device__ __forceinline__ void log_rec(uint8_t kind, int gpu, int job, uint8_t x,
                                                 uint32_t a, uint32_t b, double v) {
    if constexpr (LOG) {
      if (g_sim_ctx.log) log_write(kind, gpu, job, x, a, b, v);
    }
  }
  static __device__ __noinline__ void log_write(uint8_t kind, int gpu, int job, uint8_t x,
                                                uint32_t a, uint32_t b, double v) {
    Ctx& c = g_sim_ctx;
    if (c.log_n < c.log_cap && lane_id() == 0) {
      LogRec r;
      r.t = c.now;
      r.kind = kind;
      r.x = x;
      r.gpu = static_cast<uint16_t>(gpu < 0 ? 0xFFFF : gpu);
      r.job = job;
      r.a = a;
      r.b = b;
      r.v = v;
      c.log[c.log_n] = r;
    }
    __syncwarp();
    CTX_SET(c.log_n, c.log_n + 1);
  }


  // ---- event slots -----------------------------------------------------------------------
  static __device__ __forceinline__ void push_event(int slot, int64_t t, uint32_t prio,
                                             uint32_t kind) {
    Ctx& c = g_sim_ctx;
    Slot s;
    s.t = t;
    s.pk = (static_cast<uint64_t>(prio) << 62) | (c.seq << 3) | kind;
    CTX_SET(c.seq, c.seq + 1);
    c.slots[slot] = s;
    if (static_cast<unsigned>(slot - (lane_id() * c.chunk)) < static_cast<unsigned>(c.chunk)) {  // owner lane
      // keeps its minimum current
      if (c.lmin_idx[lane_id()] == slot) c.lmin_valid[lane_id()] = false;
      else if (c.lmin_valid[lane_id()] && (t < c.lmin_t[lane_id()] || (t == c.lmin_t[lane_id()] && s.pk < c.lmin_pk[lane_id()]))) {
        c.lmin_t[lane_id()] = t;
        c.lmin_pk[lane_id()] = s.pk;
        c.lmin_idx[lane_id()] = slot;
      }
    }
  }

  static __device__ __forceinline__ void clear_slot(int slot) {
    Ctx& c = g_sim_ctx;
    c.slots[slot].t = kNoEvent;
    if (c.lmin_idx[lane_id()] == slot) c.lmin_valid[lane_id()] = false;  // a lane's lmin_idx lies in its own chunk
  }

  // Next event = minimum live (t, prio, seq) key. Lane l owns the contiguous slot chunk
  // [l*chunk, (l+1)*chunk) and keeps its minimum in registers (updated on push, invalidated when
  // that slot is cleared or overwritten). Invalid chunks are rescanned by the whole warp (one
  // coalesced load per lane + a warp argmin); the event is then one warp argmin over the 32
  // lane minima.
  static __device__ int next_event(Slot* out) {
    Ctx& c = g_sim_ctx;
    const int n = c.J + c.G;
    const int lane = lane_id();
    unsigned inval = __ballot_sync(0xffffffffu, !c.lmin_valid[lane]);
    while (inval) {
      const int owner = __ffs(inval) - 1;
      inval &= inval - 1;
      const int lo = owner * c.chunk;
      int hi = lo + c.chunk;
      if (hi > n) hi = n;
      int64_t bt = kNoEvent;
      uint64_t bk = ~0ull;
      int bi = -1;
      for (int i = lo + lane; i < hi; i += 32) {
        const Slot s = c.slots[i];
        if (s.t < bt || (s.t == bt && s.pk < bk)) {
          bt = s.t;
          bk = s.pk;
          bi = i;
        }
      }
      if (lane == warp_argmin_key(bt, bk)) {  // the chunk's minimum becomes the owner's
        c.lmin_t[owner] = bt;
        c.lmin_pk[owner] = bk;
        c.lmin_idx[owner] = bi;
        c.lmin_valid[owner] = true;
      }
    }
    __syncwarp();
    const int w = warp_argmin_key(c.lmin_t[lane], c.lmin_pk[lane]);
    const int64_t bt = c.lmin_t[w];
    out->t = bt;
    out->pk = c.lmin_pk[w];
    return bt == kNoEvent ? -1 : c.lmin_idx[w];
  }

  // ---- job state ---------------------------------------------------------------------------
  // sim.hpp:319-329
  static __device__ void advance_job(DJob& j) {
    Ctx& c = g_sim_ctx;
    const int64_t dt = c.now - j.last_update_us;
    j.last_update_us = c.now;
    if (dt <= 0 || (j.flags & kDone)) return;
    j.acc[j.phase] += dt;
    if (progressing(j.phase)) {
      const double w = j.rate * s_from_us(dt);
      j.remaining -= w;
      j.consumed += w;
    }
  }


  // sim.hpp:333-343 (+ slot invalidation: every epoch bump retires the job's pending event)
  static __device__ void set_phase(int ji, uint8_t phase, double rate) {
    Ctx& c = g_sim_ctx;
    DJob& j = c.jobs[ji];
    advance_job(j);
    // the job's current STP term (== rate_eff[ji], which every term change keeps in step)
    const double old_term = (progressing(j.phase) && !(j.flags & kDone)) ? j.rate : 0.0;
    (void)old_term;
    if constexpr (PRUNE) {
    if (c.prune && j.first_progress_us >= 0 && !(j.flags & kDone)) {  // retire the old-rate term
      LB_SET(c.lb_p, c.lb_p - (j.lbp));
      LB_SET(c.lb_v, c.lb_v - (j.rate / prune_mx(j)));
    }
    }
    j.phase = phase;
    j.rate = progressing(phase) ? rate : 0.0;
    ++j.epoch;
    clear_slot(ji);
    if (progressing(phase)) {
      j.flags |= kRunState;
      if (j.first_progress_us < 0) j.first_progress_us = c.now;
      if (c.first_progress < 0) CTX_SET(c.first_progress, c.now);
    }
    // the STP window's sums only need redoing from ji if the job's term actually changed
    const double re = (progressing(phase) && !(j.flags & kDone)) ? j.rate : 0.0;
    if constexpr (ASYNC) {  // the helper warp owns rate_eff: post the change
      if (__double_as_longlong(re) != __double_as_longlong(old_term)) stp_post(kStpChange, ji, __double_as_longlong(re));
    } else if (__double_as_longlong(re) != __double_as_longlong(c.rate_eff[ji])) {
      c.rate_eff[ji] = re;
      if (re != 0.0 && ji >= c.stp_hi) {  // the summed range grows: its new blocks need sums
        if constexpr (STP) {
          const int h = c.stp_hi;
          CTX_SET(c.stp_cmin, h < c.stp_cmin ? h : c.stp_cmin);
        }
        CTX_SET(c.stp_hi, ji + 1);
      }
      if constexpr (STP) {
        c.stp_dirty = true;
        CTX_SET(c.stp_cmin, ji < c.stp_cmin ? ji : c.stp_cmin);
      }
    }
    sync_jst(ji, j);
    if constexpr (PRUNE) {
    if (c.prune && j.first_progress_us >= 0 && !(j.flags & kDone)) {  // remaining / mx, from now
      const double mx = prune_mx(j);
      j.lbp = (j.remaining + j.rate * s_from_us(c.now)) / mx;
      LB_SET(c.lb_p, c.lb_p + (j.lbp));
      LB_SET(c.lb_v, c.lb_v + (j.rate / mx));
    }
    }
  }

  // sim.hpp:345-351
  static __device__ void schedule_completion(int ji) {
    Ctx& c = g_sim_ctx;
    DJob& j = c.jobs[ji];
    if ((j.flags & kDone) || !(j.rate > 0)) return;
    const double dt_s = (j.remaining > 0.0 ? j.remaining : 0.0) / j.rate;  // std::max(0.0, r)
    int64_t dt = us_from_s(dt_s);
    if (dt < 0) dt = 0;
    push_event(ji, c.now + dt, 0, kEvCompletion);
  }

  // sim.hpp:353-361: s = sum over jobs in index order of rate (progressing, not done). Only
  // jobs in [stp_lo, stp_hi) can have a nonzero term (below stp_lo every job is done; at and
  // above stp_hi none has progressed yet -- under FCFS admission the queued tail of the arrived
  // jobs); rate_eff holds 0.0 for the others, and s + 0.0 == s for the non-negative partial
  // sums, so the sequential FP64 sum over that window is bit-identical to the reference's loop
  // over all jobs. Partial sums are cached per index and
  // the chain restarts at the smallest index changed since the previous refresh.
  static __device__ void refresh_stp() {
    Ctx& c = g_sim_ctx;
    if constexpr (!STP || ASYNC) return;
    if (!c.stp_dirty) return;
    c.stp_dirty = false;
    const int lo = c.stp_lo, hi = c.stp_hi;
    const double s = stp_sum(c.stp_cmin, lo, hi);
    c.stp_cmin = INT32_MAX;
    if (s != c.stp_cur) {
      c.stp_cur = s;
      if (c.stp_series && c.stp_points < c.stp_cap && lane_id() == 0) {
        c.stp_series[2 * c.stp_points] = s_from_us(c.now);
        c.stp_series[2 * c.stp_points + 1] = s;
      }
      __syncwarp();
      CTX_SET(c.stp_points, c.stp_points + 1);
    }
  }

  // The window's sequential sum after changes at indices >= cmin: rate_eff[lo, hi) (zeros
  // outside), restarting from the cached partial sum before cmin's block. (Called by all lanes
  // of one warp; lane 0 updates the cache.)
  static __device__ __forceinline__ double stp_sum(int cmin, int lo, int hi) {
    Ctx& c = g_sim_ctx;
    const double* r = c.rate_eff;
    double* P = c.stp_prefix;  // P[q]: the sum through index 8q + 7, cached at block ends
    int i0 = cmin > lo ? cmin : lo;
    if (i0 > hi) i0 = hi;  // changes at not-yet-arrived indices: the window's sum is unchanged
    // restart at i0's 8-aligned block from the cached sum before it: the block's terms below i0
    // are unchanged, so re-adding them reproduces the same partial sums (and jobs below lo are
    // done, contributing +0.0, so a start below lo is exact too)
    int i = i0 & ~7;
    double s = (i > 0 && i - 1 >= lo) ? P[(i >> 3) - 1] : 0.0;
    // 64-byte aligned blocks of eight terms, four 16-byte loads each, loaded one block ahead of
    // the additions (the chain of dependent adds, not the loads, sets the pace); the partial
    // last block is loaded whole (rate_eff is padded by 32 entries) and added term by term
    const double2* r2 = reinterpret_cast<const double2*>(r + i);
    const bool lane0 = lane_id() == 0;
    double2 a01 = r2[0], a23 = r2[1], a45 = r2[2], a67 = r2[3];
    double2 b01, b23, b45, b67;
#define MISO_STP_ADD8(x01, x23, x45, x67) \
    s = s + x01.x;                        \
    s = s + x01.y;                        \
    s = s + x23.x;                        \
    s = s + x23.y;                        \
    s = s + x45.x;                        \
    s = s + x45.y;                        \
    s = s + x67.x;                        \
    s = s + x67.y
    for (; i + 16 <= hi; i += 16) {  // two blocks per trip: no register copies between them
      b01 = r2[4], b23 = r2[5], b45 = r2[6], b67 = r2[7];
      MISO_STP_ADD8(a01, a23, a45, a67);
      if (lane0) P[i >> 3] = s;
      r2 += 8;
      a01 = r2[0], a23 = r2[1], a45 = r2[2], a67 = r2[3];
      MISO_STP_ADD8(b01, b23, b45, b67);
      if (lane0) P[(i >> 3) + 1] = s;
    }
    if (i + 8 <= hi) {
      b01 = r2[4], b23 = r2[5], b45 = r2[6], b67 = r2[7];
      MISO_STP_ADD8(a01, a23, a45, a67);
      if (lane0) P[i >> 3] = s;
      i += 8;
      a01 = b01, a23 = b23, a45 = b45, a67 = b67;
    }
#undef MISO_STP_ADD8
    const double t[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
#pragma unroll
    for (int k = 0; k < 7; ++k)
      if (i + k < hi) s = s + t[k];
    __syncwarp();
    return hi <= lo ? 0.0 : s;
  }

  // ---- asynchronous STP (ASYNC kernels) ----------------------------------------------------
  // Engine side: one message into the ring, waiting only if the helper is a whole ring behind.
  static __device__ __forceinline__ void stp_post(int32_t kind, int32_t idx, int64_t bits) {
    // every lane of the converged engine warp executes the same stores (identical values at the
    // same addresses): no divergent branch, no reconvergence (the atomic build: lane 0 alone)
    if (!MISO_SIM_STP_ATOMIC_RING || lane_id() == 0) {
      StpRing& R = g_stp_ring;
      const uint32_t t = ring_ld(&R.tail);
      if (t - ring_ld(&R.head) >= static_cast<uint32_t>(kStpRing)) {  // full: the helper is behind
        uint32_t spins = 0;
        while (t - ring_ld(&R.head) >= static_cast<uint32_t>(kStpRing)) {
          __nanosleep(64);
          if (++spins > (1u << 26)) {  // watchdog (never expected): flag it, do not hang
            R.quit = 2;
            break;
          }
        }
      }
      StpMsg& m = R.msg[t % kStpRing];
      ring_st(&m.head, static_cast<unsigned long long>(static_cast<uint32_t>(idx)) |
                           (static_cast<unsigned long long>(static_cast<uint32_t>(kind)) << 32));
      ring_st(&m.bits, static_cast<unsigned long long>(bits));
      __threadfence_block();
      ring_st(&R.tail, t + 1);
    }
    if (MISO_SIM_STP_ATOMIC_RING) __syncwarp();
  }

  // Helper warp: replays the engine's messages in order -- term changes into rate_eff, and at
  // each event's end the reference's integral step (with the sum after the previous event) and
  // then refresh_stp (sim.hpp:227-232, 353-361), exactly the synchronous path's operations.
  static __device__ void stp_helper() {
    Ctx& c = g_sim_ctx;
    StpRing& R = g_stp_ring;
    const int lane = lane_id();
    int hi = 0, cmin = INT32_MAX;
    bool dirty = false;
    double cur = 0.0, integ = 0.0;
    int64_t last = 0, pts = 0;
    uint32_t h = 0;
    uint32_t idle = 0;
    for (;;) {
      const uint32_t t = __shfl_sync(0xffffffffu, lane == 0 ? ring_ld(&R.tail) : 0u, 0);  // one view
      if (t == h) {
        __nanosleep(32);
        if (++idle > (1u << 28)) {  // watchdog (never expected): the engine stopped posting
          if (lane == 0) R.quit = 2;  // the engine reports the run as failed
          __syncwarp();
          return;
        }
        continue;
      }
      idle = 0;
      __threadfence_block();
      for (; h != t; ++h) {
        StpMsg& slot = R.msg[h % kStpRing];
        const unsigned long long mh = ring_ld(&slot.head);
        const int64_t mbits = static_cast<int64_t>(ring_ld(&slot.bits));
        const int32_t kind = static_cast<int32_t>(mh >> 32);
        if (kind == kStpChange) {
          const int ji = static_cast<int32_t>(mh & 0xffffffffu);
          if (mbits != __double_as_longlong(c.rate_eff[ji])) {
            if (lane == 0) c.rate_eff[ji] = __longlong_as_double(mbits);
            __syncwarp();
            if (mbits != 0 && ji >= hi) {  // the summed range grows: its new blocks need sums
              cmin = hi < cmin ? hi : cmin;
              hi = ji + 1;
            }
            cmin = ji < cmin ? ji : cmin;
            dirty = true;
          }
        } else if (kind == kStpEvent) {
          const int64_t te = mbits;
          integ = integ + cur * s_from_us(te - last);
          last = te;
          if (dirty) {
            dirty = false;
            const double sum = stp_sum(cmin, 0, hi);
            cmin = INT32_MAX;
            if (sum != cur) {
              cur = sum;
              if (c.stp_series && pts < c.stp_cap && lane == 0) {
                c.stp_series[2 * pts] = s_from_us(te);
                c.stp_series[2 * pts + 1] = sum;
              }
              ++pts;
            }
          }
        } else {  // kStpEnd
          if (lane == 0) {
            c.stp_integral = integ;
            c.stp_points = pts;
            c.stp_cur = cur;
          }
          __syncwarp();
          return;
        }
      }
      __syncwarp();
      if (lane == 0) ring_st(&R.head, h);
    }
  }

  // the helper warp's whole life: wait for the engine's init, replay, meet the engine at the end
  static __device__ void stp_helper_main() {
    stp_pair_barrier();
    if (g_stp_ring.quit == 1) return;  // the task was rejected: no event loop
    stp_helper();
    stp_pair_barrier();
  }

  // ---- queue (std::set ordered by (arrival_us, entry_seq == idx)) -------------------------
  static __device__ void enqueue(int ji) {
    Ctx& c = g_sim_ctx;
    const int64_t a = c.arr_us[ji];  // (dense copy of arrival_us)
    int pos = c.qtail;
    while (pos > c.qhead) {  // sorted insert; arrivals append at the tail
      const int prev = c.queue[pos - 1];
      const int64_t pa = c.arr_us[prev];
      if (pa < a || (pa == a && prev < ji)) break;
      __syncwarp();
      c.queue[pos] = prev;
      __syncwarp();
      --pos;
    }
    c.queue[pos] = ji;
    __syncwarp();
    CTX_SET(c.qtail, c.qtail + 1);
  }

  // ---- GPU roster helpers -----------------------------------------------------------------

  // miso/oracle: place_dynamic's view of GPU g, one byte per GPU so the placement scan reads a
  // few dense sectors instead of one per GPU record: 0x0F if the GPU takes no job (mode other
  // than idle/MIG, or 7 jobs), else (allow + 1) << 4 | nroster, where allow is the largest
  // min-kind it accepts (any when empty, its spare slice otherwise; a spare of -1 accepts none).
  static __device__ __forceinline__ void sync_place(const DGpu& g) {
    if constexpr (POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE) {
      Ctx& c = g_sim_ctx;
      uint8_t v = 0x0F;
      if ((g.mode == kGpuIdle || g.mode == kGpuMig) && g.nroster < 7)
        v = static_cast<uint8_t>(((g.nroster == 0 ? 5 : g.spare + 1) << 4) | g.nroster);
      c.gplace[&g - c.gpus] = v;
    }
  }

  static __device__ void roster_push(DGpu& g, int ji) {
    Ctx& c = g_sim_ctx;
    g.roster[g.nroster] = ji;
    __syncwarp();
    ++g.nroster;
    ++g.kind_cnt[c.jobs[ji].min_kind];
    g.spare = g.nroster >= 7 ? -1 : c.spare_lut[lut_index(g.kind_cnt)];
    sync_place(g);
  }

  static __device__ void roster_erase(DGpu& g, int ji) {
    Ctx& c = g_sim_ctx;
    const int ln = lane_id();  // the job's roster position, one lane per entry
    const unsigned hit = __ballot_sync(0xffffffffu, ln < g.nroster && g.roster[ln < 7 ? ln : 0] == ji);
    const int i = hit ? __ffs(hit) - 1 : g.nroster;
    {  // close the gap: lane k moves entry k + 1 down (all reads before any write)
      const bool mv = ln >= i && ln + 1 < g.nroster;
      const int v = mv ? g.roster[ln + 1] : 0;
      __syncwarp();
      if (mv) g.roster[ln] = v;
      __syncwarp();
    }
    --g.nroster;
    --g.kind_cnt[c.jobs[ji].min_kind];
    g.spare = g.nroster >= 7 ? -1 : c.spare_lut[lut_index(g.kind_cnt)];
    sync_place(g);
  }

  // Lane-parallel roster reads (one lane per roster entry, one load round trip instead of a
  // chain of roster -> job loads per entry): bit i = the predicate for roster entry i.
  static __device__ __forceinline__ unsigned roster_flag_mask(const DGpu& g, uint8_t flag) {
    const int ln = lane_id();
    const bool p = ln < g.nroster && (g_sim_ctx.jobs[g.roster[ln < 7 ? ln : 0]].flags & flag);
    return __ballot_sync(0xffffffffu, p);
  }
  // entry i's job already runs on the planned slice (begin_reconfig / apply_assignment skip it)
  static __device__ __forceinline__ unsigned roster_on_plan_mask(const DGpu& g) {
    const int ln = lane_id();
    bool p = false;
    if (ln < g.nroster) {
      const DJob& j = g_sim_ctx.jobs[g.roster[ln]];
      p = j.phase == kRunning && j.slice == g.plan_slice[ln];
    }
    return __ballot_sync(0xffffffffu, p);
  }

  // ---- forward declarations of the mutually recursive steps ---------------------------------

  // sim.hpp:480-489
  static __device__ void start_running(int ji, int s) {
    Ctx& c = g_sim_ctx;
    DJob& j = c.jobs[ji];
    if constexpr (PRUNE) {
    if (c.prune && j.first_progress_us < 0) LB_SET(c.lb_unstarted, c.lb_unstarted - runtime_floor_us(j));
    }
    const double r = c.efftruth[size_t(s) * c.J + ji];  // == true_rate(j, s)
    if (c.prm.check_invariants && !(r > 0)) fail(MISO_B200_SIM_INFEASIBLE_SLICE);
    j.slice = static_cast<uint8_t>(s);
    set_phase(ji, kRunning, r);  // also syncs jst
    schedule_completion(ji);
    log_rec(kLogStart, j.gpu, ji, static_cast<uint8_t>(s), 0, 0, r);
  }

  // sim.hpp:432-455: a multi-instance job's clones are appended at its first admission (nopart,
  // optsta) or estimate caching (miso, oracle): copies of the profile ("parent#k"), the parent's
  // arrival as FCFS position and JCT baseline, the parent's estimates, queued in FCFS order
  // (arrival_us, index == entry_seq). The STP window grows to the clone's index; jobs in between
  // that have not arrived yet contribute +0.0 (exact).
  // (the common single-instance case is decided inline; the spawning itself is out of line)
  static __device__ __forceinline__ void spawn_instances(int pi) {
    const DJob& par = g_sim_ctx.jobs[pi];
    if (!(par.flags & kSpawned) && par.inst > 1) spawn_clones(pi);
  }
  static __device__ __noinline__ void spawn_clones(int pi) {
    Ctx& c = g_sim_ctx;
    DJob& par = c.jobs[pi];
    par.flags |= kSpawned;
    for (int k = 1; k < par.inst; ++k) {
      const int ci = c.J_used;
      if (ci >= c.J) {  // capacity is the trace's instance total; cannot happen
        fail(MISO_B200_SIM_INVARIANT);
        return;
      }
      DJob& j = c.jobs[ci];
      j.base = par.base;
      j.remaining = par.base;
      j.consumed = 0;
      j.rate = 0;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        j.truth[q] = par.truth[q];
        j.est[q] = par.est[q];
        j.acc[q] = 0;
      }
      j.arrival_us = par.arrival_us;
      j.last_update_us = par.arrival_us;
      j.first_progress_us = -1;
      j.completion_us = -1;
      j.epoch = 0;
      j.gpu = -1;
      j.phase = kQueued;
      j.slice = 4;
      j.mem = par.mem;
      j.min_kind = par.min_kind;
      j.qos = par.qos;
      j.flags = static_cast<uint8_t>((par.flags & kHasEst) | kSpawned);
      j.slot = -1;
      j.inst = 1;
      j.clone_k = static_cast<int16_t>(k);
      j.parent = pi;
#pragma unroll
      for (int q = 0; q < 5; ++q) c.efftruth[size_t(q) * c.J + ci] = c.efftruth[size_t(q) * c.J + pi];
      c.arr_us[ci] = par.arrival_us;
      __syncwarp();
      c.J_used = ci + 1;
      sync_jst(ci, j);
      if (ci + 1 > c.n_arrived) c.n_arrived = ci + 1;
      log_rec(kLogSpawn, -1, ci, 0, static_cast<uint32_t>(pi), 0, 0);
      enqueue(ci);
    }
  }

  // sim.hpp:457-461
  static __device__ void cache_estimates(int ji, const double* est) {
    Ctx& c = g_sim_ctx;
    DJob& j = c.jobs[ji];
#pragma unroll
    for (int k = 0; k < 5; ++k) j.est[k] = est[k];
    j.flags |= kHasEst;
    spawn_instances(ji);
  }

  // sim.hpp:670-680 with simulate_mps_rates / interp_speed (profiles.hpp:391-431)
  static __device__ void rate_roster_mps(int gi, int level) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const int n = g.nroster;
    double share = static_cast<double>(level);
    const double eq = 100.0 / static_cast<double>(n);
    if (eq < share) share = eq;  // std::min(level, 100/n)
    const double gpc = clampd(share / 100.0 * 7.0, 1.0, 7.0);
    double my_rate = 0.0;  // lane i: roster entry i's MPS rate (the loads in parallel)
    if (lane_id() < n) {
      const DJob& j = c.jobs[g.roster[lane_id()]];
      double sp;
      if (gpc <= 1.0) {
        sp = j.truth[0];
      } else if (gpc >= 7.0) {
        sp = j.truth[4];
      } else {
        const double knots[5] = {1, 2, 3, 4, 7};
        int k = 1;
        while (!(gpc <= knots[k])) ++k;
        const double wgt = (gpc - knots[k - 1]) / (knots[k] - knots[k - 1]);
        sp = j.truth[k - 1] + wgt * (j.truth[k] - j.truth[k - 1]);
      }
      my_rate = clampd(c.prm.interference * sp, kSpeedFloor, 1.0);
    }
    __syncwarp();
    for (int i = 0; i < n; ++i) {
      const int ji = g.roster[i];
      set_phase(ji, kMps, __shfl_sync(0xffffffffu, my_rate, i));
      schedule_completion(ji);
    }
  }

  // sim.hpp:660-666
  static __device__ void start_mps_window(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const int level = g.mps_level == 0 ? 100 : (g.mps_level == 1 ? 50 : 14);  // kMpsLevels
    rate_roster_mps(gi, level);
    ++g.epoch;
    push_event(c.J + gi, c.now + c.prm.window_us, 2, kEvMpsEnd);
    log_rec(kLogMpsWindow, gi, -1, 0, static_cast<uint32_t>(level), 0, 0);
  }

  // sim.hpp:654-658
  static __device__ void begin_mps_windows(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    g.mps_level = 0;
    log_rec(kLogMpsStart, gi, -1, 0, g.nroster, 0, 0);
    start_mps_window(gi);
  }

  // sim.hpp:625-652
  static __device__ __noinline__ void start_profiling_session(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    g.mode = kGpuMps;
    sync_place(g);
#pragma unroll
    for (int k = 0; k < 5; ++k) g.part[k] = 0;
    g.objective = 0;
    if (c.prm.window_us == 0) {
      finish_profiling(gi);
      return;
    }
    CTX_SET(c.mps_sessions, c.mps_sessions + 1);
    const unsigned ran = roster_flag_mask(g, kRunState);
    const bool need_ckpt = c.prm.ckpt_us > 0 && ran != 0;
    if (need_ckpt) {
      for (int i = 0; i < g.nroster; ++i) {
        const int ji = g.roster[i];
        set_phase(ji, ((ran >> i) & 1u) ? kCkpt : kQueued, 0.0);
      }
      ++g.epoch;
      push_event(c.J + gi, c.now + c.prm.ckpt_us, 2, kEvCkptDone);
      log_rec(kLogCkptStart, gi, -1, 0, g.nroster, 0, 0);
    } else {
      begin_mps_windows(gi);
    }
  }

  // sim.hpp:691-714. Noisy mode: lane c predicts roster column c (predict_mig_speeds with call
  // nonce ++predictor_nonce_, then extrapolate_small_slices); columns are exchanged by shuffles.
  static __device__ __noinline__ void finish_profiling(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const int n = g.nroster;
    if (!c.prm.noisy) {
      for (int i = 0; i < n; ++i) {
        const int ji = g.roster[i];
        cache_estimates(ji, c.jobs[ji].truth);
      }
    } else {
      const uint64_t nonce = c.nonce + 1;
      CTX_SET(c.nonce, nonce);
      double e[5] = {0, 0, 0, 0, 0};
      const int ln = lane_id();
      if (ln < n) {
        const DJob& j = c.jobs[g.roster[ln]];
        if (c.draws && nonce <= static_cast<uint64_t>(c.draws_k) && c.prm.target_mae > 0.0) {
          // the call's draws were computed ahead (sim_draws_kernel): same bits, no seeding here
          const double* d = c.draws + ((nonce - 1) * 7 + ln) * 2;
          predict_column_drawn(j.truth[4], j.truth[3], j.truth[2], unpack_draw(d[0]),
                               unpack_draw(d[1]), c.prm.target_mae, c.w, e);
        } else {
          predict_column(j.truth[4], j.truth[3], j.truth[2], ln, c.rng_seed, nonce, true,
                         c.prm.target_mae, c.w, e);
        }
      }
      __syncwarp();  // reconverge
      // cache_estimates for every column: lane i stores its own column's estimates (no column
      // exchange), then the spawns run in roster order (they read only their own job's row)
      if (ln < n) {
        DJob& j = c.jobs[g.roster[ln]];
#pragma unroll
        for (int k = 0; k < 5; ++k) j.est[k] = e[k];
        j.flags |= kHasEst;
      }
      __syncwarp();
      for (int i = 0; i < n; ++i) spawn_instances(g.roster[i]);
    }
    reopt_and_apply(gi, true);
  }

  // sim.hpp:765-794
  static __device__ void apply_assignment(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    if (!g.plan_valid) {
      fail(MISO_B200_SIM_INVARIANT);
      return;
    }
    g.plan_valid = 0;
    if (g.plan_n != g.nroster) {
      fail(MISO_B200_SIM_INVARIANT);
      return;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) g.part[k] = g.plan_part[k];
    g.objective = g.plan_obj;
    g.mode = kGpuMig;
    sync_place(g);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) cnt += g.plan_part[k];
    if (c.prm.check_invariants && cnt != g.nroster) fail(MISO_B200_SIM_INVARIANT);
    for (int i = 0; i < g.nroster; ++i)
      if (g.plan_job[i] != g.roster[i]) fail(MISO_B200_SIM_INVARIANT);
    log_rec(kLogPartition, gi, -1, static_cast<uint8_t>(g.nroster), pack_part(g.part), 0, 0);
    for (int i = 0; i < g.nroster; ++i)
      log_rec(kLogAssign, gi, g.roster[i], g.plan_slice[i], 0, 0, 0);
    const unsigned keep = roster_on_plan_mask(g);
    for (int i = 0; i < g.nroster; ++i) {
      if ((keep >> i) & 1u) continue;
      start_running(g.roster[i], g.plan_slice[i]);
    }
  }

  // sim.hpp:739-763
  static __device__ void begin_reconfig(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const unsigned all = (1u << g.nroster) - 1u;
    const unsigned move = ~roster_on_plan_mask(g) & all;  // entries whose job changes slice
    const unsigned ran = roster_flag_mask(g, kRunState);
    const bool any = move != 0, restart = (move & ran) != 0;
    const int64_t pause = c.prm.reconfig_us + (restart ? c.prm.ckpt_us : 0);
    g.plan_valid = 1;
    if (!any || pause == 0) {
      apply_assignment(gi);
      return;
    }
    g.mode = kGpuReconfig;
    sync_place(g);
    for (int i = 0; i < g.nroster; ++i) {
      if (!((move >> i) & 1u)) continue;
      set_phase(g.roster[i], ((ran >> i) & 1u) ? kCkpt : kQueued, 0.0);
    }
    ++g.epoch;
    push_event(c.J + gi, c.now + pause, 2, kEvReconfigDone);
    log_rec(kLogReconfigStart, gi, -1, 0, static_cast<uint32_t>(pause & 0xFFFFFFFF),
            static_cast<uint32_t>(pause >> 32), 0);
  }

  // sim.hpp:716-733
  static __device__ __noinline__ void reopt_and_apply(int gi, bool force) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const int m = g.nroster;
    double* rows = g_sim_rows;  // effective estimated speeds, one entry per lane
    for (int q = lane_id(); q < 5 * m && q < 35; q += 32) {
      const int i = q / 5;
      rows[q] = est_rate(c.jobs[g.roster[i]], q - 5 * i);
    }
    __syncwarp();
    double obj = 0.0;
    const uint8_t cand = warp_search(rows, m, c.prm.en0, c.prm.en1, kCandPlaceD, &obj);
    if (cand >= kNumCands) {  // nullopt (or m out of range): SimInvariantError
      __syncwarp();
      fail(MISO_B200_SIM_NO_PARTITION);
      return;
    }
    if (!force && !(obj > g.objective + 1e-12)) return;
    CTX_SET(c.repartitions, c.repartitions + 1);
    g.plan_obj = obj;
    g.plan_n = static_cast<uint8_t>(m);
#pragma unroll
    for (int k = 0; k < 5; ++k) g.plan_part[k] = 0;
    for (int i = 0; i < m; ++i) {
      const int s = kCandPlaceD[cand][i];
      g.plan_slice[i] = static_cast<uint8_t>(s);
      g.plan_job[i] = g.roster[i];
      g.plan_speed[i] = rows[i * 5 + s];
      ++g.plan_part[s];
    }
    __syncwarp();  // (rows are rewritten by the next search)
    begin_reconfig(gi);
  }

  // sim.hpp:612-623
  static __device__ __noinline__ void settle_admissions(int gi) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    if constexpr (POL == MISO_B200_POLICY_ORACLE)
      for (int i = 0; i < g.nroster; ++i) {
        const int ji = g.roster[i];
        if (!(c.jobs[ji].flags & kHasEst)) cache_estimates(ji, c.jobs[ji].truth);
      }
    const bool all_est = roster_flag_mask(g, kHasEst) == (1u << g.nroster) - 1u;
    if (all_est) reopt_and_apply(gi, true);
    else start_profiling_session(gi);
  }

  // sim.hpp:581-607: least-loaded GPU whose spare slice covers the job's minimum (ties: id)
  static __device__ int place_dynamic(int ji) {
    Ctx& c = g_sim_ctx;
    const int need = c.jobs[ji].min_kind;
    int best = -1, best_cnt = 8;
    for (int gi = lane_id(); gi < c.G; gi += 32) {
      const int v = c.gplace[gi];  // (allow + 1) << 4 | nroster, see sync_place
      if ((v >> 4) <= need) continue;
      if ((v & 15) < best_cnt) {
        best = gi;
        best_cnt = v & 15;
      }
    }
    if (!__ballot_sync(0xffffffffu, best >= 0)) return -1;
    {  // the least-loaded candidate, ties to the lowest GPU id
      const uint32_t key[2] = {best >= 0 ? static_cast<uint32_t>(best_cnt) : 0xffffffffu,
                               static_cast<uint32_t>(best)};
      best = __shfl_sync(0xffffffffu, best, warp_argmin_words(key));
    }
    CTX_SET(c.qhead, c.qhead + 1);  // pop_queue: the placed job is always the queue head
    DGpu& g = c.gpus[best];
    roster_push(g, ji);
    c.jobs[ji].gpu = static_cast<int16_t>(best);
    log_rec(kLogAdmit, best, ji, 0, 0, 0, 0);
    return best;
  }

  // optsta free-slot bookkeeping: per GPU and kind a free count, per kind a GPU bitmask.
  static __device__ __forceinline__ void occupy_slot(int gi, int i, int ji) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const int k = g.slot_kind[i];
    g.slot_job[i] = ji;
    if (--g.fcnt[k] == 0) {
      uint32_t* w = c.freemask + k * c.W + (gi >> 5);
      const uint32_t v = *w & ~(1u << (gi & 31));
      __syncwarp();
      *w = v;
    }
  }

  static __device__ __forceinline__ void free_slot(int gi, int i) {
    Ctx& c = g_sim_ctx;
    CTX_SET(c.cap_gen, c.cap_gen + 1);
    DGpu& g = c.gpus[gi];
    const int k = g.slot_kind[i];
    g.slot_job[i] = -1;
    if (g.fcnt[k]++ == 0) {
      uint32_t* w = c.freemask + k * c.W + (gi >> 5);
      const uint32_t v = *w | (1u << (gi & 31));
      __syncwarp();
      *w = v;
    }
  }

  // sim.hpp:495-520: the largest free slot the job can use, ties to the first (gpu, slot). Kinds
  // have distinct GPC counts, so this is: the largest feasible kind with a free slot anywhere,
  // on the lowest-numbered GPU having one, at that GPU's first free slot of the kind.
  static __device__ bool admit_optsta(int ji) {
    Ctx& c = g_sim_ctx;
    if (ji == c.fail_job && c.fail_gen == c.cap_gen) return false;  // nothing freed since
    const int lane = lane_id();
    // the job's feasible kinds (true_rate > 0), one lane per kind: one load round trip
    const bool fk = lane < 5 && c.efftruth[size_t(lane < 5 ? lane : 0) * c.J + ji] > 0;
    const unsigned feas = __ballot_sync(0xffffffffu, fk);
    int bg = -1, bk = -1;
    if (5 * c.W <= 32) {  // every kind's free-GPU words in one load (lane = k * W + word)
      const uint32_t word = lane < 5 * c.W ? c.freemask[lane] : 0u;
      const unsigned nz = __ballot_sync(0xffffffffu, word != 0);
      const unsigned grp = (1u << c.W) - 1u;
      for (int k = 4; k >= 0; --k) {
        const unsigned g = (nz >> (k * c.W)) & grp;
        if (!((feas >> k) & 1u) || !g) continue;
        const int l = k * c.W + __ffs(g) - 1;
        const uint32_t wv = __shfl_sync(0xffffffffu, word, l);
        bg = ((l - k * c.W) << 5) + __ffs(wv) - 1;
        bk = k;
        break;
      }
    } else {
      for (int k = 4; k >= 0 && bg < 0; --k) {
        if (!((feas >> k) & 1u)) continue;
        for (int w0 = 0; w0 < c.W && bg < 0; w0 += 32) {
          const int wi = w0 + lane;
          const uint32_t word = wi < c.W ? c.freemask[k * c.W + wi] : 0u;
          const unsigned nz = __ballot_sync(0xffffffffu, word != 0);
          if (nz) {
            const int l = __ffs(nz) - 1;
            const uint32_t wv = __shfl_sync(0xffffffffu, word, l);
            bg = ((w0 + l) << 5) + __ffs(wv) - 1;
            bk = k;
          }
        }
      }
    }
    if (bg < 0) {
      c.fail_job = ji;
      c.fail_gen = c.cap_gen;
      return false;
    }
    DGpu& g = c.gpus[bg];
    // the GPU's first free slot of kind bk, one lane per slot
    const bool fs = lane < g.nslots && g.slot_kind[lane < 7 ? lane : 0] == bk &&
                    g.slot_job[lane < 7 ? lane : 0] == -1;
    const int bi = __ffs(__ballot_sync(0xffffffffu, fs)) - 1;
    CTX_SET(c.qhead, c.qhead + 1);
    occupy_slot(bg, bi, ji);
    roster_push(g, ji);
    DJob& jm = c.jobs[ji];
    jm.gpu = static_cast<int16_t>(bg);
    jm.slot = static_cast<int8_t>(bi);
    log_rec(kLogAdmitSlot, bg, ji, static_cast<uint8_t>(bi), 0, 0, 0);
    start_running(ji, g.slot_kind[bi]);
    spawn_instances(ji);
    return true;
  }

  // sim.hpp:465-478
  static __device__ bool admit_nopart(int ji) {
    Ctx& c = g_sim_ctx;
    if (ji == c.fail_job && c.fail_gen == c.cap_gen) return false;  // no GPU went idle since
    int best = -1;
    for (int gi = lane_id(); gi < c.G; gi += 32)
      if (c.gpus[gi].mode == kGpuIdle) {
        best = gi;
        break;
      }
    const unsigned any = __ballot_sync(0xffffffffu, best >= 0);
    if (!any) {
      c.fail_job = ji;
      c.fail_gen = c.cap_gen;
      return false;
    }
    // lowest id among lanes' first idle GPUs
    const int b = static_cast<int>(__reduce_min_sync(0xffffffffu, best >= 0 ? static_cast<uint32_t>(best) : 0xffffffffu));
    CTX_SET(c.qhead, c.qhead + 1);
    DGpu& g = c.gpus[b];
    g.mode = kGpuMig;
    roster_push(g, ji);
    c.jobs[ji].gpu = static_cast<int16_t>(b);
    log_rec(kLogAdmit, b, ji, 0, 0, 0, 0);
    start_running(ji, 4);
    spawn_instances(ji);
    return true;
  }

  // sim.hpp:398-418
  static __device__ void drain_queue() {
    Ctx& c = g_sim_ctx;
    if constexpr (POL == MISO_B200_POLICY_NOPART) {
      while (c.qhead < c.qtail && c.status == 0)
        if (!admit_nopart(c.queue[c.qhead])) break;
    } else if constexpr (POL == MISO_B200_POLICY_OPTSTA) {
      while (c.qhead < c.qtail && c.status == 0)
        if (!admit_optsta(c.queue[c.qhead])) break;
    } else {
      drain_dynamic();
    }
  }

  static __device__ void drain_dynamic() {
    Ctx& c = g_sim_ctx;
    for (;;) {
      int touched[32];
      int nt = 0;
      while (c.qhead < c.qtail && c.status == 0) {
        const int gi = place_dynamic(c.queue[c.qhead]);
        if (gi < 0) break;
        bool seen = false;
        for (int i = 0; i < nt; ++i) seen = seen || touched[i] == gi;
        if (!seen) {
          if (nt == 32) {  // flush early (rare: > 32 GPUs touched at one instant)
            for (int i = 0; i < nt; ++i) settle_admissions(touched[i]);
            nt = 0;
          }
          touched[nt++] = gi;
        }
      }
      if (nt == 0) return;
      for (int i = 0; i < nt && c.status == 0; ++i) settle_admissions(touched[i]);
    }
  }

  // sim.hpp:837-890
  static __device__ void complete_dynamic(int gi, int ji) {
    Ctx& c = g_sim_ctx;
    DGpu& g = c.gpus[gi];
    const DJob& j = c.jobs[ji];
    if (g.mode == kGpuMps) {
      if (g.nroster == 0) {
        ++g.epoch;
        clear_slot(c.J + gi);
        g.mode = kGpuIdle;
        sync_place(g);
        return;
      }
      const int lv = g.mps_level == 0 ? 100 : (g.mps_level == 1 ? 50 : 14);
      rate_roster_mps(gi, lv);
      return;
    }
    if (g.mode == kGpuReconfig) {
      for (int i = 0; i < g.plan_n; ++i) {
        if (g.plan_job[i] != ji) continue;
        g.plan_obj -= g.plan_speed[i];
        --g.plan_part[g.plan_slice[i]];
        for (int k = i; k + 1 < g.plan_n; ++k) {
          g.plan_job[k] = g.plan_job[k + 1];
          g.plan_slice[k] = g.plan_slice[k + 1];
          g.plan_speed[k] = g.plan_speed[k + 1];
          __syncwarp();
        }
        --g.plan_n;
        break;
      }
      if (g.part[j.slice] == 0) fail(MISO_B200_SIM_INVARIANT);
      else --g.part[j.slice];
      log_rec(kLogShrink, gi, -1, 0, pack_part(g.part), 0, 0);
      return;
    }
    if (g.part[j.slice] == 0) fail(MISO_B200_SIM_INVARIANT);
    else --g.part[j.slice];
    if (g.nroster == 0) {
      g.mode = kGpuIdle;
      sync_place(g);
#pragma unroll
      for (int k = 0; k < 5; ++k) g.part[k] = 0;
      g.objective = 0;
      return;
    }
    log_rec(kLogShrink, gi, -1, 0, pack_part(g.part), 0, 0);
    // lane i: roster entry i's estimated rate and drift test (loads in parallel); the objective
    // is then summed in roster order, as the reference's loop adds it
    const int n = g.nroster;
    double my_est = 0.0;
    bool drift = false;
    if (lane_id() < n) {
      const DJob& r = c.jobs[g.roster[lane_id()]];
      my_est = est_rate(r, r.slice);
      if (c.prm.drift_threshold > 0 && POL == MISO_B200_POLICY_MISO && c.prm.window_us > 0) {
        const double truth = true_rate(r, r.slice);
        drift = my_est > 0 && fabs(truth - my_est) / my_est > c.prm.drift_threshold;
      }
    }
    double obj = 0;
    for (int i = 0; i < n; ++i) obj += __shfl_sync(0xffffffffu, my_est, i);
    g.objective = obj;
    if (__ballot_sync(0xffffffffu, drift)) {
      start_profiling_session(gi);
      return;
    }
    reopt_and_apply(gi, false);
  }

  // sim.hpp:526-572: one migration per freed slot -- the running job with the largest strictly
  // positive true-speed gain on a strictly larger slot kind (ties: earliest arrival, then entry
  // order) moves in and checkpoint-restarts; its old slot joins the worklist. The job scan is a
  // warp argmin over the window of arrived, unfinished jobs.
  static __device__ void process_freed_slots(int gi0, int si0) {
    Ctx& c = g_sim_ctx;
    int wl_g[64], wl_s[64];
    int nw = 1;
    wl_g[0] = gi0;
    wl_s[0] = si0;
    while (nw > 0 && c.status == 0) {
      --nw;
      const int gi = wl_g[nw], si = wl_s[nw];
      drain_queue();
      DGpu& g = c.gpus[gi];
      if (g.slot_job[si] != -1) continue;
      const int kind = g.slot_kind[si];
      const int kg = kind_gpc(kind);
      int best = -1;
      double bgain = 0.0;
      int64_t barr = 0;
      const double* eff_k = c.efftruth + size_t(kind) * c.J;
      // (no job can run on a smaller kind than the partition's smallest: nothing to scan)
      const int lo = c.stp_lo, hi = kg > c.part_min_gpc ? c.stp_hi : lo;  // running jobs lie below stp_hi
      // dense arrays only (coalesced): state bytes four at a time (one 4-byte load per lane
      // covers 128 jobs per warp), then for the survivors the effective true speed on `kind`,
      // the running rate (rate_eff == rate for a running job) and the arrival time. The
      // comparison is a total order, so the visiting order does not matter.
      for (int b = (lo & ~3) + 4 * lane_id(); b < hi; b += 128) {
        const uint32_t w4 = *reinterpret_cast<const uint32_t*>(c.jst + b);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int mi = b + q;
          const uint32_t st = (w4 >> (8 * q)) & 255u;
          if (mi < lo || mi >= hi || (st & 64) || (st & 7) != kRunning) continue;
          if (kind_gpc((st >> 3) & 7) >= kg) continue;
          const double ns = eff_k[mi];
          if (!(ns > 0)) continue;
          const double gain = ns - c.rate_eff[mi];
          if (gain <= 0) continue;
          const int64_t arr = c.arr_us[mi];
          if (best < 0 || gain > bgain || (gain == bgain && (arr < barr || (arr == barr && mi < best)))) {
            best = mi;
            bgain = gain;
            barr = arr;
          }
        }
      }
      if (!__ballot_sync(0xffffffffu, best >= 0)) continue;
      {  // largest gain (> 0: its bits order like the value; complemented for a minimum), then
         // earliest arrival (>= 0), then lowest index
        const uint64_t gb = ~static_cast<uint64_t>(__double_as_longlong(bgain));
        const bool has = best >= 0;
        const uint32_t key[5] = {has ? static_cast<uint32_t>(gb >> 32) : 0xffffffffu,
                                 has ? static_cast<uint32_t>(gb) : 0xffffffffu,
                                 has ? static_cast<uint32_t>(static_cast<uint64_t>(barr) >> 32) : 0xffffffffu,
                                 has ? static_cast<uint32_t>(barr) : 0xffffffffu,
                                 has ? static_cast<uint32_t>(best) : 0xffffffffu};
        best = __shfl_sync(0xffffffffu, best, warp_argmin_words(key));
      }
      DJob& m = c.jobs[best];
      DGpu& og = c.gpus[m.gpu];
      free_slot(m.gpu, m.slot);
      if (nw == 64) {
        fail(MISO_B200_SIM_INVARIANT);
        return;
      }
      wl_g[nw] = m.gpu;
      wl_s[nw] = m.slot;
      ++nw;
      roster_erase(og, best);
      roster_push(g, best);
      occupy_slot(gi, si, best);
      m.gpu = static_cast<int16_t>(gi);
      m.slot = static_cast<int8_t>(si);
      m.slice = static_cast<uint8_t>(kind);
      sync_jst(best, m);
      CTX_SET(c.migrations, c.migrations + 1);
      log_rec(kLogMigrate, gi, best, static_cast<uint8_t>(kind), static_cast<uint32_t>(si), 0, 0);
      if (c.prm.ckpt_us > 0) {
        set_phase(best, kCkpt, 0.0);
        push_event(best, c.now + c.prm.ckpt_us, 2, kEvCkptDone);
      } else {
        start_running(best, m.slice);
      }
    }
  }

  // sim.hpp:798-835
  static __device__ void on_completion(int ji) {
    Ctx& c = g_sim_ctx;
    DJob& j = c.jobs[ji];
    if constexpr (PRUNE) {
    if (c.prune) {  // the job's remaining-work term leaves with it
      LB_SET(c.lb_p, c.lb_p - (j.lbp));
      LB_SET(c.lb_v, c.lb_v - (j.rate / prune_mx(j)));
    }
    }
    advance_job(j);
    if (c.prm.check_invariants) {
      const double base = j.base;
      if (fabs(j.consumed - base) > 1e-6 * base + 1e-9) fail(MISO_B200_SIM_INVARIANT);
    }
    const double old_term = (progressing(j.phase) && !(j.flags & kDone)) ? j.rate : 0.0;
    j.remaining = 0;
    j.flags |= kDone;
    ++j.epoch;
    clear_slot(ji);
    if constexpr (ASYNC) {
      if (__double_as_longlong(old_term) != 0) stp_post(kStpChange, ji, 0);
    } else {
      c.rate_eff[ji] = 0.0;
      if constexpr (STP) {
        c.stp_dirty = true;
        CTX_SET(c.stp_cmin, ji < c.stp_cmin ? ji : c.stp_cmin);
      }
    }
    sync_jst(ji, j);
    int stp_lo = c.stp_lo;
    while (stp_lo < c.n_arrived && (c.jst[stp_lo] & 64)) ++stp_lo;
    CTX_SET(c.stp_lo, stp_lo);  // done bit, dense
    j.completion_us = c.now;
    CTX_SET(c.done_count, c.done_count + 1);
    CTX_SET(c.last_completion, c.now > c.last_completion ? c.now : c.last_completion);
    if (c.prm.check_invariants) {
      int64_t total = 0;
#pragma unroll
      for (int b = 0; b < 5; ++b) total += j.acc[b];
      if (total != c.now - j.arrival_us) fail(MISO_B200_SIM_INVARIANT);
    }
    const int64_t jct = c.now - j.arrival_us;
    if constexpr (PRUNE) {
    if (c.prune) {
      LB_SET(c.lb_fin, c.lb_fin + (jct));
      LB_SET(c.lb_narr, c.lb_narr - 1);
      LB_SET(c.lb_arrsum, c.lb_arrsum - (j.arrival_us));
    }
    }
    log_rec(kLogComplete, -1, ji, 0, static_cast<uint32_t>(jct & 0xFFFFFFFF),
            static_cast<uint32_t>(jct >> 32), 0);
    const int gi = j.gpu;
    DGpu& g = c.gpus[gi];
    roster_erase(g, ji);
    if constexpr (POL == MISO_B200_POLICY_NOPART) {
      g.mode = kGpuIdle;
      CTX_SET(c.cap_gen, c.cap_gen + 1);
    } else if constexpr (POL == MISO_B200_POLICY_OPTSTA) {
      free_slot(gi, j.slot);
      process_freed_slots(gi, j.slot);
    } else {
      complete_dynamic(gi, ji);
    }
  }

  // sim.hpp:301-313
  static __device__ void dispatch(int slot, uint32_t kind) {
    Ctx& c = g_sim_ctx;
    if (slot < c.J) {
      const int ji = slot;
      if (kind == kEvArrival) {
        if (ji + 1 > c.n_arrived) c.n_arrived = ji + 1;
        log_rec(kLogArrival, -1, ji, 0, 0, 0, 0);
    if constexpr (PRUNE) {
        if (c.prune) {
          LB_SET(c.lb_narr, c.lb_narr + 1);
          LB_SET(c.lb_arrsum, c.lb_arrsum + (c.now));  // == arrival_us
        }
    }
        enqueue(ji);
      } else if (kind == kEvCompletion) {
        on_completion(ji);
      } else if (kind == kEvCkptDone) {  // on_migration_restart, sim.hpp:574
        start_running(ji, c.jobs[ji].slice);
      }
      return;
    }
    if constexpr (POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE) {
      // GPU-scoped events exist only under the dynamic policies
      const int gi = slot - c.J;
      DGpu& g = c.gpus[gi];
      if (kind == kEvMpsEnd) {  // on_mps_phase_end, sim.hpp:682-689
        if (++g.mps_level < 3) {
          start_mps_window(gi);
        } else {
          log_rec(kLogMpsEnd, gi, -1, 0, 0, 0, 0);
          finish_profiling(gi);
        }
      } else if (kind == kEvReconfigDone) {
        apply_assignment(gi);
      } else if (kind == kEvCkptDone) {
        begin_mps_windows(gi);
      }
    }
  }

  // validate_profile (profiles.hpp:67-87) and init_jobs' arrival checks (sim.hpp:246-254) for
  // trace job i: the first failing check, as a MISO_B200_SIM_BAD_* detail code (0 = valid).
  static __device__ int job_check(const SimBatch& b, int J0, int i) {
    const int q = J0 + i;
    if (!(b.base_s[q] > 0)) return MISO_B200_BAD_BASE;
    if (b.mem_gb[q] == 0 || b.mem_gb[q] > 40) return MISO_B200_BAD_MEM;
    const double* sp = b.speeds5 + size_t(q) * 5;
    for (int k = 0; k < 5; ++k)
      if (!(sp[k] > 0.0 && sp[k] <= 1.0)) return MISO_B200_BAD_SPEED_RANGE + k;
    if (sp[4] != 1.0) return MISO_B200_BAD_SPEED_7G;
    for (int k = 1; k < 5; ++k)
      if (sp[k] < sp[k - 1]) return MISO_B200_BAD_MONOTONE;
    if (b.instances && b.instances[q] < 1) return MISO_B200_BAD_INSTANCES;
    const int64_t a = us_from_s(b.arrival_s[q]);
    if (i == 0 && a != 0) return MISO_B200_BAD_FIRST_ARRIVAL;
    if (i > 0 && a < us_from_s(b.arrival_s[q - 1])) return MISO_B200_BAD_ARRIVAL_ORDER;
    return 0;
  }

  static __device__ __forceinline__ void run(const SimBatch& b, const SimParams& prm, const ModelW& w) {
    const int warp = static_cast<int>(blockIdx.x);  // one warp (block) per task
    if (warp >= b.n_seeds) return;
    const int lane = lane_id();
    Ctx& c = g_sim_ctx;
    // ---- input checks (the reference's invalid_argument cases; per-task status here) ----
    int bad = 0;
    const int tr = b.task_trace ? b.task_trace[warp] : warp;  // task -> trace
    int J0 = 0, JT = 0, extra = 0;
    if (tr < 0 || tr >= b.n_traces) {
      bad = MISO_B200_BAD_TASK_TRACE;
    } else {
      J0 = b.job_offsets[tr];
      JT = b.job_offsets[tr + 1] - J0;  // trace jobs
      if (JT < 1) bad = MISO_B200_BAD_NO_JOBS;  // sim.hpp:210
    }
    if (!bad && POL == MISO_B200_POLICY_OPTSTA) {  // a feasible static partition
      const uint8_t* sc = b.static_counts + size_t(warp) * 5;
      int tot = 0, gp = 0, un = 0;
      const int maxc[5] = {7, 3, 2, 1, 1}, units[5] = {1, 2, 4, 4, 8};
      for (int k = 0; k < 5; ++k) {
        if (sc[k] > maxc[k]) tot = 99;
        tot += sc[k];
        gp += sc[k] * kind_gpc(k);
        un += sc[k] * units[k];
      }
      if (tot < 1 || tot > 7 || gp > 7 || un > 8 || (sc[3] > 0 && sc[2] > 0)) bad = MISO_B200_BAD_STATIC;
    }
    if (!bad) {
      // first failing trace job in job order (the reference validates in that order)
      int first = INT32_MAX, code = 0;
      for (int i = lane; i < JT; i += 32) {
        if (b.instances) extra += b.instances[J0 + i] > 1 ? b.instances[J0 + i] - 1 : 0;
        if (i < first) {
          const int e = job_check(b, J0, i);
          if (e) {
            first = i;
            code = e;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        extra += __shfl_xor_sync(0xffffffffu, extra, off);
        const int of = __shfl_xor_sync(0xffffffffu, first, off);
        const int oc = __shfl_xor_sync(0xffffffffu, code, off);
        if (of < first) {
          first = of;
          code = oc;
        }
      }
      if (code) {
        bad = code | (first << 8);
      } else if (JT + extra > b.max_jobs) {  // capacity: every job's instance_count (sim.hpp:242)
        bad = MISO_B200_BAD_CAPACITY;
      }
    }
    if (bad) {
      if (lane == 0) {
        SimMetrics m{};
        m.status = MISO_B200_SIM_BAD_INPUT;
        m.detail = bad;
        b.metrics[warp] = m;
      }
      if constexpr (ASYNC) {  // release the helper warp
        if (lane == 0) g_stp_ring.quit = 1;
        __syncwarp();
        stp_pair_barrier();
      }
      return;
    }
    const int J = JT + extra;  // clones occupy [JT, J)
    const int G = prm.cluster_size;
    unsigned char* ws = b.workspace + size_t(warp) * b.ws_stride;
    c.jobs = reinterpret_cast<DJob*>(ws);  // stride kSimJobBytes == sizeof rounded (asserted)
    c.gpus = reinterpret_cast<DGpu*>(ws + sim_ws_gpus_off(b.max_jobs));
    c.slots = reinterpret_cast<Slot*>(ws + sim_ws_slots_off(b.max_jobs, G));
    c.queue = reinterpret_cast<int32_t*>(ws + sim_ws_queue_off(b.max_jobs, G));
    c.rate_eff = reinterpret_cast<double*>(ws + sim_ws_scratch_off(b.max_jobs, G));
    c.stp_prefix = reinterpret_cast<double*>(ws + sim_ws_prefix_off(b.max_jobs, G));
    c.jst = ws + sim_ws_jst_off(b.max_jobs, G);
    c.freemask = reinterpret_cast<uint32_t*>(ws + sim_ws_freemask_off(b.max_jobs, G));
    c.efftruth = reinterpret_cast<double*>(ws + sim_ws_efftruth_off(b.max_jobs, G));
    c.arr_us = reinterpret_cast<int64_t*>(ws + sim_ws_arrival_off(b.max_jobs, G));
    c.gplace = ws + sim_ws_gplace_off(b.max_jobs, G);
    c.W = (G + 31) / 32;
    c.part_min_gpc = 99;
    if (POL == MISO_B200_POLICY_OPTSTA) {
      const uint8_t* sc = b.static_counts + size_t(warp) * 5;
      for (int k = 4; k >= 0; --k)
        if (sc[k] > 0) c.part_min_gpc = kind_gpc(k);
    }
    c.stp_cmin = INT32_MAX;
    c.stp_lo = 0;
    c.n_arrived = 0;
    c.stp_hi = 0;
    c.lmin_t[lane] = kNoEvent;
    c.lmin_pk[lane] = ~0ull;
    c.lmin_idx[lane] = -1;
    c.lmin_valid[lane] = false;
    c.chunk = (J + G + 31) / 32;
    c.log = b.log ? b.log + size_t(warp) * b.log_cap : nullptr;
    c.log_cap = b.log_cap;
    c.log_n = 0;
    c.stp_series = b.stp_series ? b.stp_series + size_t(warp) * 2 * b.stp_cap : nullptr;
    c.stp_cap = b.stp_cap;
    c.J = J;
    c.J_used = JT;
    c.cap_gen = 0;
    c.fail_gen = 0;
    c.fail_job = -1;
    c.G = G;
    c.qhead = c.qtail = 0;
    c.now = 0;
    c.seq = 0;
    c.nonce = 0;
    c.stp_cur = 0;
    c.stp_integral = 0;
    c.stp_last = 0;
    c.stp_points = 0;
    c.stp_dirty = false;
    c.repartitions = c.migrations = c.mps_sessions = c.done_count = 0;
    c.first_progress = -1;
    c.last_completion = -1;
    c.status = 0;
    c.detail = 0;
    c.processed = 0;
    c.prune = PRUNE && b.prune_bound != nullptr && J == JT;
    c.lb_fin = c.lb_narr = c.lb_arrsum = c.lb_unstarted = 0;
    c.lb_p = c.lb_v = 0.0;
    c.prm = prm;
    c.spare_lut = b.spare_lut;
    c.rng_seed = b.rng_seed[warp];  // per task
    c.w = w;
    c.draws = b.draws ? b.draws + size_t(warp) * size_t(b.draws_k) * 14 : nullptr;
    c.draws_k = b.draws_k;
    int64_t lb_unstarted = 0;  // (pruned search) per-lane partial sum, reduced below
    __syncwarp();

    // ---- init_jobs / init_gpus (sim.hpp:240-276), lanes in parallel ----
    for (int i = lane; i < JT; i += 32) {
      DJob& j = c.jobs[i];
      const int64_t a = us_from_s(b.arrival_s[J0 + i]);
      j.remaining = b.base_s[J0 + i];
      j.base = j.remaining;
      j.consumed = 0;
      j.rate = 0;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        j.truth[k] = b.speeds5[(size_t(J0) + i) * 5 + k];
        j.est[k] = 0;
        j.acc[k] = 0;
      }
      j.arrival_us = a;
      j.last_update_us = a;
      j.first_progress_us = -1;
      j.completion_us = -1;
      j.epoch = 0;
      j.gpu = -1;
      j.phase = kQueued;
      j.slice = 4;
      j.mem = b.mem_gb[J0 + i];
      j.qos = b.qos_kind[J0 + i];
      const int qg = j.qos >= 0 ? kind_gpc(j.qos) : 0;
      int mk = -1;  // min_slice_for (topology.hpp:68-72)
      for (int k = 4; k >= 0; --k)
        if (kind_mem_gb(k) >= j.mem && kind_gpc(k) >= qg) mk = k;
      j.min_kind = static_cast<uint8_t>(mk < 0 ? 0xFF : mk);
      j.flags = 0;
      j.slot = -1;
      j.inst = b.instances ? b.instances[J0 + i] : 1;
      j.clone_k = 0;
      j.parent = -1;
      c.jst[i] = kQueued | (4 << 3);
#pragma unroll
      for (int k = 0; k < 5; ++k) c.efftruth[size_t(k) * J + i] = effective_speed(j.truth[k], k, j.mem, j.qos);
      c.arr_us[i] = a;
      if constexpr (PRUNE)
        if (c.prune) {
          const uint8_t* sc = b.static_counts + size_t(warp) * 5;
          double mx = 0.0;
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const double r = c.efftruth[size_t(k) * J + i];
            if (sc[k] > 0 && r > mx) mx = r;
          }
          j.est[0] = mx > 0.0 ? mx : 1.0;
          lb_unstarted += runtime_floor_us(j);
        }
      Slot s;  // arrival events pushed in job order: seq = j (sim.hpp:219)
      s.t = a;
      s.pk = (1ull << 62) | (static_cast<uint64_t>(i) << 3) | kEvArrival;
      c.slots[i] = s;
    }
    for (int gi = lane; gi < G; gi += 32) {
      DGpu& g = c.gpus[gi];
      g.objective = 0;
      g.plan_obj = 0;
      g.epoch = 0;
      g.mode = kGpuIdle;
      g.mps_level = 0;
      g.nroster = 0;
      g.plan_n = 0;
      g.plan_valid = 0;
      for (int k = 0; k < 5; ++k) g.part[k] = g.plan_part[k] = g.kind_cnt[k] = 0;
      g.spare = 4;
      g.nslots = 0;
      for (int k = 0; k < 5; ++k) g.fcnt[k] = 0;
      if (POL == MISO_B200_POLICY_OPTSTA) {  // init_gpus, sim.hpp:266-276
        const uint8_t* sc = b.static_counts + size_t(warp) * 5;
        for (int k = 0; k < 5; ++k) g.fcnt[k] = sc[k];
        for (int k = 4; k >= 0; --k)
          for (int r = 0; r < sc[k]; ++r) {
            g.slot_kind[g.nslots] = static_cast<uint8_t>(k);
            g.slot_job[g.nslots] = -1;
            ++g.nslots;
          }
        for (int k = 0; k < 5; ++k) g.part[k] = sc[k];
        g.mode = kGpuMig;
      }
      c.slots[J + gi].t = kNoEvent;
      c.gplace[gi] = 0x50;  // idle, no jobs: takes any job (sync_place)
    }
    for (int i = JT + lane; i < J; i += 32) {  // clone slots: no event, not arrived
      c.slots[i].t = kNoEvent;
      c.jst[i] = kQueued | (4 << 3);
    }
    for (int i = lane; i < J; i += 32) c.rate_eff[i] = 0.0;
    if (POL == MISO_B200_POLICY_OPTSTA)
      for (int wi = lane; wi < 5 * c.W; wi += 32) {  // every GPU starts with all slots free
        const int k = wi / c.W, wd = wi % c.W;
        const uint8_t* sc = b.static_counts + size_t(warp) * 5;
        uint32_t v = 0;
        if (sc[k] > 0) {
          const int nb = G - (wd << 5);
          v = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
        }
        c.freemask[wi] = v;
      }
    if constexpr (PRUNE) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) lb_unstarted += __shfl_xor_sync(0xffffffffu, lb_unstarted, off);
      c.lb_unstarted = lb_unstarted;
    }
    if constexpr (ASYNC) {  // the helper's state: an empty ring, rate_eff (zeroed above) and a
                            // zeroed partial-sum cache (every term starts at 0.0)
      for (int q = lane; q < (J + 7) / 8 + 1; q += 32) c.stp_prefix[q] = 0.0;
      if (lane == 0) {
        g_stp_ring.tail = 0;
        g_stp_ring.head = 0;
        g_stp_ring.quit = 0;
      }
      __syncwarp();
      stp_pair_barrier();
    }
    c.seq = static_cast<uint64_t>(JT);  // one arrival event per trace job (sim.hpp:219)
    bool bad_job = false;
    for (int i = lane; i < JT; i += 32) bad_job = bad_job || c.jobs[i].min_kind == 0xFF;
    bad_job = __any_sync(0xffffffffu, bad_job);
    __syncwarp();

    // ---- event loop (sim.hpp:221-233) ----
    if (bad_job && (POL == MISO_B200_POLICY_MISO || POL == MISO_B200_POLICY_ORACLE))
      c.status = MISO_B200_SIM_INVARIANT;  // "fits no slice kind" (sim.hpp:381)
    uint64_t processed = 0;  // warp-uniform, in a register (stored to Ctx after the loop)
    while (c.status == 0) {
      Slot ev;
      const int slot = next_event(&ev);
      if (slot < 0) break;
      ++processed;
      if (processed > prm.max_events) {
        c.status = MISO_B200_SIM_EVENT_BUDGET;
        break;
      }
      clear_slot(slot);
      __syncwarp();
      if constexpr (STP && !ASYNC) {
        CTX_SET(c.stp_integral, c.stp_integral + (c.stp_cur * s_from_us(ev.t - c.stp_last)));
        c.stp_last = ev.t;
      }
      c.now = ev.t;
      dispatch(slot, static_cast<uint32_t>(ev.pk & 7));
      drain_queue();
      if constexpr (ASYNC) stp_post(kStpEvent, 0, ev.t);  // the helper's integral step + refresh
      refresh_stp();
      __syncwarp();
    if constexpr (PRUNE) {
      if (c.prune && (processed & 31) == 0) {
        // chosen-only search: stop once this run's JCT sum provably exceeds a completed
        // candidate's (then its avg_jct_s > that candidate's, so it cannot be the first minimum)
        bool stop = false;
        if (lane == 0) {
          const int64_t thr = *reinterpret_cast<volatile const int64_t*>(b.prune_bound + tr);
          // exact integer part + the started jobs' remaining-work floor (FP sums: 1 s of margin,
          // far above their rounding error)
          const int64_t lbi = c.lb_fin + c.lb_narr * c.now - c.lb_arrsum + c.lb_unstarted;
          const double lb = static_cast<double>(lbi) + (c.lb_p - c.lb_v * s_from_us(c.now)) * 1e6 - 1e6;
          stop = thr != INT64_MAX && lb > static_cast<double>(thr) * (1.0 + 1e-9) + 2.0 * JT;
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) {
          c.status = MISO_B200_SIM_PRUNED;
          break;
        }
      }
    }
    }
    c.processed = processed;
    if constexpr (ASYNC) {  // the helper finishes the STP; its results are in Ctx after this
      stp_post(kStpEnd, 0, 0);
      stp_pair_barrier();
      if (g_stp_ring.quit == 2) c.status = MISO_B200_SIM_INVARIANT;
    }
    // every pushed event is popped by the reference exactly once (live or stale), so its
    // max_events budget (sim.hpp:224, stale pops included) is exceeded iff the pushes exceed it
    CTX_SET(c.status, (c.status == 0 && c.seq > prm.max_events) ? MISO_B200_SIM_EVENT_BUDGET : c.status);
    if constexpr (PRUNE) {
    if (c.prune && c.status == 0 && c.done_count == JT && lane == 0)
      atomicMin(reinterpret_cast<long long*>(b.prune_bound + tr), static_cast<long long>(c.lb_fin));
    }

    // ---- finalize (sim.hpp:902-949) ----
    const int JU = c.J_used;  // jobs_.size(): trace jobs + spawned clones (sim.hpp:903-913)
    if (b.job_out) {  // per-job report inputs (sim.hpp:916-929), lanes in parallel
      int64_t* o = b.job_out + size_t(warp) * size_t(b.max_jobs) * kJobOutFields;
      for (int i = lane; i < JU; i += 32) {
        const DJob& j = c.jobs[i];
        int64_t* r = o + size_t(kJobOutFields) * i;
        r[0] = (j.flags & kDone) ? j.completion_us : -1;
#pragma unroll
        for (int k = 0; k < 5; ++k) r[1 + k] = j.acc[k];
        r[6] = j.parent;
        r[7] = j.clone_k;
      }
      for (int i = JU + lane; i < b.max_jobs; i += 32)  // rows past the task's jobs: zeros
        for (int f = 0; f < kJobOutFields; ++f) o[size_t(kJobOutFields) * i + f] = 0;
    }
    SimMetrics m{};  // value-initialised: the padding bytes are deterministic too
    m.status = c.status;
    m.detail = c.detail;
    m.job_count = JU;
    m.completed_count = c.done_count;
    m.completed = c.done_count == JU;
    m.repartitions = c.repartitions;
    m.migrations = c.migrations;
    m.mps_sessions = c.mps_sessions;
    m.events = static_cast<int64_t>(c.processed);
    m.log_records = c.log_n;
    m.stp_points = c.stp_points;
    // sim.hpp:914-928: sums in job order over completed jobs. 32 jobs are loaded per step (one
    // memory round trip instead of one per job) and summed sequentially through shuffles --
    // the same additions in the same order.
    double totals[5] = {0, 0, 0, 0, 0};
    double jct_sum = 0;
    for (int base = 0; base < JU; base += 32) {
      const int i = base + lane;
      double v = 0, a[5] = {0, 0, 0, 0, 0};
      bool done = false;
      if (i < JU) {
        const DJob& j = c.jobs[i];
        done = (j.flags & kDone) != 0;
        if (b.job_jct_us && !b.task_trace && i < JT)
          b.job_jct_us[J0 + i] = done ? j.completion_us - j.arrival_us : -1;
        if (done) {
          v = s_from_us(j.completion_us - j.arrival_us);
#pragma unroll
          for (int k = 0; k < 5; ++k) a[k] = s_from_us(j.acc[k]);
        }
      }
      const unsigned dm = __ballot_sync(0xffffffffu, done);
      const int cnt = JU - base < 32 ? JU - base : 32;
      for (int t = 0; t < cnt; ++t) {
        const double vt = __shfl_sync(0xffffffffu, v, t);
        double at[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) at[k] = __shfl_sync(0xffffffffu, a[k], t);
        if ((dm >> t) & 1u) {
          jct_sum += vt;
#pragma unroll
          for (int k = 0; k < 5; ++k) totals[k] += at[k];
        }
      }
    }
    m.queue_frac = m.mps_frac = m.checkpoint_frac = m.run_frac = m.idle_frac = 0;
    if (jct_sum > 0) {
      m.queue_frac = totals[0] / jct_sum;
      m.mps_frac = totals[1] / jct_sum;
      m.checkpoint_frac = totals[2] / jct_sum;
      m.run_frac = totals[3] / jct_sum;
      m.idle_frac = totals[4] / jct_sum;
    }
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    m.avg_jct_s = inf;
    m.makespan_s = inf;
    m.stp_time_avg = 0;
    if (m.completed) {
      m.avg_jct_s = jct_sum / static_cast<double>(JU);
      m.makespan_s = s_from_us(c.last_completion - c.first_progress);
      if (c.last_completion > c.first_progress)
        m.stp_time_avg = c.stp_integral / s_from_us(c.last_completion - c.first_progress);
    }
    m.jct_sum_s = jct_sum;
    if (lane == 0) b.metrics[warp] = m;
  }
};

}  // namespace simk
}  // namespace miso_b200
