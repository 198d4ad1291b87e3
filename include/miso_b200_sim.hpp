// miso_b200_sim.hpp -- the simulator half of the drop-in binding: the reference's
// run_simulation (sim.hpp:976-992) and best_static_partition (sim.hpp:1031-1066) routed to the
// B200 event-step kernel, plus batch forms that run many independent simulations in ONE
// launch (one warp per simulation). Header-only, C++20, included after the reference's
// "miso/sim.hpp"; it uses the reference's types (JobTrace, SimOptions, MetricsReport,
// StaticSearchResult, ...) unchanged and keeps signatures, argument meaning and error
// behaviour:
//
//   miso::b200::run_simulation(trace, options)            == run_simulation (sim.hpp:976)
//   miso::b200::run_simulation(trace, n, policy, o, p, s) == the 6-argument overload (:981)
//   miso::b200::best_static_partition(trace, n, o, cat)   == best_static_partition (:1031)
//   miso::b200::run_simulation_batch(...)                 many traces / seeds / partitions
//   miso::b200::best_static_partition_batch(...)          every (trace, candidate) at once
//
// The MetricsReport is complete: scalars, per_job (phase times from the device's per-job
// accumulators), jct_sorted, stp_series, and the event log text written to
// options.event_log in the reference's format (sim.hpp:365-367). Errors: std::invalid_argument
// for bad options/traces (validated with the reference's own validators, in its order),
// SimInvariantError for engine failures, InfeasibleError from the static search.
// Multi-instance jobs (JobProfile::instance_count > 1) spawn their clones on the device as in
// SimEngine::spawn_instances. A caller-fitted SimOptions::small_slice_model is used as the
// reference uses it (sim.hpp:894-896). Batches are spread over every device
// (miso_b200_simulate_batch_sharded; Device::all()).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <optional>
#include <ostream>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "miso/sim.hpp"
#include "miso_b200_ref.hpp"

namespace miso {
namespace b200 {
namespace detail {

// Traces in CSR form for miso_b200_simulate_batch_host.
struct TraceArrays {
  std::vector<int32_t> offsets{0};
  std::vector<double> arrival, base, speeds;
  std::vector<uint8_t> mem, inst;
  std::vector<int8_t> qos;

  void add(const JobTrace& t) {
    for (const TraceJob& j : t.jobs) {
      inst.push_back(static_cast<uint8_t>(std::clamp(j.profile.instance_count, 1, 255)));
      arrival.push_back(j.arrival_s);
      base.push_back(j.profile.base_duration_s);
      for (int k = 0; k < 5; ++k) speeds.push_back(j.profile.speed_table.v[k]);
      mem.push_back(static_cast<uint8_t>(j.profile.mem_demand_gb));
      qos.push_back(j.profile.qos_min_slice ? static_cast<int8_t>(slice_index(*j.profile.qos_min_slice))
                                            : int8_t(-1));
    }
    offsets.push_back(offsets.back() + static_cast<int32_t>(t.jobs.size()));
  }
};

// SimEngine's constructor and init_jobs checks (sim.hpp:204-212, 240-258), same order.
inline void validate(const JobTrace& trace, const SimOptions& opt) {
  validate_overheads(opt.overheads);
  validate_predictor_spec(opt.predictor);
  if (opt.cluster_size < 1) throw std::invalid_argument("cluster_size must be >= 1");
  if (opt.policy == Policy::optsta && !opt.static_partition)
    throw std::invalid_argument("optsta requires a static partition");
  if (trace.jobs.empty()) throw std::invalid_argument("trace has no jobs");
  std::set<std::string> ids;
  int64_t prev = 0;
  for (size_t i = 0; i < trace.jobs.size(); ++i) {
    const TraceJob& t = trace.jobs[i];
    validate_profile(t.profile);
    if (!ids.insert(t.profile.job_id).second)
      throw std::invalid_argument("duplicate job id '" + t.profile.job_id + "'");
    const int64_t a = ::miso::detail::us_from_s(t.arrival_s);
    if (i == 0 && a != 0) throw std::invalid_argument("first arrival must be at t=0");
    if (a < prev) throw std::invalid_argument("arrival times must be non-decreasing");
    prev = a;
    if (t.profile.instance_count > 255)
      throw std::invalid_argument("miso_b200: instance_count above 255");
  }
  if (opt.cluster_size > 32767) throw std::invalid_argument("miso_b200: cluster_size above 32767");
}

inline miso_b200_sim_options to_c(const SimOptions& o) {
  miso_b200_sim_options c{};
  c.policy = o.policy == Policy::nopart   ? MISO_B200_POLICY_NOPART
             : o.policy == Policy::optsta ? MISO_B200_POLICY_OPTSTA
             : o.policy == Policy::oracle ? MISO_B200_POLICY_ORACLE
                                          : MISO_B200_POLICY_MISO;
  c.cluster_size = o.cluster_size;
  c.mig_reconfig_s = o.overheads.mig_reconfig_s;
  c.checkpoint_restart_s = o.overheads.checkpoint_restart_s;
  c.mps_window_s = o.overheads.mps_window_s;
  c.interference = o.overheads.interference;
  c.predictor_noisy = o.predictor.mode == PredictorSpec::Mode::noisy ? 1 : 0;
  c.target_mae = o.predictor.target_mae;
  c.check_invariants = o.check_invariants ? 1 : 0;
  c.reprofile_drift_threshold = o.reprofile_drift_threshold;
  c.max_events = o.max_events;
  c.small_slice_model_fitted = o.small_slice_model.fitted ? 1 : 0;  // sim.hpp:894-896
  for (int i = 0; i < 4; ++i) {
    c.small_slice_w2[i] = o.small_slice_model.w_2g[static_cast<size_t>(i)];
    c.small_slice_w1[i] = o.small_slice_model.w_1g[static_cast<size_t>(i)];
  }
  return c;
}

// MISO_B200_SIM_BAD_INPUT's detail as the reference's std::invalid_argument text.
inline std::string bad_input_message(const JobTrace* trace, int detail) {
  const int code = detail & 0xFF, job = detail >> 8;
  std::string id = trace && static_cast<size_t>(job) < trace->jobs.size()
                       ? trace->jobs[static_cast<size_t>(job)].profile.job_id
                       : "j" + std::to_string(job);
  const std::string pre = "job '" + id + "': ";
  static const char* kinds[5] = {"1g", "2g", "3g", "4g", "7g"};
  if (code >= MISO_B200_BAD_SPEED_RANGE && code < MISO_B200_BAD_SPEED_RANGE + 5)
    return pre + "speed on " + kinds[code - MISO_B200_BAD_SPEED_RANGE] + " outside (0,1]";
  switch (code) {
    case MISO_B200_BAD_BASE: return pre + "base duration must be positive";
    case MISO_B200_BAD_MEM: return pre + "memory demand must be in (0, 40] GB";
    case MISO_B200_BAD_SPEED_7G: return pre + "speed on 7g must be exactly 1";
    case MISO_B200_BAD_MONOTONE: return pre + "speed table not monotone in gpc count";
    case MISO_B200_BAD_INSTANCES: return pre + "instance count must be >= 1";
    case MISO_B200_BAD_FIRST_ARRIVAL: return "first arrival must be at t=0";
    case MISO_B200_BAD_ARRIVAL_ORDER: return "arrival times must be non-decreasing";
    case MISO_B200_BAD_NO_JOBS: return "trace has no jobs";
    case MISO_B200_BAD_STATIC: return "static partition is not a feasible partition";
    default: return "miso_b200: invalid simulation input (detail " + std::to_string(detail) + ")";
  }
}

[[noreturn]] inline void throw_status(int status, int detail = 0, const JobTrace* trace = nullptr) {
  switch (status) {
    case MISO_B200_SIM_BAD_INPUT: throw std::invalid_argument(bad_input_message(trace, detail));
    case MISO_B200_SIM_EVENT_BUDGET: throw SimInvariantError("event budget exhausted");
    case MISO_B200_SIM_NO_PARTITION: throw SimInvariantError("no feasible partition for admitted roster");
    case MISO_B200_SIM_INFEASIBLE_SLICE: throw SimInvariantError("job placed on infeasible slice");
    default: throw SimInvariantError("simulation invariant violated (device engine)");
  }
}

inline const char* kind_name(int k) { return slice_name(kAllSlices[static_cast<size_t>(k)]); }

inline PartitionConfig unpack_part(uint32_t a) {
  std::array<uint8_t, kSliceKinds> c{};
  for (int k = 0; k < 5; ++k) c[static_cast<size_t>(k)] = static_cast<uint8_t>((a >> (4 * k)) & 15);
  return PartitionConfig::from_counts(c);
}

// Job ids in SimEngine order: the trace's, then clones "parent#k" in spawn order (job_out
// carries each clone's parent and k).
inline std::vector<std::string> job_ids(const JobTrace& trace, const int64_t* job_out, int n) {
  std::vector<std::string> ids;
  ids.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    if (static_cast<size_t>(i) < trace.jobs.size()) {
      ids.push_back(trace.jobs[static_cast<size_t>(i)].profile.job_id);
    } else {
      const int64_t* o = job_out + size_t(MISO_B200_JOB_OUT_FIELDS) * static_cast<size_t>(i);
      ids.push_back(ids[static_cast<size_t>(o[6])] + "#" + std::to_string(o[7]));
    }
  }
  return ids;
}

// The reference's event-log text (sim.hpp:365-367 and its log() call sites) from the device's
// compact records.
inline void render_log(const std::vector<std::string>& ids, const miso_b200_log_record* r,
                       int64_t n, std::ostream& out) {
  auto jid = [&](int j) -> const std::string& { return ids[static_cast<size_t>(j)]; };
  for (int64_t i = 0; i < n; ++i) {
    const miso_b200_log_record& e = r[i];
    const int g = e.gpu;
    const uint64_t ab = uint64_t(e.a) | (uint64_t(e.b) << 32);
    out << e.t << ' ';
    switch (e.kind) {
      case MISO_B200_LOG_ARRIVAL: out << "arrival job=" << jid(e.job); break;
      case MISO_B200_LOG_ADMIT: out << "admit gpu=" << g << " job=" << jid(e.job); break;
      case MISO_B200_LOG_START:
        out << "start job=" << jid(e.job) << " gpu=" << g << " slice=" << kind_name(e.x)
            << " rate=" << fmt_g(e.v);
        break;
      case MISO_B200_LOG_CKPT_START: out << "ckpt_start gpu=" << g << " jobs=" << e.a; break;
      case MISO_B200_LOG_MPS_START: out << "mps_start gpu=" << g << " jobs=" << e.a; break;
      case MISO_B200_LOG_MPS_WINDOW: out << "mps_window gpu=" << g << " level=" << e.a; break;
      case MISO_B200_LOG_MPS_END: out << "mps_end gpu=" << g; break;
      case MISO_B200_LOG_RECONFIG_START:
        out << "reconfig_start gpu=" << g << " pause_us=" << static_cast<int64_t>(ab);
        break;
      case MISO_B200_LOG_PARTITION: {
        out << "partition gpu=" << g << " shape=" << unpack_part(e.a).name() << " assign=";
        const int m = e.x;
        for (int q = 0; q < m && i + 1 < n; ++q) {
          ++i;
          out << (q ? "," : "") << jid(r[i].job) << '@' << kind_name(r[i].x);
        }
        break;
      }
      case MISO_B200_LOG_COMPLETE:
        out << "complete job=" << jid(e.job) << " jct_us=" << static_cast<int64_t>(ab);
        break;
      case MISO_B200_LOG_SHRINK: out << "shrink gpu=" << g << " shape=" << unpack_part(e.a).name(); break;
      case MISO_B200_LOG_ADMIT_SLOT:
        out << "admit gpu=" << g << " job=" << jid(e.job) << " slot=" << int(e.x);
        break;
      case MISO_B200_LOG_MIGRATE:
        out << "migrate job=" << jid(e.job) << " gpu=" << g << " slot=" << e.a
            << " slice=" << kind_name(e.x);
        break;
      case MISO_B200_LOG_SPAWN:
        out << "spawn job=" << jid(e.job) << " parent=" << jid(static_cast<int>(e.a));
        break;
      default: out << "?kind=" << int(e.kind); break;
    }
    out << '\n';
  }
}

// finalize (sim.hpp:902-949) from the device's scalars and per-job accumulators.
inline MetricsReport make_report(const JobTrace& trace, Policy policy,
                                 const miso_b200_sim_metrics& m, const int64_t* job_out,
                                 const std::vector<std::string>* ids, const double* stp,
                                 int64_t stp_n) {
  MetricsReport r;
  r.policy = policy_label(policy);
  r.seed = trace.spec.seed;
  r.job_count = m.job_count;
  r.completed_count = m.completed_count;
  r.completed = m.completed != 0;
  r.repartitions = m.repartitions;
  r.migrations = m.migrations;
  r.mps_sessions = m.mps_sessions;
  r.avg_jct_s = m.avg_jct_s;
  r.makespan_s = m.makespan_s;
  r.stp_time_avg = m.stp_time_avg;
  r.queue_frac = m.queue_frac;
  r.mps_frac = m.mps_frac;
  r.checkpoint_frac = m.checkpoint_frac;
  r.run_frac = m.run_frac;
  r.idle_frac = m.idle_frac;
  if (job_out) {
    r.per_job.reserve(static_cast<size_t>(m.job_count));
    std::vector<int64_t> arr_us(static_cast<size_t>(m.job_count));
    for (int i = 0; i < m.job_count; ++i) {
      const int64_t* o = job_out + size_t(MISO_B200_JOB_OUT_FIELDS) * static_cast<size_t>(i);
      arr_us[static_cast<size_t>(i)] =
          o[6] < 0 ? ::miso::detail::us_from_s(trace.jobs[static_cast<size_t>(i)].arrival_s)
                   : arr_us[static_cast<size_t>(o[6])];  // clones keep the parent's arrival
      JobMetrics jm;
      jm.job_id = (*ids)[static_cast<size_t>(i)];
      const int64_t arr = arr_us[static_cast<size_t>(i)];
      jm.arrival_s = ::miso::detail::s_from_us(arr);
      jm.queue_s = ::miso::detail::s_from_us(o[1]);
      jm.mps_s = ::miso::detail::s_from_us(o[2]);
      jm.checkpoint_s = ::miso::detail::s_from_us(o[3]);
      jm.run_s = ::miso::detail::s_from_us(o[4]);
      jm.idle_s = ::miso::detail::s_from_us(o[5]);
      if (o[0] >= 0) {
        jm.completion_s = ::miso::detail::s_from_us(o[0]);
        jm.jct_s = ::miso::detail::s_from_us(o[0] - arr);
        r.jct_sorted.push_back(jm.jct_s);
      }
      r.per_job.push_back(std::move(jm));
    }
    std::sort(r.jct_sorted.begin(), r.jct_sorted.end());
  }
  for (int64_t i = 0; stp && i < stp_n; ++i) r.stp_series.emplace_back(stp[2 * i], stp[2 * i + 1]);
  return r;
}

}  // namespace detail

// Runs traces[t] (t < traces.size()) under `options` in one launch. rng_seeds (optional, one per
// trace) override options.predictor.rng_seed per simulation; static_parts (optional) override
// options.static_partition per simulation (optsta). full = false returns scalar metrics only
// (no per_job / jct_sorted / stp_series, STP not tracked: stp_time_avg reads 0) -- the
// best-static search's form. Errors are thrown for the first failing simulation.
inline std::vector<MetricsReport> run_simulation_batch(
    const std::vector<const JobTrace*>& traces, const SimOptions& options,
    const std::vector<uint64_t>* rng_seeds = nullptr,
    const std::vector<std::optional<PartitionConfig>>* static_parts = nullptr, bool full = true) {
  const size_t n = traces.size();
  std::vector<MetricsReport> out;
  if (n == 0) return out;
  detail::TraceArrays ta;
  std::vector<uint64_t> seeds(n, options.predictor.rng_seed);
  std::vector<uint8_t> sc;
  const bool optsta = options.policy == Policy::optsta;
  int max_jobs = 0;
  for (size_t i = 0; i < n; ++i) {
    SimOptions oi = options;
    if (static_parts) oi.static_partition = (*static_parts)[i];
    detail::validate(*traces[i], oi);
    ta.add(*traces[i]);
    if (rng_seeds) seeds[i] = (*rng_seeds)[i];
    if (optsta)
      for (int k = 0; k < 5; ++k) sc.push_back(oi.static_partition->counts()[static_cast<size_t>(k)]);
    int cap = 0;
    for (const TraceJob& j : traces[i]->jobs) cap += std::max(1, j.profile.instance_count);
    max_jobs = std::max(max_jobs, cap);
  }
  const miso_b200_sim_options c = detail::to_c(options);
  AllDevices all(options.catalog);
  if (!all.catalog_ok() && (options.policy == Policy::miso || options.policy == Policy::oracle))
    throw SimInvariantError("no feasible partition for admitted roster on gpu 0");  // sim.hpp:728
  std::vector<miso_b200_sim_metrics> met(n);
  std::vector<int64_t> job_out(full ? n * size_t(max_jobs) * MISO_B200_JOB_OUT_FIELDS : 0);
  const bool want_log = full && options.event_log != nullptr;
  int64_t log_cap = want_log ? 64 * int64_t(max_jobs) + 1024 : 0;
  int64_t stp_cap = full ? 16 * int64_t(max_jobs) + 64 : 0;
  std::vector<miso_b200_log_record> log;
  std::vector<double> stp;
  for (int attempt = 0; attempt < 2; ++attempt) {
    log.assign(want_log ? n * size_t(log_cap) : 0, miso_b200_log_record{});
    stp.assign(full ? n * 2 * size_t(stp_cap) : 0, 0.0);
    Device::check(miso_b200_simulate_batch_sharded(
        all.contexts(), all.size(), &c, static_cast<int>(n), static_cast<int>(n), nullptr,
        optsta ? sc.data() : nullptr,
        ta.offsets.data(), ta.arrival.data(), ta.base.data(), ta.speeds.data(), ta.mem.data(),
        ta.qos.data(), ta.inst.data(), seeds.data(), met.data(), full ? job_out.data() : nullptr,
        want_log ? log.data() : nullptr, log_cap, full ? stp.data() : nullptr, stp_cap,
        full ? 0u : MISO_B200_SIM_JCT_ONLY));
    int64_t need_log = 0, need_stp = 0;
    for (const auto& m : met) {
      need_log = std::max<int64_t>(need_log, m.log_records);
      need_stp = std::max<int64_t>(need_stp, m.stp_points);
    }
    if ((!want_log || need_log <= log_cap) && (!full || need_stp <= stp_cap)) break;
    log_cap = std::max(log_cap, need_log);  // rerun once with exact capacities
    stp_cap = std::max(stp_cap, need_stp);
  }
  out.reserve(n);
  for (size_t i = 0; i < n; ++i) {
    if (met[i].status) detail::throw_status(met[i].status, met[i].detail, traces[i]);
    const int64_t* jo = full ? job_out.data() + i * size_t(max_jobs) * MISO_B200_JOB_OUT_FIELDS : nullptr;
    std::vector<std::string> ids;
    if (full) ids = detail::job_ids(*traces[i], jo, met[i].job_count);
    out.push_back(detail::make_report(*traces[i], options.policy, met[i], jo, full ? &ids : nullptr,
                                      full ? stp.data() + i * 2 * size_t(stp_cap) : nullptr,
                                      full ? std::min<int64_t>(met[i].stp_points, stp_cap) : 0));
    if (want_log)
      detail::render_log(ids, log.data() + i * size_t(log_cap),
                         std::min<int64_t>(met[i].log_records, log_cap), *options.event_log);
  }
  return out;
}

// Drop-in for run_simulation (sim.hpp:976-979).
inline MetricsReport run_simulation(const JobTrace& trace, const SimOptions& options) {
  return b200::run_simulation_batch({&trace}, options).front();
}

// Drop-in for the 6-argument overload (sim.hpp:981-992).
inline MetricsReport run_simulation(const JobTrace& trace, int cluster_size, Policy policy,
                                    const OverheadSpec& overheads, const PredictorSpec& predictor,
                                    const std::optional<PartitionConfig>& static_partition =
                                        std::nullopt) {
  SimOptions opt;
  opt.policy = policy;
  opt.cluster_size = cluster_size;
  opt.overheads = overheads;
  opt.predictor = predictor;
  opt.static_partition = static_partition;
  return b200::run_simulation(trace, opt);
}

// best_static_partition for many traces: every (trace, feasible candidate) pair is one optsta
// simulation of a single launch (JCT-only: the search reads avg_jct_s alone). Same table,
// choice (strict <, first in catalog order) and InfeasibleError cases as sim.hpp:1031-1066.
inline std::vector<StaticSearchResult> best_static_partition_batch(
    const std::vector<const JobTrace*>& traces, int cluster_size, const OverheadSpec& overheads,
    const PartitionCatalog& catalog = default_catalog()) {
  std::vector<const JobTrace*> task_trace;
  std::vector<std::optional<PartitionConfig>> parts;
  std::vector<std::vector<int>> task_of(traces.size(), std::vector<int>(catalog.entries.size(), -1));
  for (size_t ti = 0; ti < traces.size(); ++ti) {
    int need = 0;  // largest minimal slice kind over all jobs
    for (const auto& t : traces[ti]->jobs) {
      auto k = min_slice_for(t.profile.mem_demand_gb,
                             t.profile.qos_min_slice ? gpc_count(*t.profile.qos_min_slice) : 0);
      if (!k) throw InfeasibleError("job '" + t.profile.job_id + "' fits no slice kind");
      need = std::max(need, slice_index(*k));
    }
    for (size_t e = 0; e < catalog.entries.size(); ++e) {
      const auto& cand = catalog.entries[e];
      if (slice_index(cand.slices_desc().front()) >= need) {
        task_of[ti][e] = static_cast<int>(task_trace.size());
        task_trace.push_back(traces[ti]);
        parts.emplace_back(cand);
      }
    }
  }
  SimOptions opt;
  opt.policy = Policy::optsta;
  opt.cluster_size = cluster_size;
  opt.overheads = overheads;
  opt.catalog = catalog;
  std::vector<MetricsReport> reps;
  if (!task_trace.empty()) reps = b200::run_simulation_batch(task_trace, opt, nullptr, &parts, false);
  std::vector<StaticSearchResult> out(traces.size());
  for (size_t ti = 0; ti < traces.size(); ++ti) {
    StaticSearchResult& res = out[ti];
    double best = std::numeric_limits<double>::infinity();
    bool found = false;
    for (size_t e = 0; e < catalog.entries.size(); ++e) {
      const int t = task_of[ti][e];
      const double jct = t < 0 ? std::numeric_limits<double>::infinity()
                               : reps[static_cast<size_t>(t)].avg_jct_s;
      res.table.emplace_back(catalog.entries[e], jct);
      if (jct < best) {
        best = jct;
        res.chosen = catalog.entries[e];
        found = true;
      }
    }
    if (!found) throw InfeasibleError("no static partition can host this trace");
  }
  return out;
}

// run_trial_unit's use of best_static_partition (experiment.hpp:337 reads only .chosen): the
// same chosen entries from one pruned launch (MISO_B200_SIM_PRUNE). Every trace is uploaded
// once, its two likeliest winners (most GPCs, then slice count nearest 3) run first, and every
// other candidate stops once its JCT sum provably exceeds a completed candidate's
// (miso_b200_simulate_batch_pruned). Traces with multi-instance jobs take the full search.
// Error-behaviour divergence (by design): a candidate stopped early never reaches a later
// SimInvariantError or event-budget exhaustion, so where the reference's best_static_partition
// (sim.hpp:1031-1066) would throw from a losing candidate, this returns the chosen entry.
// Callers that need the reference's throw-on-any-candidate behaviour use
// best_static_partition (full search), which reports every candidate's status.
inline std::vector<PartitionConfig> best_static_chosen_batch(
    const std::vector<const JobTrace*>& traces, int cluster_size, const OverheadSpec& overheads,
    const PartitionCatalog& catalog = default_catalog()) {
  std::vector<PartitionConfig> out;
  bool multi = false;
  for (const JobTrace* t : traces)
    for (const TraceJob& j : t->jobs) multi = multi || j.profile.instance_count > 1;
  if (multi) {
    for (auto& r : best_static_partition_batch(traces, cluster_size, overheads, catalog))
      out.push_back(r.chosen);
    return out;
  }
  const size_t E = catalog.entries.size();
  std::vector<int> prio(E);
  for (size_t e = 0; e < E; ++e) prio[e] = static_cast<int>(e);
  auto gpcs = [&](size_t e) {
    int g = 0;
    for (int k = 0; k < 5; ++k) g += catalog.entries[e].counts()[static_cast<size_t>(k)] * gpc_count(static_cast<Slice>(k));
    return g;
  };
  auto nsl = [&](size_t e) {
    int n = 0;
    for (int k = 0; k < 5; ++k) n += catalog.entries[e].counts()[static_cast<size_t>(k)];
    return n;
  };
  std::stable_sort(prio.begin(), prio.end(), [&](int a, int b) {
    const int ga = gpcs(size_t(a)), gb = gpcs(size_t(b));
    if (ga != gb) return ga > gb;
    return std::abs(nsl(size_t(a)) - 3) < std::abs(nsl(size_t(b)) - 3);
  });
  SimOptions opt;
  opt.policy = Policy::optsta;
  opt.cluster_size = cluster_size;
  opt.overheads = overheads;
  opt.catalog = catalog;
  opt.static_partition = catalog.entries.front();
  detail::TraceArrays ta;
  std::vector<int32_t> probe_tt, rest_tt;
  std::vector<uint8_t> probe_sc, rest_sc;
  std::vector<int> probe_e, rest_e;
  for (size_t ti = 0; ti < traces.size(); ++ti) {
    detail::validate(*traces[ti], opt);
    int need = 0;  // largest minimal slice kind over all jobs (sim.hpp:1036-1041)
    for (const auto& t : traces[ti]->jobs) {
      auto k = min_slice_for(t.profile.mem_demand_gb,
                             t.profile.qos_min_slice ? gpc_count(*t.profile.qos_min_slice) : 0);
      if (!k) throw InfeasibleError("job '" + t.profile.job_id + "' fits no slice kind");
      need = std::max(need, slice_index(*k));
    }
    ta.add(*traces[ti]);
    int taken = 0;
    for (int e : prio) {
      const auto& cand = catalog.entries[size_t(e)];
      if (slice_index(cand.slices_desc().front()) < need) continue;
      const bool probe = taken++ < 2;
      (probe ? probe_tt : rest_tt).push_back(static_cast<int32_t>(ti));
      (probe ? probe_e : rest_e).push_back(e);
      for (int k = 0; k < 5; ++k)
        (probe ? probe_sc : rest_sc).push_back(cand.counts()[static_cast<size_t>(k)]);
    }
  }
  probe_tt.insert(probe_tt.end(), rest_tt.begin(), rest_tt.end());
  probe_sc.insert(probe_sc.end(), rest_sc.begin(), rest_sc.end());
  probe_e.insert(probe_e.end(), rest_e.begin(), rest_e.end());
  const size_t n = probe_tt.size();
  std::vector<miso_b200_sim_metrics> met(n);
  if (n) {
    std::vector<uint64_t> seeds(n, opt.predictor.rng_seed);
    const miso_b200_sim_options c = detail::to_c(opt);
    AllDevices all(catalog);
    Device::check(miso_b200_simulate_batch_sharded(
        all.contexts(), all.size(), &c, static_cast<int>(n), static_cast<int>(traces.size()), probe_tt.data(),
        probe_sc.data(), ta.offsets.data(), ta.arrival.data(), ta.base.data(), ta.speeds.data(),
        ta.mem.data(), ta.qos.data(), nullptr, seeds.data(), met.data(), nullptr, nullptr, 0,
        nullptr, 0, MISO_B200_SIM_JCT_ONLY | MISO_B200_SIM_PRUNE));
  }
  std::vector<std::vector<double>> table(traces.size(),
                                         std::vector<double>(E, std::numeric_limits<double>::infinity()));
  for (size_t i = 0; i < n; ++i) {
    if (met[i].status && met[i].status != MISO_B200_SIM_PRUNED)
      detail::throw_status(met[i].status, met[i].detail, traces[size_t(probe_tt[i])]);
    table[size_t(probe_tt[i])][size_t(probe_e[i])] = met[i].avg_jct_s;
  }
  for (size_t ti = 0; ti < traces.size(); ++ti) {
    double best = std::numeric_limits<double>::infinity();
    std::optional<PartitionConfig> chosen;
    for (size_t e = 0; e < E; ++e)  // first minimum in catalog order (sim.hpp:1058)
      if (table[ti][e] < best) {
        best = table[ti][e];
        chosen = catalog.entries[e];
      }
    if (!chosen) throw InfeasibleError("no static partition can host this trace");
    out.push_back(*chosen);
  }
  return out;
}

// Drop-in for best_static_partition (sim.hpp:1031-1066).
inline StaticSearchResult best_static_partition(const JobTrace& trace, int cluster_size,
                                                const OverheadSpec& overheads,
                                                const PartitionCatalog& catalog = default_catalog()) {
  return b200::best_static_partition_batch({&trace}, cluster_size, overheads, catalog).front();
}

}  // namespace b200
}  // namespace miso
