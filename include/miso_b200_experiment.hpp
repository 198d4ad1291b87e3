// miso_b200_experiment.hpp -- run_experiment_in_memory (experiment.hpp:364-415) on the B200:
// instead of a CPU worker pool over (sweep point, trial) units, every policy of a sweep point
// runs all of that point's trials in ONE device launch (one warp per simulation), and the
// best-static search of all trials is one more launch (every (trial, candidate) pair). Rows are
// assembled exactly as run_trial_unit (experiment.hpp:299-362) does, so the reference's own
// write_csv / summarize / run_experiment file writers produce byte-identical output.
// Header-only; include after "miso/experiment.hpp".
#pragma once

#include <fstream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "miso/experiment.hpp"
#include "miso_b200_sim.hpp"

namespace miso {
namespace b200 {

// Trace generation for many seeds on the device (miso_b200_generate_traces_device_host: one
// warp per trace, glibc-exact libm restatements), identical to generate_trace(spec) per seed
// (job ids "j<i>", workload.hpp:97-114).
inline std::vector<JobTrace> generate_traces(const TraceSpec& spec, const std::vector<uint64_t>& seeds) {
  validate_trace_spec(spec);
  const size_t n = seeds.size(), J = static_cast<size_t>(spec.job_count);
  std::vector<double> a(n * J), d(n * J), sp(n * J * 5);
  std::vector<int> mem(n * J);
  const int kind = spec.duration_dist.kind == DurationDist::Kind::lognormal ? 0
                   : spec.duration_dist.kind == DurationDist::Kind::fixed   ? 1
                                                                            : 2;
  if (n) {
    Device& dev = Device::get();
    std::lock_guard<std::mutex> lock(dev.mu());
    Device::check(miso_b200_generate_traces_device_host(
        dev.ctx(), seeds.data(), static_cast<int>(n), spec.job_count, spec.lambda_s,
        spec.max_duration_s, kind, spec.duration_dist.sigma, spec.duration_dist.fixed_s,
        spec.duration_dist.lo_s, spec.duration_dist.hi_s, a.data(), d.data(), sp.data(),
        mem.data()));
  }
  std::vector<JobTrace> out(n);
  for (size_t r = 0; r < n; ++r) {
    JobTrace& t = out[r];
    t.spec = spec;
    t.spec.seed = seeds[r];
    t.jobs.resize(J);
    for (size_t i = 0; i < J; ++i) {
      TraceJob& j = t.jobs[i];
      const size_t o = r * J + i;
      j.arrival_s = a[o];
      JobProfile& p = j.profile;
      p.job_id = "j" + std::to_string(i);
      p.base_duration_s = d[o];
      for (int k = 0; k < 5; ++k) p.speed_table.v[static_cast<size_t>(k)] = sp[5 * o + static_cast<size_t>(k)];
      p.mem_demand_gb = mem[o];
      // make_synthetic_profile's placeholder solo-run rates (profiles.hpp:460-463)
      p.mps_rates[0] = 1.0;
      p.mps_rates[1] = std::clamp(interp_speed(p.speed_table, 3.5), kSpeedFloor, 1.0);
      p.mps_rates[2] = p.speed_table[Slice::k1g];
    }
  }
  return out;
}

// Drop-in for generate_trace (workload.hpp:97-114), on the device.
inline JobTrace generate_trace(const TraceSpec& spec) {
  return std::move(generate_traces(spec, {spec.seed}).front());
}

// Drop-in for run_experiment_in_memory (experiment.hpp:364-415). config.workers is ignored
// (the device runs every trial of a sweep point concurrently); results do not depend on it,
// as in the reference (experiment_test ParallelWorkersMatchSerialByteForByte).
inline ExperimentResult run_experiment_in_memory(const ExperimentConfig& config) {
  validate_experiment_config(config);
  std::optional<JobTrace> fixed;
  if (!config.trace_path.empty()) fixed = load_trace(config.trace_path);

  const std::vector<double> values =
      config.sweep_param.empty() ? std::vector<double>{0} : config.sweep_values;
  std::vector<Policy> run_policies = config.policies;
  bool had_nopart = false;
  for (Policy p : run_policies) had_nopart |= (p == Policy::nopart);
  if (!had_nopart) run_policies.insert(run_policies.begin(), Policy::nopart);  // baseline
  bool want_optsta = false;
  for (Policy p : run_policies) want_optsta |= (p == Policy::optsta);

  ExperimentResult res;
  res.config = config;
  const int T = config.trials;
  for (double value : values) {
    // run_trial_unit's per-point settings (experiment.hpp:303-311)
    OverheadSpec overheads = config.overheads;
    PredictorSpec predictor = config.predictor;
    TraceSpec spec = config.trace_spec;
    if (!config.sweep_param.empty()) {
      if (config.sweep_param == "checkpoint_restart_s") overheads.checkpoint_restart_s = value;
      else if (config.sweep_param == "target_mae") predictor.target_mae = value;
      else spec.lambda_s = value;
    }
    std::vector<uint64_t> seeds(static_cast<size_t>(T));
    for (int t = 0; t < T; ++t) seeds[static_cast<size_t>(t)] = config.base_seed + static_cast<uint64_t>(t);
    std::vector<JobTrace> generated;
    std::vector<const JobTrace*> traces;
    if (fixed) {
      traces.assign(static_cast<size_t>(T), &*fixed);
    } else {
      generated = b200::generate_traces(spec, seeds);
      for (const auto& g : generated) traces.push_back(&g);
    }
    std::vector<std::optional<PartitionConfig>> static_part(static_cast<size_t>(T));
    if (want_optsta) {
      // run_trial_unit reads only .chosen (experiment.hpp:337): the pruned chosen-only search
      auto st = b200::best_static_chosen_batch(traces, config.cluster_size, overheads);
      for (int t = 0; t < T; ++t) static_part[static_cast<size_t>(t)] = st[static_cast<size_t>(t)];
    }
    std::map<std::string, std::vector<MetricsReport>> reports;
    for (Policy p : run_policies) {
      SimOptions opt;
      opt.policy = p;
      opt.cluster_size = config.cluster_size;
      opt.overheads = overheads;
      opt.predictor = predictor;
      opt.reprofile_drift_threshold = config.reprofile_drift_threshold;
      auto reps = b200::run_simulation_batch(traces, opt, &seeds,
                                       p == Policy::optsta ? &static_part : nullptr, true);
      for (int t = 0; t < T; ++t) reps[static_cast<size_t>(t)].seed = seeds[static_cast<size_t>(t)];
      reports[policy_label(p)] = std::move(reps);
    }
    const auto& base = reports.at("nopart");
    for (int t = 0; t < T; ++t) {
      const MetricsReport& b = base[static_cast<size_t>(t)];
      for (Policy p : config.policies) {
        TrialRow row;
        row.sweep_param = config.sweep_param.empty() ? "none" : config.sweep_param;
        row.sweep_value = value;
        row.trial = t;
        row.seed = seeds[static_cast<size_t>(t)];
        row.report = reports.at(policy_label(p))[static_cast<size_t>(t)];
        row.jct_norm = row.report.avg_jct_s / b.avg_jct_s;
        row.makespan_norm = row.report.makespan_s / b.makespan_s;
        row.stp_norm = b.stp_time_avg > 0 ? row.report.stp_time_avg / b.stp_time_avg : 0;
        res.rows.push_back(std::move(row));
      }
    }
  }
  return res;
}

// Drop-in for run_experiment (experiment.hpp:417-431): the trials on the device, then the
// reference's own CSV and summary writers.
inline ExperimentResult run_experiment(const ExperimentConfig& config) {
  ExperimentResult res = b200::run_experiment_in_memory(config);
  {
    std::ofstream out(config.csv_path);
    if (!out) throw IoError("cannot open csv output: " + config.csv_path);
    write_csv(res, out);
  }
  {
    std::ofstream out(config.json_path);
    if (!out) throw IoError("cannot open json output: " + config.json_path);
    out << summarize(res).dump(2) << '\n';
    if (!out) throw IoError("json write failed");
  }
  return res;
}

// Drop-in for optsta_search (experiment.hpp:434-446): the offline static-partition search on
// the experiment's trace (trial 0 seed), trace generation and every candidate on the device.
inline StaticSearchResult optsta_search(const ExperimentConfig& config) {
  validate_experiment_config(config);
  JobTrace trace;
  if (!config.trace_path.empty()) {
    trace = load_trace(config.trace_path);
  } else {
    TraceSpec spec = config.trace_spec;
    spec.seed = config.base_seed;
    trace = b200::generate_trace(spec);
  }
  return b200::best_static_partition(trace, config.cluster_size, config.overheads);
}

}  // namespace b200
}  // namespace miso
