// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference headers
// (/root/reference/proj/include, included read-only via -I by oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY. The resulting oracle/_ref/libmiso_ref.so is the reference
// itself, callable from Python tests and from bench.py's CPU legs (cpu_baseline and
// --impl reference). Nothing here is shipped or measured as the product.
//
// Each entry point names the reference call it drives.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "miso/optimizer.hpp"
#include "miso/profiles.hpp"
#include "miso/sim.hpp"
#include "miso/topology.hpp"
#include "miso/workload.hpp"

namespace {

int catalog_index(const miso::PartitionCatalog& cat, const miso::PartitionConfig& p) {
  for (size_t i = 0; i < cat.entries.size(); ++i)
    if (cat.entries[i] == p) return static_cast<int>(i);
  return -1;
}

template <class F>
void parallel_for(size_t n, int nthreads, size_t chunk, F&& f) {
  if (nthreads <= 1 || n <= chunk) {
    f(size_t{0}, n);
    return;
  }
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&]() {
      for (;;) {
        size_t b = next.fetch_add(chunk);
        if (b >= n) break;
        f(b, std::min(n, b + chunk));
      }
    });
  for (auto& th : pool) th.join();
}

const miso::LinearMap& default_model() {
  static const miso::LinearMap m =
      miso::fit_small_slice_model(miso::make_training_corpus(3000, 0x5eedull));
  return m;
}

}  // namespace

extern "C" {

// topology.hpp:205-208 default_catalog(): counts per entry in catalog order.
int ref_catalog(uint8_t* counts /* [36][5] */) {
  const auto& cat = miso::default_catalog();
  for (size_t e = 0; e < cat.entries.size(); ++e)
    for (int k = 0; k < 5; ++k) counts[e * 5 + k] = cat.entries[e].counts()[k];
  return static_cast<int>(cat.entries.size());
}

// optimizer.hpp:62-115 optimize_partition over a packed batch (speeds: sum(m) x 5, kind order
// 1g..7g; offsets: n+1). entry = default-catalog index, -1 = nullopt, -2 = invalid_argument.
void ref_optimize_batch(const double* speeds, const uint32_t* offsets, size_t n, int nthreads,
                        int16_t* entry, uint8_t* place, double* obj) {
  const auto& cat = miso::default_catalog();
  parallel_for(n, nthreads, 4096, [&](size_t b, size_t e) {
    std::vector<miso::JobSpeeds> jobs;
    for (size_t i = b; i < e; ++i) {
      uint32_t o = offsets[i];
      size_t m = offsets[i + 1] - o;
      jobs.resize(m);
      for (size_t j = 0; j < m; ++j) {
        jobs[j].job_id = "j" + std::to_string(j);
        for (int k = 0; k < 5; ++k) jobs[j].speeds.v[k] = speeds[(o + j) * 5 + k];
      }
      try {
        auto r = miso::optimize_partition(jobs, cat);
        if (!r) {
          entry[i] = -1;
          obj[i] = 0;
          continue;
        }
        entry[i] = static_cast<int16_t>(catalog_index(cat, r->partition));
        obj[i] = r->objective;
        for (size_t j = 0; j < m; ++j) place[o + j] = static_cast<uint8_t>(r->assignments[j].slice);
      } catch (const std::invalid_argument&) {
        entry[i] = -2;
        obj[i] = 0;
      }
    }
  });
}

// acceptance_test.cpp:72-85 generator (reference DetRng), the config-2 input stream.
size_t ref_gen_mixes(uint64_t seed, size_t n, double* speeds, uint32_t* offsets, size_t max_jobs) {
  miso::DetRng rng(seed);
  size_t jobs = 0;
  offsets[0] = 0;
  for (size_t t = 0; t < n; ++t) {
    int m = 1 + rng.index(7);
    if (jobs + m > max_jobs) return static_cast<size_t>(-1);
    for (int i = 0; i < m; ++i) {
      double f4 = rng.uniform(0.2, 1.0);
      double f3 = rng.uniform(0.15, f4);
      double f2 = rng.uniform(0.1, f3);
      double f1 = rng.uniform(0.05, f2);
      if (rng.uniform01() < 0.25) f1 = 0.0;
      double* v = speeds + 5 * (jobs + i);
      v[0] = f1; v[1] = f2; v[2] = f3; v[3] = f4; v[4] = 1.0;
    }
    jobs += m;
    offsets[t + 1] = static_cast<uint32_t>(jobs);
  }
  return jobs;
}

// Config-3 input stream: make_synthetic_profile (profiles.hpp:443-465) from
// DetRng(mix_seed(seed, 0x50)). truth3 = f7,f4,f3; small2 = f2,f1 (may be null).
void ref_gen_profiles(uint64_t seed, size_t n, double* truth3, double* small2) {
  miso::DetRng rng(miso::mix_seed(seed, 0x50));
  for (size_t i = 0; i < n; ++i) {
    auto p = miso::make_synthetic_profile(rng, "p");
    truth3[3 * i + 0] = p.speed_table.v[4];
    truth3[3 * i + 1] = p.speed_table.v[3];
    truth3[3 * i + 2] = p.speed_table.v[2];
    if (small2) {
      small2[2 * i] = p.speed_table.v[1];
      small2[2 * i + 1] = p.speed_table.v[0];
    }
  }
}

// sim.hpp:894-898 shared default model.
void ref_default_model(double* w2, double* w1) {
  const auto& m = default_model();
  for (int i = 0; i < 4; ++i) {
    w2[i] = m.w_2g[i];
    w1[i] = m.w_1g[i];
  }
}

// profiles.hpp:106-113, 151-167, 214-253, 370-384: pad_to_seven -> build_mps_matrix ->
// predict_mig_speeds(nonce) -> extrapolate_small_slices, per group of `cpg` real columns.
// Column j is column j%cpg of group j/cpg with nonce first_nonce + j/cpg.
// out5 per column in kind order 1g..7g.
void ref_predict_batch(const double* truth3, size_t ncols, int cpg, uint64_t first_nonce,
                       uint64_t rng_seed, int noisy, double target_mae, int nthreads,
                       double* out5) {
  miso::PredictorSpec spec;
  spec.mode = noisy ? miso::PredictorSpec::Mode::noisy : miso::PredictorSpec::Mode::oracle;
  spec.target_mae = target_mae;
  spec.rng_seed = rng_seed;
  const auto& model = default_model();
  size_t groups = (ncols + cpg - 1) / cpg;
  static const char* kIds[7] = {"c0", "c1", "c2", "c3", "c4", "c5", "c6"};
  parallel_for(groups, nthreads, 1024, [&](size_t gb, size_t ge) {
    std::vector<miso::JobProfile> profs;
    for (size_t g = gb; g < ge; ++g) {
      size_t j0 = g * cpg, j1 = std::min(ncols, j0 + cpg);
      profs.clear();
      for (size_t j = j0; j < j1; ++j) {
        miso::JobProfile p;
        p.job_id = kIds[j - j0];
        p.base_duration_s = 1;
        p.mem_demand_gb = 5;
        p.speed_table.v = {0.1, 0.2, truth3[3 * j + 2], truth3[3 * j + 1], truth3[3 * j + 0]};
        p.mps_rates = {1.0, 0.7, 0.4};
        profs.push_back(p);
      }
      auto mps = miso::build_mps_matrix(miso::pad_to_seven(profs));
      auto mig = miso::predict_mig_speeds(mps, profs, spec, first_nonce + g);
      auto small = miso::extrapolate_small_slices(mig, model);
      for (size_t j = j0; j < j1; ++j) {
        int c = static_cast<int>(j - j0);
        const auto& s = small.at(kIds[c]);
        double* o = out5 + 5 * j;
        o[0] = s.f1;
        o[1] = s.f2;
        o[2] = mig.values[2][c];
        o[3] = mig.values[1][c];
        o[4] = mig.values[0][c];
      }
    }
  });
}

// profiles.hpp:193-205
double ref_perturb_speed(double truth, double target_mae, uint64_t entry_seed) {
  return miso::detail::perturb_speed(truth, target_mae, entry_seed);
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t tag) { return miso::mix_seed(seed, tag); }

// topology.hpp:227-252
int ref_max_spare_slice_for(const int* kinds, int m) {
  std::vector<miso::Slice> v;
  for (int i = 0; i < m; ++i) v.push_back(static_cast<miso::Slice>(kinds[i]));
  auto r = miso::max_spare_slice_for(miso::default_catalog(), v);
  return r ? static_cast<int>(*r) : -1;
}

// workload.hpp:97-114 generate_trace. Arrays sized job_count; speeds5 kind order 1g..7g.
void ref_gen_trace(uint64_t seed, int job_count, double lambda_s, double max_duration_s,
                   double sigma, double* arrival_s, double* duration_s, double* speeds5,
                   int* mem_gb) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.lambda_s = lambda_s;
  spec.max_duration_s = max_duration_s;
  spec.duration_dist.sigma = sigma;
  spec.seed = seed;
  auto tr = miso::generate_trace(spec);
  for (int i = 0; i < job_count; ++i) {
    const auto& j = tr.jobs[i];
    arrival_s[i] = j.arrival_s;
    duration_s[i] = j.profile.base_duration_s;
    for (int k = 0; k < 5; ++k) speeds5[5 * i + k] = j.profile.speed_table.v[k];
    mem_gb[i] = j.profile.mem_demand_gb;
  }
}

struct RefSimOut {
  int completed, job_count, completed_count, repartitions, migrations, mps_sessions;
  double avg_jct_s, makespan_s, stp_time_avg;
  double queue_frac, mps_frac, checkpoint_frac, run_frac, idle_frac;
  int64_t stp_points;
};

// sim.hpp:976-979 run_simulation(generate_trace(spec), opt). policy: 0 nopart 1 optsta
// 2 oracle 3 miso. static_entry: default-catalog index for optsta. Event log text is written
// to log_buf (truncated to log_cap; returns full length) when log_buf != null.
int64_t ref_simulate(uint64_t seed, int job_count, double lambda_s, double max_duration_s,
                     double sigma, int cluster_size, int policy, double mig_reconfig_s,
                     double checkpoint_restart_s, double mps_window_s, double interference,
                     int noisy, double target_mae, int static_entry, RefSimOut* out,
                     char* log_buf, int64_t log_cap) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.lambda_s = lambda_s;
  spec.max_duration_s = max_duration_s;
  spec.duration_dist.sigma = sigma;
  spec.seed = seed;
  auto trace = miso::generate_trace(spec);
  miso::SimOptions opt;
  opt.policy = static_cast<miso::Policy>(policy);
  opt.cluster_size = cluster_size;
  opt.overheads.mig_reconfig_s = mig_reconfig_s;
  opt.overheads.checkpoint_restart_s = checkpoint_restart_s;
  opt.overheads.mps_window_s = mps_window_s;
  opt.overheads.interference = interference;
  opt.predictor.mode = noisy ? miso::PredictorSpec::Mode::noisy : miso::PredictorSpec::Mode::oracle;
  opt.predictor.target_mae = target_mae;
  opt.predictor.rng_seed = seed;  // experiment.hpp:305
  if (static_entry >= 0) opt.static_partition = miso::default_catalog().entries[static_entry];
  std::ostringstream log;
  if (log_buf) opt.event_log = &log;
  auto r = miso::run_simulation(trace, opt);
  out->completed = r.completed;
  out->job_count = r.job_count;
  out->completed_count = r.completed_count;
  out->repartitions = r.repartitions;
  out->migrations = r.migrations;
  out->mps_sessions = r.mps_sessions;
  out->avg_jct_s = r.avg_jct_s;
  out->makespan_s = r.makespan_s;
  out->stp_time_avg = r.stp_time_avg;
  out->queue_frac = r.queue_frac;
  out->mps_frac = r.mps_frac;
  out->checkpoint_frac = r.checkpoint_frac;
  out->run_frac = r.run_frac;
  out->idle_frac = r.idle_frac;
  out->stp_points = static_cast<int64_t>(r.stp_series.size());
  if (!log_buf) return 0;
  std::string s = log.str();
  size_t n = std::min<size_t>(s.size(), static_cast<size_t>(log_cap));
  std::memcpy(log_buf, s.data(), n);
  return static_cast<int64_t>(s.size());
}

// run_simulation on an explicit trace (arrays; job ids "j<i>", qos kind -1 = none).
int64_t ref_simulate_trace(int job_count, const double* arrival_s, const double* duration_s,
                           const double* speeds5, const int* mem_gb, const int* qos_kind,
                           uint64_t seed, int cluster_size, int policy, double mig_reconfig_s,
                           double checkpoint_restart_s, double mps_window_s, double interference,
                           int noisy, double target_mae, uint64_t rng_seed, int static_entry,
                           RefSimOut* out, char* log_buf, int64_t log_cap, double* stp_series,
                           int64_t stp_cap) {
  miso::JobTrace trace;
  trace.spec.job_count = job_count;
  trace.spec.seed = seed;
  for (int i = 0; i < job_count; ++i) {
    miso::TraceJob j;
    j.arrival_s = arrival_s[i];
    j.profile.job_id = "j" + std::to_string(i);
    j.profile.base_duration_s = duration_s[i];
    for (int k = 0; k < 5; ++k) j.profile.speed_table.v[k] = speeds5[5 * i + k];
    j.profile.mem_demand_gb = mem_gb[i];
    if (qos_kind[i] >= 0) j.profile.qos_min_slice = static_cast<miso::Slice>(qos_kind[i]);
    j.profile.mps_rates = {1.0, 0.7, 0.4};
    trace.jobs.push_back(j);
  }
  miso::SimOptions opt;
  opt.policy = static_cast<miso::Policy>(policy);
  opt.cluster_size = cluster_size;
  opt.overheads.mig_reconfig_s = mig_reconfig_s;
  opt.overheads.checkpoint_restart_s = checkpoint_restart_s;
  opt.overheads.mps_window_s = mps_window_s;
  opt.overheads.interference = interference;
  opt.predictor.mode = noisy ? miso::PredictorSpec::Mode::noisy : miso::PredictorSpec::Mode::oracle;
  opt.predictor.target_mae = target_mae;
  opt.predictor.rng_seed = rng_seed;
  if (static_entry >= 0) opt.static_partition = miso::default_catalog().entries[static_entry];
  std::ostringstream log;
  if (log_buf) opt.event_log = &log;
  miso::MetricsReport r;
  try {
    r = miso::run_simulation(trace, opt);
  } catch (const std::exception& e) {
    out->completed = -1;
    return -1;
  }
  out->completed = r.completed;
  out->job_count = r.job_count;
  out->completed_count = r.completed_count;
  out->repartitions = r.repartitions;
  out->migrations = r.migrations;
  out->mps_sessions = r.mps_sessions;
  out->avg_jct_s = r.avg_jct_s;
  out->makespan_s = r.makespan_s;
  out->stp_time_avg = r.stp_time_avg;
  out->queue_frac = r.queue_frac;
  out->mps_frac = r.mps_frac;
  out->checkpoint_frac = r.checkpoint_frac;
  out->run_frac = r.run_frac;
  out->idle_frac = r.idle_frac;
  out->stp_points = static_cast<int64_t>(r.stp_series.size());
  if (stp_series)
    for (size_t i = 0; i < r.stp_series.size() && static_cast<int64_t>(i) < stp_cap; ++i) {
      stp_series[2 * i] = r.stp_series[i].first;
      stp_series[2 * i + 1] = r.stp_series[i].second;
    }
  if (!log_buf) return 0;
  std::string s = log.str();
  size_t n = std::min<size_t>(s.size(), static_cast<size_t>(log_cap));
  std::memcpy(log_buf, s.data(), n);
  return static_cast<int64_t>(s.size());
}

// best_static_partition (sim.hpp:1031-1066) on an explicit trace; table[36] avg JCT per entry.
int ref_best_static(int job_count, const double* arrival_s, const double* duration_s,
                    const double* speeds5, const int* mem_gb, int cluster_size,
                    double mig_reconfig_s, double checkpoint_restart_s, double mps_window_s,
                    double interference, double* table) {
  miso::JobTrace trace;
  trace.spec.job_count = job_count;
  for (int i = 0; i < job_count; ++i) {
    miso::TraceJob j;
    j.arrival_s = arrival_s[i];
    j.profile.job_id = "j" + std::to_string(i);
    j.profile.base_duration_s = duration_s[i];
    for (int k = 0; k < 5; ++k) j.profile.speed_table.v[k] = speeds5[5 * i + k];
    j.profile.mem_demand_gb = mem_gb[i];
    j.profile.mps_rates = {1.0, 0.7, 0.4};
    trace.jobs.push_back(j);
  }
  miso::OverheadSpec o;
  o.mig_reconfig_s = mig_reconfig_s;
  o.checkpoint_restart_s = checkpoint_restart_s;
  o.mps_window_s = mps_window_s;
  o.interference = interference;
  auto res = miso::best_static_partition(trace, cluster_size, o);
  for (size_t e = 0; e < res.table.size(); ++e) table[e] = res.table[e].second;
  return catalog_index(miso::default_catalog(), res.chosen);
}

// One trial of the config-4 experiment (experiment.hpp:299-360 run_trial_unit without the
// file/JSON plumbing): generate_trace(seed) -> nopart, best_static_partition + optsta, miso
// (noisy predictor, rng_seed = seed). out[0..2] = avg JCT nopart/optsta/miso; returns the
// chosen static catalog index.
int ref_trial(uint64_t seed, int job_count, double lambda_s, int cluster_size, double target_mae,
              double* out) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.lambda_s = lambda_s;
  spec.seed = seed;
  auto trace = miso::generate_trace(spec);
  miso::OverheadSpec o;
  miso::PredictorSpec ps;
  ps.mode = miso::PredictorSpec::Mode::noisy;
  ps.target_mae = target_mae;
  ps.rng_seed = seed;
  out[0] = miso::run_simulation(trace, cluster_size, miso::Policy::nopart, o, ps).avg_jct_s;
  auto st = miso::best_static_partition(trace, cluster_size, o);
  out[1] = miso::run_simulation(trace, cluster_size, miso::Policy::optsta, o, ps, st.chosen).avg_jct_s;
  out[2] = miso::run_simulation(trace, cluster_size, miso::Policy::miso, o, ps).avg_jct_s;
  return catalog_index(miso::default_catalog(), st.chosen);
}

// save_trace (workload.hpp:149-170) text of generate_trace({job_count, lambda_s, seed}).
// Returns the length (the text is truncated to cap).
size_t ref_trace_text(uint64_t seed, int job_count, double lambda_s, char* buf, size_t cap) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.lambda_s = lambda_s;
  spec.seed = seed;
  std::ostringstream o;
  miso::save_trace(miso::generate_trace(spec), o);
  const std::string t = o.str();
  std::memcpy(buf, t.data(), std::min(cap, t.size()));
  return t.size();
}

// load_trace (workload.hpp:172-243) of `text`: 0 if it parses (job_count written), else the
// ParseError line and its what() text in msg.
int ref_load_trace(const char* text, int* job_count, char* msg, size_t cap) {
  std::istringstream in{std::string(text)};
  try {
    auto t = miso::load_trace(in);
    *job_count = static_cast<int>(t.jobs.size());
    return 0;
  } catch (const miso::ParseError& e) {
    std::snprintf(msg, cap, "%s", e.what());
    return e.line() > 0 ? e.line() : -1;
  }
}

// parse_profile_record (profiles.hpp:564-568) of `line` at `lineno`, then
// format_profile_record (:493-495) of the result: 0 and the record text in out, or the
// ParseError line (-1 when it is 0) / -2 for std::invalid_argument, and what() in out.
int ref_profile_record(const char* line, int lineno, char* out, size_t cap) {
  try {
    const std::string t = miso::format_profile_record(miso::parse_profile_record(line, lineno));
    std::snprintf(out, cap, "%s", t.c_str());
    return 0;
  } catch (const miso::ParseError& e) {
    std::snprintf(out, cap, "%s", e.what());
    return e.line() > 0 ? e.line() : -1;
  } catch (const std::invalid_argument& e) {
    std::snprintf(out, cap, "%s", e.what());
    return -2;
  }
}

// Raw std::mt19937_64 draws of DetRng(seed) (common.hpp:85-119), for fixture generators.
void ref_rng_raw(uint64_t seed, size_t n, uint64_t* out) {
  miso::DetRng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.raw();
}

// Config 1 (BASELINE.json configs[0], the reference CPU example): 3 jobs from
// generate_trace({job_count=3, seed}) -> simulate_mps_rates at 100/50/14 (interference) ->
// build_mps_matrix(pad_to_seven) -> predict_mig_speeds(noisy target_mae, rng_seed=seed, nonce)
// -> extrapolate_small_slices(default model) -> effective_speed -> optimize_partition.
// Outputs: truth3/mem per job (for the GPU path), est5 per job (post-zeroing), decision.
// Config 1 latency: the reference CPU example's decision chain (build_mps_matrix ->
// predict_mig_speeds -> extrapolate_small_slices -> effective_speed -> optimize_partition,
// profiles.hpp:151-167, 214-253, 370-384, 60-65; optimizer.hpp:62-115) on the anchor roster,
// repeated `reps` times on the calling thread with call nonce 1..reps. Inputs (trace, MPS rates)
// are built once outside the timed loop. Returns seconds; *checksum sums the objectives.
double ref_c1_time(uint64_t seed, int job_count, double interference, double target_mae,
                   int reps, double* checksum) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.seed = seed;
  auto tr = miso::generate_trace(spec);
  std::vector<miso::JobProfile> profs;
  for (auto& j : tr.jobs) profs.push_back(j.profile);
  for (int level : miso::kMpsLevels) miso::simulate_mps_rates(profs, level, interference);
  miso::PredictorSpec ps;
  ps.mode = miso::PredictorSpec::Mode::noisy;
  ps.target_mae = target_mae;
  ps.rng_seed = seed;
  const auto& model = default_model();
  double acc = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    auto mps = miso::build_mps_matrix(miso::pad_to_seven(profs));
    auto mig = miso::predict_mig_speeds(mps, profs, ps, static_cast<uint64_t>(r + 1));
    auto small = miso::extrapolate_small_slices(mig, model);
    std::vector<miso::JobSpeeds> jobs;
    for (int c = 0; c < job_count; ++c) {
      const auto& p = profs[c];
      miso::SpeedTable est;
      est.v = {small.at(p.job_id).f1, small.at(p.job_id).f2, mig.values[2][c], mig.values[1][c],
               mig.values[0][c]};
      miso::JobSpeeds js;
      js.job_id = p.job_id;
      for (miso::Slice k : miso::kAllSlices)
        js.speeds[k] = miso::effective_speed(est[k], k, p.mem_demand_gb, p.qos_min_slice);
      jobs.push_back(js);
    }
    auto res = miso::optimize_partition(jobs, miso::default_catalog());
    if (res) acc += res->objective;
  }
  const auto t1 = std::chrono::steady_clock::now();
  *checksum = acc;
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_c1_chain(uint64_t seed, int job_count, double interference, double target_mae,
                 uint64_t nonce, double* truth3, int* mem_gb, double* est5, int* entry,
                 uint8_t* place, double* obj) {
  miso::TraceSpec spec;
  spec.job_count = job_count;
  spec.seed = seed;
  auto tr = miso::generate_trace(spec);
  std::vector<miso::JobProfile> profs;
  for (auto& j : tr.jobs) profs.push_back(j.profile);
  for (int level : miso::kMpsLevels) miso::simulate_mps_rates(profs, level, interference);
  miso::PredictorSpec ps;
  ps.mode = miso::PredictorSpec::Mode::noisy;
  ps.target_mae = target_mae;
  ps.rng_seed = seed;
  auto mps = miso::build_mps_matrix(miso::pad_to_seven(profs));
  auto mig = miso::predict_mig_speeds(mps, profs, ps, nonce);
  auto small = miso::extrapolate_small_slices(mig, default_model());
  std::vector<miso::JobSpeeds> jobs;
  for (int c = 0; c < job_count; ++c) {
    const auto& p = profs[c];
    truth3[3 * c + 0] = p.speed_table.v[4];
    truth3[3 * c + 1] = p.speed_table.v[3];
    truth3[3 * c + 2] = p.speed_table.v[2];
    mem_gb[c] = p.mem_demand_gb;
    miso::SpeedTable est;
    est.v = {small.at(p.job_id).f1, small.at(p.job_id).f2, mig.values[2][c], mig.values[1][c],
             mig.values[0][c]};
    miso::JobSpeeds js;
    js.job_id = p.job_id;
    for (miso::Slice k : miso::kAllSlices)
      js.speeds[k] = miso::effective_speed(est[k], k, p.mem_demand_gb, p.qos_min_slice);
    for (int k = 0; k < 5; ++k) est5[5 * c + k] = js.speeds.v[k];
    jobs.push_back(js);
  }
  auto r = miso::optimize_partition(jobs, miso::default_catalog());
  if (!r) return 0;
  *entry = catalog_index(miso::default_catalog(), r->partition);
  for (int c = 0; c < job_count; ++c) place[c] = static_cast<uint8_t>(r->assignments[c].slice);
  *obj = r->objective;
  return 1;
}

}  // extern "C"
