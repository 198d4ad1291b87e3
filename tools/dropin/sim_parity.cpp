// Simulator parity (GPU box): the reference's run_simulation (CPU engine, sim.hpp:976) and
// miso::b200::run_simulation (device engine) on generated traces with multi-instance jobs
// (clones), QoS floors and every policy: format_report text (scalars, per-job phases incl.
// clones, STP series) and the event-log text must be byte-identical. Exit 0 iff all match.
#include <cstdio>
#include <sstream>
#include <string>

#include "miso/sim.hpp"
#include "miso/workload.hpp"
#include "miso_b200_sim.hpp"

int main() {
  int bad = 0, runs = 0;
  for (int trial = 0; trial < 12; ++trial) {
    miso::TraceSpec spec;
    spec.job_count = 40 + 10 * (trial % 3);
    spec.lambda_s = 20 + 10 * (trial % 4);
    spec.seed = 7100 + static_cast<uint64_t>(trial);
    auto trace = miso::generate_trace(spec);
    trace.jobs[3].profile.instance_count = 3;
    trace.jobs[11].profile.instance_count = 2;
    if (trial % 2) trace.jobs[20].profile.instance_count = 4;
    if (trial % 3 == 0) trace.jobs[5].profile.qos_min_slice = miso::Slice::k3g;
    const int cluster = 2 + trial % 3;
    auto st = miso::best_static_partition(trace, cluster, miso::OverheadSpec{});
    auto st_dev = miso::b200::best_static_partition(trace, cluster, miso::OverheadSpec{});
    if (!(st.chosen == st_dev.chosen)) {
      std::printf("trial %d: static partition differs\n", trial);
      ++bad;
    }
    for (miso::Policy p : {miso::Policy::nopart, miso::Policy::optsta, miso::Policy::oracle,
                           miso::Policy::miso}) {
      miso::SimOptions o;
      o.policy = p;
      o.cluster_size = cluster;
      o.predictor.mode = miso::PredictorSpec::Mode::noisy;
      o.predictor.target_mae = 0.09;
      o.predictor.rng_seed = spec.seed;
      if (p == miso::Policy::optsta) o.static_partition = st.chosen;
      std::ostringstream log_ref, log_dev;
      o.event_log = &log_ref;
      auto r = miso::run_simulation(trace, o);
      o.event_log = &log_dev;
      auto d = miso::b200::run_simulation(trace, o);
      const bool rep_ok = miso::format_report(r) == miso::format_report(d);
      const bool log_ok = log_ref.str() == log_dev.str();
      ++runs;
      if (!rep_ok || !log_ok) {
        std::printf("trial %d policy %s: report %s, log %s (jobs %zu vs %zu)\n", trial,
                    miso::policy_label(p), rep_ok ? "ok" : "DIFFER", log_ok ? "ok" : "DIFFER",
                    r.per_job.size(), d.per_job.size());
        ++bad;
      }
    }
  }
  // A caller-fitted small-slice model (SimOptions::small_slice_model, sim.hpp:88, 894-896): a
  // model fitted on another corpus drives the miso/oracle estimates on both engines.
  const miso::LinearMap custom = miso::fit_small_slice_model(miso::make_training_corpus(400, 0xc0ffee));
  for (int trial = 0; trial < 4; ++trial) {
    miso::TraceSpec spec;
    spec.job_count = 60;
    spec.lambda_s = 25;
    spec.seed = 9100 + static_cast<uint64_t>(trial);
    auto trace = miso::generate_trace(spec);
    for (miso::Policy p : {miso::Policy::oracle, miso::Policy::miso}) {
      miso::SimOptions o;
      o.policy = p;
      o.cluster_size = 3;
      o.predictor.mode = miso::PredictorSpec::Mode::noisy;
      o.predictor.rng_seed = spec.seed;
      o.small_slice_model = custom;
      std::ostringstream log_ref, log_dev;
      o.event_log = &log_ref;
      auto r = miso::run_simulation(trace, o);
      o.event_log = &log_dev;
      auto d = miso::b200::run_simulation(trace, o);
      ++runs;
      if (miso::format_report(r) != miso::format_report(d) || log_ref.str() != log_dev.str()) {
        std::printf("custom model trial %d policy %s: DIFFER\n", trial, miso::policy_label(p));
        ++bad;
      }
    }
  }
  // max_events (sim.hpp:224) counts every heap pop, stale ones included: find the reference's
  // smallest budget that completes (= its pop count) and check both sides of it on the device.
  for (int trial = 0; trial < 3; ++trial) {
    miso::TraceSpec spec;
    spec.job_count = 30;
    spec.lambda_s = 15;
    spec.seed = 9300 + static_cast<uint64_t>(trial);
    auto trace = miso::generate_trace(spec);
    for (miso::Policy p : {miso::Policy::optsta, miso::Policy::miso}) {
      miso::SimOptions o;
      o.policy = p;
      o.cluster_size = 2;
      o.predictor.mode = miso::PredictorSpec::Mode::noisy;
      o.predictor.rng_seed = spec.seed;
      if (p == miso::Policy::optsta) o.static_partition = miso::default_catalog().entries[8];
      auto completes = [&](bool device, uint64_t budget) {
        o.max_events = budget;
        try {
          if (device) miso::b200::run_simulation(trace, o);
          else miso::run_simulation(trace, o);
          return 1;
        } catch (const miso::SimInvariantError& e) {
          return std::string(e.what()) == "event budget exhausted" ? 0 : -1;
        }
      };
      uint64_t lo = 1, hi = 1;
      while (completes(false, hi) == 0) hi *= 2;
      while (lo < hi) {  // smallest budget that completes
        const uint64_t mid = (lo + hi) / 2;
        if (completes(false, mid) == 1) hi = mid;
        else lo = mid + 1;
      }
      const int at = completes(true, lo), below = completes(true, lo - 1);
      ++runs;
      if (at != 1 || below != 0) {
        std::printf("max_events trial %d policy %s: reference needs %llu pops; device %d at it, %d below\n",
                    trial, miso::policy_label(p), static_cast<unsigned long long>(lo), at, below);
        ++bad;
      }
    }
  }
  std::printf("%d runs, %d mismatches\n%s\n", runs, bad, bad ? "SIM PARITY FAILED" : "SIM PARITY OK");
  return bad ? 1 : 0;
}
