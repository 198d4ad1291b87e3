// Experiment parity (GPU box): the reference's run_experiment_in_memory (CPU engine,
// experiment.hpp:364) and miso::b200::run_experiment_in_memory (device engine) on the same
// configs must give byte-identical write_csv output and summarize().dump(2) text, and
// bit-identical per-row scalars. Prints one line per config and exits non-zero on a mismatch.
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "miso/experiment.hpp"
#include "miso_b200_experiment.hpp"

namespace {

struct Case {
  const char* name;
  miso::ExperimentConfig cfg;
};

std::string csv(const miso::ExperimentResult& r) {
  std::ostringstream o;
  miso::write_csv(r, o);
  return o.str();
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

}  // namespace

int main() {
  std::vector<Case> cases;
  {
    miso::ExperimentConfig c;  // all four policies, MAE sweep (noisy predictor)
    c.cluster_size = 8;
    c.trials = 6;
    c.base_seed = 300;
    c.trace_spec.job_count = 80;
    c.trace_spec.lambda_s = 30;
    c.predictor.mode = miso::PredictorSpec::Mode::noisy;
    c.sweep_param = "target_mae";
    c.sweep_values = {0.017, 0.09};
    cases.push_back({"mae-sweep", c});
  }
  {
    miso::ExperimentConfig c;  // lambda sweep, implicit nopart baseline, drift re-profiling
    c.cluster_size = 6;
    c.trials = 4;
    c.base_seed = 9;
    c.trace_spec.job_count = 60;
    c.policies = {miso::Policy::optsta, miso::Policy::miso};
    c.predictor.mode = miso::PredictorSpec::Mode::noisy;
    c.reprofile_drift_threshold = 0.05;
    c.sweep_param = "lambda_s";
    c.sweep_values = {20, 60};
    cases.push_back({"lambda-sweep", c});
  }
  {
    miso::ExperimentConfig c;  // checkpoint sweep, oracle predictor, uniform durations
    c.cluster_size = 10;
    c.trials = 5;
    c.base_seed = 77;
    c.trace_spec.job_count = 100;
    c.trace_spec.lambda_s = 15;
    c.trace_spec.duration_dist.kind = miso::DurationDist::Kind::uniform;
    c.sweep_param = "checkpoint_restart_s";
    c.sweep_values = {0, 30, 120};
    cases.push_back({"ckpt-sweep", c});
  }
  int bad = 0;
  for (auto& k : cases) {
    k.cfg.workers = 8;
    auto ref = miso::run_experiment_in_memory(k.cfg);
    auto dev = miso::b200::run_experiment_in_memory(k.cfg);
    const bool csv_ok = csv(ref) == csv(dev);
    const bool json_ok = miso::summarize(ref).dump(2) == miso::summarize(dev).dump(2);
    bool rows_ok = ref.rows.size() == dev.rows.size();
    for (size_t i = 0; rows_ok && i < ref.rows.size(); ++i) {
      const auto& a = ref.rows[i].report;
      const auto& b = dev.rows[i].report;
      rows_ok = a.policy == b.policy && a.seed == b.seed && a.completed == b.completed &&
                same_bits(a.avg_jct_s, b.avg_jct_s) && same_bits(a.makespan_s, b.makespan_s) &&
                same_bits(a.stp_time_avg, b.stp_time_avg) && a.jct_sorted == b.jct_sorted &&
                a.stp_series == b.stp_series && a.repartitions == b.repartitions &&
                a.migrations == b.migrations && a.mps_sessions == b.mps_sessions &&
                same_bits(ref.rows[i].jct_norm, dev.rows[i].jct_norm) &&
                miso::format_report(a) == miso::format_report(b);
    }
    std::printf("%s: rows=%zu csv=%s json=%s reports=%s\n", k.name, ref.rows.size(),
                csv_ok ? "identical" : "DIFFER", json_ok ? "identical" : "DIFFER",
                rows_ok ? "identical" : "DIFFER");
    bad += !(csv_ok && json_ok && rows_ok);
  }
  std::printf(bad ? "PARITY FAILED\n" : "PARITY OK\n");
  return bad ? 1 : 0;
}
