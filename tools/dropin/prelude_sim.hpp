// Force-included (-include) before a reference simulator/experiment test file to run it against
// the B200 library: every reference header is compiled first (their real definitions, including
// the reference's own run_experiment / optsta_search), then later mentions of run_simulation,
// best_static_partition, run_experiment_in_memory, run_experiment and optsta_search in the
// test file resolve to the B200 binding (include/miso_b200_sim.hpp, miso_b200_experiment.hpp),
// so no test reaches the reference's CPU engine.
#pragma once
#include "miso/common.hpp"
#include "miso/topology.hpp"
#include "miso/profiles.hpp"
#include "miso/optimizer.hpp"
#include "miso/workload.hpp"
#include "miso/sim.hpp"
#include "miso/experiment.hpp"
#include "miso_b200_experiment.hpp"
namespace miso {
inline MetricsReport b200_run_simulation_dropin(const JobTrace& t, const SimOptions& o) {
  return b200::run_simulation(t, o);
}
inline MetricsReport b200_run_simulation_dropin(const JobTrace& t, int n, Policy p,
                                                const OverheadSpec& o, const PredictorSpec& ps,
                                                const std::optional<PartitionConfig>& s = std::nullopt) {
  return b200::run_simulation(t, n, p, o, ps, s);
}
inline StaticSearchResult b200_best_static_partition_dropin(const JobTrace& t, int n,
                                                            const OverheadSpec& o,
                                                            const PartitionCatalog& c = default_catalog()) {
  return b200::best_static_partition(t, n, o, c);
}
inline ExperimentResult b200_run_experiment_in_memory_dropin(const ExperimentConfig& c) {
  return b200::run_experiment_in_memory(c);
}
inline ExperimentResult b200_run_experiment_dropin(const ExperimentConfig& c) {
  return b200::run_experiment(c);
}
inline StaticSearchResult b200_optsta_search_dropin(const ExperimentConfig& c) {
  return b200::optsta_search(c);
}
}  // namespace miso
#define run_simulation b200_run_simulation_dropin
#define best_static_partition b200_best_static_partition_dropin
#define run_experiment_in_memory b200_run_experiment_in_memory_dropin
#define run_experiment b200_run_experiment_dropin
#define optsta_search b200_optsta_search_dropin
