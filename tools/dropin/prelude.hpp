// Force-included (-include) before a reference test file to run it against the B200 library:
// the reference optimizer is compiled first (its real definition), then every later mention of
// `optimize_partition` in the test file resolves to the B200 binding (include/miso_b200_ref.hpp).
#pragma once
#include "miso/optimizer.hpp"
#include "miso_b200_ref.hpp"
namespace miso {
inline std::optional<AssignmentVector> b200_optimize_partition_dropin(
    const std::vector<JobSpeeds>& jobs, const PartitionCatalog& catalog) {
  return b200::optimize_partition(jobs, catalog);
}
}  // namespace miso
#define optimize_partition b200_optimize_partition_dropin
