// Force-included (-include) before the reference's topology_test.cpp: the reference headers are
// compiled first (their real definitions), then later mentions of max_spare_slice_for in the
// test file resolve to the B200 binding (include/miso_b200_ref.hpp), i.e. to the spare-slice
// table the device simulator's placement reads.
#pragma once
#include "miso/common.hpp"
#include "miso/topology.hpp"
#include "miso/optimizer.hpp"
#include "miso_b200_ref.hpp"
namespace miso {
inline std::optional<Slice> b200_max_spare_slice_for_dropin(const PartitionCatalog& catalog,
                                                            std::vector<Slice> pinned) {
  return b200::max_spare_slice_for(catalog, std::move(pinned));
}
}  // namespace miso
#define max_spare_slice_for b200_max_spare_slice_for_dropin
