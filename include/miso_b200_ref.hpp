// miso_b200_ref.hpp -- the binding a maintainer of the reference library adds to route its
// hot path to the B200 C ABI (include/miso_b200.h). Header-only, C++20, to be included after
// the reference's own headers ("miso/optimizer.hpp", "miso/sim.hpp"): it uses the reference's
// types (JobSpeeds, PartitionCatalog, AssignmentVector, ...) unchanged and keeps each
// function's signature, argument meaning and error behaviour:
//
//   miso::b200::optimize_partition(jobs, catalog)   == optimize_partition (optimizer.hpp:62-63)
//   miso::b200::optimize_partition_batch(batch, catalog)   many independent rosters, one launch
//
// Errors: std::invalid_argument for m outside 1..7 (optimizer.hpp:65-66), std::nullopt when no
// assignment is valid (:102), std::runtime_error for device failures.
#pragma once

#include <cstdint>
#include <cstring>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "miso/optimizer.hpp"
#include "miso_b200.h"

namespace miso {
namespace b200 {

class Device {
 public:
  static Device& get(int device = 0) {
    static Device d(device);
    return d;
  }
  miso_b200_ctx* ctx() { return ctx_; }
  std::mutex& mu() { return mu_; }

  // Installs `catalog` on the context when it differs from the active one.
  void use_catalog(const PartitionCatalog& catalog) {
    std::vector<uint8_t> counts;
    counts.reserve(catalog.entries.size() * 5);
    for (const auto& e : catalog.entries)
      for (int k = 0; k < 5; ++k) counts.push_back(e.counts()[k]);
    if (counts == active_) return;
    check(miso_b200_set_catalog(ctx_, counts.data(), static_cast<int>(catalog.entries.size())));
    active_ = std::move(counts);
  }

  static void check(int rc) {
    if (rc == MISO_B200_E_INVALID) throw std::invalid_argument(miso_b200_last_error());
    if (rc < 0) throw std::runtime_error(std::string("miso_b200: ") + miso_b200_last_error());
  }

 private:
  explicit Device(int device) { check(miso_b200_create(device, &ctx_)); }
  ~Device() { miso_b200_destroy(ctx_); }
  miso_b200_ctx* ctx_ = nullptr;
  std::vector<uint8_t> active_;
  std::mutex mu_;
};

namespace detail {

inline std::optional<AssignmentVector> decode(miso_b200_ctx* ctx, const std::vector<JobSpeeds>& jobs,
                                              const PartitionCatalog& catalog, uint8_t cand,
                                              double obj) {
  if (cand == MISO_B200_CAND_BAD_M)
    throw std::invalid_argument("optimize_partition needs 1..7 jobs, got " +
                                std::to_string(jobs.size()));
  if (cand == MISO_B200_CAND_INFEASIBLE) return std::nullopt;
  int entry = -1, m = 0;
  uint8_t place[7];
  Device::check(miso_b200_candidate(ctx, cand, &entry, &m, place));
  AssignmentVector out;
  out.partition = catalog.entries.at(static_cast<size_t>(entry));
  out.objective = obj;
  out.assignments.reserve(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i) {
    Assignment a;
    a.job_id = jobs[i].job_id;
    a.slice = kAllSlices[place[i]];
    a.speed = jobs[i].speeds.v[place[i]];
    out.assignments.push_back(std::move(a));
  }
  return out;
}

}  // namespace detail

// Drop-in for optimize_partition (optimizer.hpp:62-115).
inline std::optional<AssignmentVector> optimize_partition(const std::vector<JobSpeeds>& jobs,
                                                          const PartitionCatalog& catalog) {
  const size_t m = jobs.size();
  if (m < 1 || m > 7)
    throw std::invalid_argument("optimize_partition needs 1..7 jobs, got " + std::to_string(m));
  Device& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  d.use_catalog(catalog);
  double speeds[35];
  for (size_t i = 0; i < m; ++i) std::memcpy(speeds + 5 * i, jobs[i].speeds.v.data(), 40);
  int entry = -1;
  uint8_t place[7];
  double obj = 0;
  const int r = miso_b200_optimize(d.ctx(), speeds, static_cast<int>(m), &entry, place, &obj);
  Device::check(r);
  if (r == 0) return std::nullopt;
  AssignmentVector out;
  out.partition = catalog.entries.at(static_cast<size_t>(entry));
  out.objective = obj;
  for (size_t i = 0; i < m; ++i) {
    Assignment a;
    a.job_id = jobs[i].job_id;
    a.slice = kAllSlices[place[i]];
    a.speed = jobs[i].speeds.v[place[i]];
    out.assignments.push_back(std::move(a));
  }
  return out;
}

// Many independent rosters in one launch (host buffers; H2D/search/D2H pipelined inside).
// Rosters with m outside 1..7 throw std::invalid_argument like the scalar call.
inline std::vector<std::optional<AssignmentVector>> optimize_partition_batch(
    const std::vector<std::vector<JobSpeeds>>& batch, const PartitionCatalog& catalog) {
  Device& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  d.use_catalog(catalog);
  std::vector<uint32_t> offsets(batch.size() + 1, 0);
  for (size_t i = 0; i < batch.size(); ++i)
    offsets[i + 1] = offsets[i] + static_cast<uint32_t>(batch[i].size());
  std::vector<double> speeds(size_t(offsets.back()) * 5 + 1);
  for (size_t i = 0; i < batch.size(); ++i)
    for (size_t j = 0; j < batch[i].size(); ++j)
      std::memcpy(&speeds[(offsets[i] + j) * 5], batch[i][j].speeds.v.data(), 40);
  std::vector<uint8_t> cand(batch.size());
  std::vector<double> obj(batch.size());
  Device::check(miso_b200_optimize_batch_host(d.ctx(), speeds.data(), offsets.data(), batch.size(),
                                              cand.data(), obj.data()));
  std::vector<std::optional<AssignmentVector>> out;
  out.reserve(batch.size());
  for (size_t i = 0; i < batch.size(); ++i)
    out.push_back(detail::decode(d.ctx(), batch[i], catalog, cand[i], obj[i]));
  return out;
}

// Drop-in for max_spare_slice_for (topology.hpp:227-252), answered from the spare-slice table
// the simulator's placement reads on the device (miso_b200_max_spare_slice).
inline std::optional<Slice> max_spare_slice_for(const PartitionCatalog& catalog,
                                                std::vector<Slice> pinned_min_kinds) {
  std::vector<uint8_t> kinds;
  kinds.reserve(pinned_min_kinds.size());
  for (Slice s : pinned_min_kinds) kinds.push_back(static_cast<uint8_t>(slice_index(s)));
  Device& d = Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  d.use_catalog(catalog);
  int kind = -1;
  Device::check(miso_b200_max_spare_slice(d.ctx(), kinds.data(), static_cast<int>(kinds.size()), &kind));
  if (kind < 0) return std::nullopt;
  return kAllSlices[static_cast<size_t>(kind)];
}

}  // namespace b200
}  // namespace miso
