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

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "miso/optimizer.hpp"
#include "miso_b200.h"

namespace miso {
namespace b200 {

// One context per CUDA device, created on first use and shared by every caller in the process
// (a context serves one host thread at a time: callers hold mu()). Batch calls spread their
// work over all() -- every visible device, or the first MISO_B200_DEVICES of them.
class Device {
 public:
  static constexpr int kMaxDevices = 64;

  static Device& get(int device = 0) {
    if (device < 0 || device >= kMaxDevices) throw std::invalid_argument("miso_b200: device index");
    static std::mutex reg_mu;
    static std::unique_ptr<Device> reg[kMaxDevices];
    std::lock_guard<std::mutex> lock(reg_mu);
    if (!reg[device]) reg[device].reset(new Device(device));
    return *reg[device];
  }

  static int count() {
    static const int n = [] {
      int d = miso_b200_device_count();
      if (const char* e = std::getenv("MISO_B200_DEVICES")) d = std::min(d, std::max(1, std::atoi(e)));
      return std::max(1, std::min(d, kMaxDevices));
    }();
    return n;
  }

  static std::vector<Device*> all() {
    std::vector<Device*> v;
    for (int i = 0; i < count(); ++i) v.push_back(&get(i));
    return v;
  }

  miso_b200_ctx* ctx() { return ctx_; }
  std::mutex& mu() { return mu_; }

  // Installs `catalog` on the context when it differs from the active one. Returns false for
  // an empty catalog (nothing installed: callers answer it as the reference does -- no entry).
  bool use_catalog(const PartitionCatalog& catalog) {
    if (catalog.entries.empty()) return false;
    std::vector<uint8_t> counts;
    counts.reserve(catalog.entries.size() * 5);
    for (const auto& e : catalog.entries)
      for (int k = 0; k < 5; ++k) counts.push_back(e.counts()[k]);
    if (counts == active_) return true;
    check(miso_b200_set_catalog(ctx_, counts.data(), static_cast<int>(catalog.entries.size())));
    active_ = std::move(counts);
    return true;
  }

  static void check(int rc) {
    if (rc == MISO_B200_E_INVALID) throw std::invalid_argument(miso_b200_last_error());
    if (rc < 0) throw std::runtime_error(std::string("miso_b200: ") + miso_b200_last_error());
  }

  ~Device() { miso_b200_destroy(ctx_); }

 private:
  explicit Device(int device) {
    check(miso_b200_create(device, &ctx_));
    uint8_t c[36 * 5];  // the context's real active catalog
    const int n = miso_b200_get_catalog(ctx_, c);
    active_.assign(c, c + 5 * std::max(0, n));
  }
  miso_b200_ctx* ctx_ = nullptr;
  std::vector<uint8_t> active_;
  std::mutex mu_;
};

// Holds every device's lock (in index order) for a call spread over Device::all(), with the
// catalog installed on each. contexts() lists their contexts in the same order.
class AllDevices {
 public:
  explicit AllDevices(const PartitionCatalog& catalog) : devs_(Device::all()) {
    for (Device* d : devs_) locks_.emplace_back(d->mu());
    for (Device* d : devs_) ok_ = d->use_catalog(catalog);
    for (Device* d : devs_) ctxs_.push_back(d->ctx());
  }
  bool catalog_ok() const { return ok_; }
  miso_b200_ctx* const* contexts() const { return ctxs_.data(); }
  int size() const { return static_cast<int>(ctxs_.size()); }

 private:
  std::vector<Device*> devs_;
  std::vector<std::unique_lock<std::mutex>> locks_;
  std::vector<miso_b200_ctx*> ctxs_;
  bool ok_ = true;
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
  if (!d.use_catalog(catalog)) return std::nullopt;  // no entry can host the jobs (:102)
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

// Many independent rosters in one call (host buffers; H2D/search/D2H pipelined inside), spread
// over every device (miso_b200_optimize_batch_sharded: contiguous instance ranges, one host
// thread per device). Rosters with m outside 1..7 throw std::invalid_argument like the scalar
// call.
inline std::vector<std::optional<AssignmentVector>> optimize_partition_batch(
    const std::vector<std::vector<JobSpeeds>>& batch, const PartitionCatalog& catalog) {
  AllDevices all(catalog);
  if (!all.catalog_ok()) {  // empty catalog: every roster is nullopt (or invalid_argument)
    std::vector<std::optional<AssignmentVector>> out;
    for (const auto& r : batch) {
      if (r.empty() || r.size() > 7)
        throw std::invalid_argument("optimize_partition needs 1..7 jobs, got " + std::to_string(r.size()));
      out.push_back(std::nullopt);
    }
    return out;
  }
  std::vector<uint32_t> offsets(batch.size() + 1, 0);
  for (size_t i = 0; i < batch.size(); ++i)
    offsets[i + 1] = offsets[i] + static_cast<uint32_t>(batch[i].size());
  std::vector<double> speeds(size_t(offsets.back()) * 5 + 1);
  for (size_t i = 0; i < batch.size(); ++i)
    for (size_t j = 0; j < batch[i].size(); ++j)
      std::memcpy(&speeds[(offsets[i] + j) * 5], batch[i][j].speeds.v.data(), 40);
  std::vector<uint8_t> cand(batch.size());
  std::vector<double> obj(batch.size());
  Device::check(miso_b200_optimize_batch_sharded(all.contexts(), all.size(), speeds.data(),
                                                 offsets.data(), batch.size(), cand.data(),
                                                 obj.data()));
  std::vector<std::optional<AssignmentVector>> out;
  out.reserve(batch.size());
  for (size_t i = 0; i < batch.size(); ++i)
    out.push_back(detail::decode(all.contexts()[0], batch[i], catalog, cand[i], obj[i]));
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
  if (!d.use_catalog(catalog)) return std::nullopt;  // no entry to spare a slice in
  int kind = -1;
  Device::check(miso_b200_max_spare_slice(d.ctx(), kinds.data(), static_cast<int>(kinds.size()), &kind));
  if (kind < 0) return std::nullopt;
  return kAllSlices[static_cast<size_t>(kind)];
}

}  // namespace b200
}  // namespace miso
