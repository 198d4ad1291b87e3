// miso_b200_profiles.hpp -- the predictor half of the binding: the reference's
// predict_mig_speeds (profiles.hpp:214-253) and extrapolate_small_slices (:370-384) on the B200
// predictor kernel (include/miso_b200.h, miso_b200_predict_host). Include after
// "miso/profiles.hpp". Same signatures, argument meaning, results (bit-identical speeds) and
// exceptions:
//
//   miso::b200::predict_mig_speeds(mps, truth, spec, call_nonce)  == predict_mig_speeds
//   miso::b200::extrapolate_small_slices(mig, model)              == extrapolate_small_slices
#pragma once

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "miso/profiles.hpp"
#include "miso_b200_ref.hpp"

namespace miso {
namespace b200 {

// Drop-in for predict_mig_speeds (profiles.hpp:214-216): one MPS group of 7 columns on the
// device (dummy columns are computed from a placeholder and overwritten with 1.0, as the
// reference pads them; each column's noise stream depends only on its own index).
inline ProfileMatrix predict_mig_speeds(const ProfileMatrix& mps, const std::vector<JobProfile>& truth,
                                        const PredictorSpec& spec, uint64_t call_nonce = 0) {
  if (mps.kind != ProfileMatrix::Kind::mps)
    throw std::invalid_argument("predict_mig_speeds expects an mps-kind matrix");
  validate_predictor_spec(spec);
  ProfileMatrix out;
  out.kind = ProfileMatrix::Kind::mig;
  out.job_ids = mps.job_ids;
  out.dummy = mps.dummy;
  double t3[21];
  size_t t = 0;
  for (int c = 0; c < 7; ++c) {
    if (mps.dummy[static_cast<size_t>(c)]) {
      t3[3 * c] = t3[3 * c + 1] = t3[3 * c + 2] = 1.0;
      continue;
    }
    if (t >= truth.size() || truth[t].job_id != mps.job_ids[static_cast<size_t>(c)])
      throw std::invalid_argument("truth profiles misaligned with mps matrix columns");
    const JobProfile& job = truth[t++];
    t3[3 * c] = job.speed_table[Slice::k7g];
    t3[3 * c + 1] = job.speed_table[Slice::k4g];
    t3[3 * c + 2] = job.speed_table[Slice::k3g];
  }
  if (t != truth.size())
    throw std::invalid_argument("truth profiles misaligned with mps matrix columns");
  double e5[35];
  {
    Device& d = Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    Device::check(miso_b200_predict_host(d.ctx(), t3, 7, 7, call_nonce, spec.rng_seed,
                                         spec.mode == PredictorSpec::Mode::noisy ? 1 : 0,
                                         spec.target_mae, nullptr, nullptr, e5));
  }
  for (int c = 0; c < 7; ++c)
    for (int r = 0; r < 3; ++r)  // rows 7g, 4g, 3g = kinds 4, 3, 2 of the speed table
      out.values[static_cast<size_t>(r)][static_cast<size_t>(c)] =
          mps.dummy[static_cast<size_t>(c)] ? 1.0 : e5[5 * c + 4 - r];
  return out;
}

// Drop-in for extrapolate_small_slices (profiles.hpp:370-371): the model's weights applied on
// the device to the matrix rows as given.
inline std::map<std::string, SmallSliceSpeeds> extrapolate_small_slices(const ProfileMatrix& mig,
                                                                        const LinearMap& model) {
  if (mig.kind != ProfileMatrix::Kind::mig)
    throw std::invalid_argument("extrapolate_small_slices expects a mig-kind matrix");
  if (!model.fitted) throw std::logic_error("small-slice model is not fitted");
  double t3[21], e5[35];
  for (int c = 0; c < 7; ++c)
    for (int r = 0; r < 3; ++r) t3[3 * c + r] = mig.values[static_cast<size_t>(r)][static_cast<size_t>(c)];
  {
    Device& d = Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    Device::check(miso_b200_predict_host(d.ctx(), t3, 7, 7, 0, 0, 2, 0.0, model.w_2g.data(),
                                         model.w_1g.data(), e5));
  }
  std::map<std::string, SmallSliceSpeeds> out;
  for (int c = 0; c < 7; ++c) {
    SmallSliceSpeeds s;
    s.f2 = e5[5 * c + 1];
    s.f1 = e5[5 * c];
    out[mig.job_ids[static_cast<size_t>(c)]] = s;
  }
  return out;
}

}  // namespace b200
}  // namespace miso
