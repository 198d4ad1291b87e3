// Force-included (-include) before the reference's profiles_test.cpp to run it against the
// B200 predictor: the reference headers are compiled first (their real definitions), then
// later mentions of predict_mig_speeds and extrapolate_small_slices in the test file resolve
// to the B200 binding (include/miso_b200_profiles.hpp).
#pragma once
#include "miso/common.hpp"
#include "miso/topology.hpp"
#include "miso/profiles.hpp"
#include "miso/optimizer.hpp"
#include "miso/workload.hpp"
#include "miso/sim.hpp"
#include "miso_b200_profiles.hpp"
namespace miso {
inline ProfileMatrix b200_predict_mig_speeds_dropin(const ProfileMatrix& mps,
                                                    const std::vector<JobProfile>& truth,
                                                    const PredictorSpec& spec, uint64_t nonce = 0) {
  return b200::predict_mig_speeds(mps, truth, spec, nonce);
}
inline std::map<std::string, SmallSliceSpeeds> b200_extrapolate_small_slices_dropin(
    const ProfileMatrix& mig, const LinearMap& model) {
  return b200::extrapolate_small_slices(mig, model);
}
}  // namespace miso
#define predict_mig_speeds b200_predict_mig_speeds_dropin
#define extrapolate_small_slices b200_extrapolate_small_slices_dropin
