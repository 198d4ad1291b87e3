// sim_pol_miso.cu -- the simulator engine (sim_engine.cuh) instantiated for policy miso: one
// TU per policy, so each kernel carries only its policy's code (and the TUs build in parallel).
#include "sim_launch.cuh"

namespace miso_b200 {

template cudaError_t launch_sim<MISO_B200_POLICY_MISO, false>(const SimBatch&, const SimParams&,
                                                              const ModelW&, cudaStream_t);

}  // namespace miso_b200
