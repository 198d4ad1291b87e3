// sim_pol_oracle.cu -- the simulator engine (sim_engine.cuh) instantiated for policy oracle: one
// TU per policy, so each kernel carries only its policy's code (and the TUs build in parallel).
#include "sim_launch.cuh"

namespace miso_b200 {

template cudaError_t launch_sim<MISO_B200_POLICY_ORACLE, false>(const SimBatch&, const SimParams&,
                                                              const ModelW&, cudaStream_t);

}  // namespace miso_b200
