// sim_pol_optsta.cu -- the simulator engine (sim_engine.cuh) instantiated for policy optsta: one
// TU per policy, so each kernel carries only its policy's code (and the TUs build in parallel).
#include "sim_launch.cuh"

namespace miso_b200 {

template cudaError_t launch_sim<MISO_B200_POLICY_OPTSTA, false>(const SimBatch&, const SimParams&,
                                                              const ModelW&, cudaStream_t);
// the chosen-only best-static search's candidate runs (miso_b200_simulate_batch_pruned)
template cudaError_t launch_sim<MISO_B200_POLICY_OPTSTA, true>(const SimBatch&, const SimParams&,
                                                              const ModelW&, cudaStream_t);

}  // namespace miso_b200
